"""NEXT-1 elimination regimes side by side: one Newton step (evaluation + elimination + back
substitution + update) of single points and small batches through each applicable regime
(PHC_NEWTON_* hooks), CUDA events after warm-up.  Prints one JSON line per (case, regime)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1109_0545_b200 as phc  # noqa: E402
from synthetic import config_system, random_system  # noqa: E402

REGIMES = {
    "cta": {"PHC_NEWTON_CLUSTER": "0", "PHC_NEWTON_WARP": "0"},
    "cluster2": {"PHC_NEWTON_CLUSTER": "1", "PHC_NEWTON_CLUSTER_SIZE": "2"},
    "cluster4": {"PHC_NEWTON_CLUSTER": "1", "PHC_NEWTON_CLUSTER_SIZE": "4"},
    "cluster8": {"PHC_NEWTON_CLUSTER": "1", "PHC_NEWTON_CLUSTER_SIZE": "8"},
    "coop": {"PHC_NEWTON_GLOBAL": "1", "PHC_NEWTON_COOP": "1"},
}
KEYS = ("PHC_NEWTON_CLUSTER", "PHC_NEWTON_CLUSTER_SIZE", "PHC_NEWTON_WARP", "PHC_NEWTON_GLOBAL", "PHC_NEWTON_COOP")


def timed(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


cases = [("c3", *config_system("c3", seed=1)), ("qd56", *random_system(56, 56, 20, 5, 4, seed=1)),
         ("qd64", *random_system(64, 64, 24, 5, 4, seed=1)), ("dd64", *random_system(64, 64, 24, 5, 2, seed=1))]
for name, s, X in cases:
    h = phc.System(s)
    Xd = torch.from_numpy(X).cuda()
    Xn = torch.empty_like(Xd)
    t_eval = timed(lambda: h.eval_batch(Xd), 20)
    ref = None
    for rname, env in REGIMES.items():
        for k in KEYS:
            os.environ.pop(k, None)
        os.environ.update(env)
        try:
            t = timed(lambda: h.newton_step(Xd, Xn), 20)
        except Exception as e:  # noqa: BLE001  (regime not applicable at this size)
            print(json.dumps(dict(case=name, regime=rname, error=str(e)[:80])), flush=True)
            continue
        out = Xn.clone()
        same = None if ref is None else bool(torch.equal(out, ref))
        ref = out if ref is None else ref
        print(json.dumps(dict(case=name, n=s.n_var, L=s.limbs, regime=rname, ms_step=round(t, 4),
                              ms_eval=round(t_eval, 4), ms_solve=round(t - t_eval, 4), bitwise_equal_first=same)),
              flush=True)
