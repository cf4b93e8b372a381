"""NEXT-1 batch elimination A/B: one Newton step on the batch config (65,536 points, n = 32,
DD) with the warp kernel, and the CTA kernel at 64 / 128 / 256 threads per point
(PHC_NEWTON_WARP, PHC_NEWTON_THREADS hooks); CUDA events after warm-up."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1109_0545_b200 as phc  # noqa: E402
from synthetic import config_system  # noqa: E402

s, X = config_system("batch", seed=1)
h = phc.System(s)
Xd = torch.from_numpy(X).cuda()
Xn = torch.empty_like(Xd)


def timed(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    b.synchronize()
    return a.elapsed_time(b) / reps


te = timed(lambda: h.eval_batch(Xd))
ref = None
for name, env in (("cta128", {"PHC_NEWTON_WARP": "0", "PHC_NEWTON_THREADS": "128"}),
                  ("cta64", {"PHC_NEWTON_WARP": "0", "PHC_NEWTON_THREADS": "64"}),
                  ("cta256", {"PHC_NEWTON_WARP": "0", "PHC_NEWTON_THREADS": "256"}),
                  ("warp", {"PHC_NEWTON_WARP": "1"})):
    for k in ("PHC_NEWTON_WARP", "PHC_NEWTON_THREADS"):
        os.environ.pop(k, None)
    os.environ.update(env)
    t = timed(lambda: h.newton_step(Xd, Xn))
    same = None if ref is None else bool(torch.equal(Xn, ref))
    ref = Xn.clone() if ref is None else ref
    print(json.dumps(dict(regime=name, ms_step=t, ms_eval=te, ms_elim=t - te, bitwise_equal_first=same)), flush=True)
