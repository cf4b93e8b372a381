"""Table 6 analog (§7): the "new" homotopy evaluator (t through the
coefficients, phc_eval_homotopy_batch) against the "old" one (t as variable n+1,
phc_homotopy_old_create), same homotopy, same points, per-eval time on one B200.
The paper's speedups (8.56-15.56, "pure" 2.85-5.19 after dividing by 3) mix in its
other algorithmic changes; here only the t handling differs."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1109_0545_b200 as phc  # noqa: E402
from synthetic import config_system, homotopy_target, random_t  # noqa: E402


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


for name, P in (("c2", 1), ("c2", 4096), ("c3", 1), ("c3", 1024), ("batch", 65536)):
    s, X = config_system(name, seed=1, points=P, workers=8)
    cf = homotopy_target(s, seed=2, workers=8)
    T = random_t(P, s.limbs, seed=3)
    new = phc.System(s, coeff_target=cf)
    old = phc.System(s, coeff_target=cf, old_homotopy=True)
    Xd, Td = torch.from_numpy(X).cuda(), torch.from_numpy(T).cuda()
    Xe = np.zeros((P, s.n_var + 1, 2, s.limbs))
    Xe[:, :s.n_var] = X
    Xe[:, s.n_var, 0, :] = T
    Xed = torch.from_numpy(Xe).cuda()
    F = torch.empty((P, s.n_eq, 2, s.limbs), dtype=torch.float64, device="cuda")
    J = torch.empty((P, s.n_eq, s.n_var, 2, s.limbs), dtype=torch.float64, device="cuda")
    Jo = torch.empty((P, s.n_eq, s.n_var + 1, 2, s.limbs), dtype=torch.float64, device="cuda")
    reps = 200 if P == 1 else 5
    t_new = timed(lambda: new.eval_homotopy_batch(Xd, Td, F, J), reps)
    t_plain = timed(lambda: new.eval_batch(Xd, F, J), reps)
    t_old = timed(lambda: old.eval_batch(Xed, F, Jo), reps)
    print(json.dumps(dict(config=name, points=P, precision="cDD" if s.limbs == 2 else "cQD",
                          us_per_eval_new=round(t_new * 1e3 / P, 4), us_per_eval_plain=round(t_plain * 1e3 / P, 4),
                          us_per_eval_old=round(t_old * 1e3 / P, 4), speedup_old_over_new=round(t_old / t_new, 3),
                          old_path=old.stats["path"], old_K=old.stats["K"])), flush=True)
