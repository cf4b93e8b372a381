"""NEXT-2 timing: the two-stage common-support evaluation (phc_system_create_common) against
the per-term path on the same polynomials (expanded system), Table 1 shape (PAPER.md
P:355-358), single point and batch; plus the 1,000-Newton-iteration workload of Table 1
(phc_newton_step_batch) on the common-support handle."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1109_0545_b200 as phc  # noqa: E402
from synthetic import common_config, expand_common  # noqa: E402


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


peak = phc.phc_fp64_peak(0, 200.0)
for name, P in (("common", 1), ("common_dd", 1), ("common", 1024), ("common_batch", 8192)):
    c, X = common_config(name, seed=1, points=P, workers=8)
    hc = phc.System(c)
    he = phc.System(expand_common(c))
    Xd = torch.from_numpy(X).cuda()
    F = torch.empty((P, c.n_eq, 2, c.limbs), dtype=torch.float64, device="cuda")
    J = torch.empty((P, c.n_eq, c.n_var, 2, c.limbs), dtype=torch.float64, device="cuda")
    reps = 200 if P == 1 else 5
    tc = timed(lambda: hc.eval_batch(Xd, F, J), reps)
    te = timed(lambda: he.eval_batch(Xd, F, J), reps)
    st = hc.stats
    out = dict(config=name, points=P, precision="cQD" if c.limbs == 4 else "cDD",
               us_per_eval_two_stage=round(tc * 1e3 / P, 3), us_per_eval_per_term=round(te * 1e3 / P, 3),
               speedup=round(te / tc, 3), exec_frac_two_stage=round(st["exec_flops_per_point"] * P / (tc * 1e-3) / 1e12 / peak, 4))
    if P == 1:
        x = Xd.clone()
        tn = timed(lambda: hc.newton_step(x, x), 50)
        out["newton_1000_iterations_s"] = round(tn * 1000 / 1e3, 4)
    print(json.dumps(out), flush=True)
