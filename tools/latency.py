"""Single-point latency of phc_eval_jacobian for the BASELINE.json single-point configs.
Times `reps` back-to-back calls with CUDA events on the launching stream (after warm-up);
reports median-free mean latency and the executed-flop rate."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1109_0545_b200 as phc  # noqa: E402
from synthetic import config_system  # noqa: E402

peak = phc.phc_fp64_peak(0, 200.0)
for name in (sys.argv[1:] or ["tiny", "c2", "c3", "large"]):
    s, X = config_system(name, seed=1)
    h = phc.System(s)
    st = h.stats
    x = torch.from_numpy(X[0]).cuda()
    f = torch.empty((s.n_eq, 2, s.limbs), dtype=torch.float64, device="cuda")
    j = torch.empty((s.n_eq, s.n_var, 2, s.limbs), dtype=torch.float64, device="cuda")
    for _ in range(10):
        h.eval(x, f, j)
    torch.cuda.synchronize()
    reps = 200 if s.n_var <= 64 else 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        h.eval(x, f, j)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps
    tf = st["exec_flops_per_point"] / (us * 1e-6) / 1e12
    print(json.dumps(dict(config=name, us_per_eval=us, evals_per_s=1e6 / us, exec_tflops=tf, exec_frac=tf / peak,
                          path=st["path"], layout=st["layout"], K=st["K"])), flush=True)
