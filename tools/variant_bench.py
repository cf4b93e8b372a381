"""A/B timing of library variants (PHC_LIB=...): single-point latency (c3, large) and the
large-QD batch throughput.  CUDA events on the launching stream, after warm-up."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1109_0545_b200 as phc  # noqa: E402
from synthetic import config_system  # noqa: E402


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


tag = os.path.basename(os.environ.get("PHC_LIB", "libphc.so"))
peak = phc.phc_fp64_peak(0, 200.0)
out = {"lib": tag, "peak": round(peak, 2)}
for name in (sys.argv[1:] or ["c3", "large"]):
    s, X = config_system(name, seed=1, points=128 if name == "large" else 1, workers=8)
    h = phc.System(s)
    st = h.stats
    x = torch.from_numpy(X[0]).cuda()
    f = torch.empty((s.n_eq, 2, s.limbs), dtype=torch.float64, device="cuda")
    j = torch.empty((s.n_eq, s.n_var, 2, s.limbs), dtype=torch.float64, device="cuda")
    ms = timed(lambda: h.eval(x, f, j), 50 if name == "large" else 200)
    out[name + "_us"] = round(ms * 1e3, 2)
    out[name + "_frac"] = round(st["exec_flops_per_point"] / (ms * 1e-3) / 1e12 / peak, 4)
    if name == "large":
        Xd = torch.from_numpy(X).cuda()
        F = torch.empty((X.shape[0], s.n_eq, 2, s.limbs), dtype=torch.float64, device="cuda")
        JJ = torch.empty((X.shape[0], s.n_eq, s.n_var, 2, s.limbs), dtype=torch.float64, device="cuda")
        ms = timed(lambda: h.eval_batch(Xd, F, JJ), 3)
        out["large128_evals_s"] = round(X.shape[0] / (ms * 1e-3), 1)
        out["large128_frac"] = round(st["exec_flops_per_point"] * X.shape[0] / (ms * 1e-3) / 1e12 / peak, 4)
print(json.dumps(out), flush=True)
