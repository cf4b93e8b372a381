"""Throughput of the DD layout-2 block kernel vs warps per SM: batch systems with k = 8 and
k = 16 (n = 32, m = 32, D = 4, 65,536 points), run with the library given by PHC_LIB."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1109_0545_b200 as phc  # noqa: E402
from synthetic import random_system  # noqa: E402

out = {"lib": os.path.basename(os.environ.get("PHC_LIB", "libphc.so"))}
peak = phc.phc_fp64_peak(0, 200.0)
for k in (8, 16):
    s, X = random_system(32, 32, k, 4, 2, seed=1, points=65536, workers=8)
    h = phc.System(s)
    Xd = torch.from_numpy(X).cuda()
    F = torch.empty((65536, 32, 2, 2), dtype=torch.float64, device="cuda")
    J = torch.empty((65536, 32, 32, 2, 2), dtype=torch.float64, device="cuda")
    for _ in range(2):
        h.eval_batch(Xd, F, J)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        h.eval_batch(Xd, F, J)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    out[f"k{k}_evals_s"] = round(65536 / (ms * 1e-3))
    out[f"k{k}_frac"] = round(h.stats["exec_flops_per_point"] * 65536 / (ms * 1e-3) / 1e12 / peak, 4)
print(json.dumps(out), flush=True)
