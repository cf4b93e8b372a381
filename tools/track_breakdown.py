"""Tracker time breakdown: wall time of a bounded tracking run (max_steps) against the sum of
its kernel durations (read from an ncu launch list of the same command, tools/ncu_summary.py
style).  Usage: python tools/track_breakdown.py n L paths max_steps"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1109_0545_b200 as phc  # noqa: E402
from synthetic import total_degree_homotopy  # noqa: E402

n, L, P, ms = (int(a) for a in (sys.argv[1:5] if len(sys.argv) > 4 else (10, 2, 1024, 40)))
s, cf, X0 = total_degree_homotopy(n, L, seed=1)
h = phc.System(s, coeff_target=cf)
X = torch.from_numpy(X0[:P]).cuda()
h.track(X[:4], max_steps=5)
torch.cuda.synchronize()
t0 = time.perf_counter()
Xe, status, stats = h.track(X, max_steps=ms)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(json.dumps(dict(n=n, L=L, paths=P, max_steps=ms, seconds=round(dt, 4), steps=int(stats[:, 1].max()),
                      us_per_step=round(dt / max(1, stats[:, 1].max()) * 1e6, 1))), flush=True)
# the same number of corrector calls through the Python API, back to back (GPU-bound floor)
from synthetic import real_limbs  # noqa: E402
T = torch.from_numpy(real_limbs([0.5] * P, L)).cuda()
Xn = torch.empty_like(X)
h.newton_step_homotopy(X, T, Xn)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(4 * ms):
    h.newton_step_homotopy(X, T, Xn)
torch.cuda.synchronize()
print(json.dumps(dict(corrector_calls=4 * ms, us_per_4_calls=round((time.perf_counter() - t0) / ms * 1e6, 1))))
