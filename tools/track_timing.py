"""NEXT-4 timing: track all 2^n paths of a total-degree homotopy (quadratic target, start
gamma (x_i^2 - 1)) with the batched tracker on one B200; reports paths/s, steps and Newton
iterations, secant vs quadratic predictor (§5, Tables 2-3 columns)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1109_0545_b200 as phc  # noqa: E402
from synthetic import total_degree_homotopy  # noqa: E402

from synthetic import as_common  # noqa: E402

for n, L, via in ((8, 2, "per-term"), (8, 2, "common"), (10, 2, "per-term"), (10, 2, "common"), (8, 4, "per-term"),
                  (8, 4, "common")):
    s, cf, X0 = total_degree_homotopy(n, L, seed=1)
    if via == "common":
        c, cft = as_common(s, cf)
        h = phc.System(c, coeff_target=cft)
    else:
        h = phc.System(s, coeff_target=cf)
    X = torch.from_numpy(X0).cuda()
    for pred in ((2, 1) if via == "per-term" else (2,)):
        h.track(X[:4], predictor=pred)  # warm-up
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        Xe, status, stats = h.track(X, predictor=pred)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        print(json.dumps(dict(n=n, precision="cDD" if L == 2 else "cQD", handle=via, paths=int(X.shape[0]),
                              predictor="quadratic" if pred == 2 else "secant", seconds=round(dt, 3),
                              paths_per_s=round(X.shape[0] / dt, 1), arrived=int((status == 1).sum()),
                              failed=int((status == 2).sum()), mean_steps=round(float(stats[:, 1].mean()), 1),
                              mean_accepted=round(float(stats[:, 0].mean()), 1),
                              mean_newton=round(float(stats[:, 2].mean()), 1),
                              min_step=float(stats[:, 3][stats[:, 3] > 0].min()) if (stats[:, 3] > 0).any() else 0.0,
                              avg_step=round(float(stats[:, 4].mean()), 5))), flush=True)
