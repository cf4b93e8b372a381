"""Wave-quantization probe for the large QD single point: time one evaluation of random
systems shaped like `large` (m = 256 terms per polynomial, k = 32, D = 8, QD) with n
polynomials (n * 8 warp-blocks on 148 SMs x 8 warps = 1,184 warp slots)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1109_0545_b200 as phc  # noqa: E402
from synthetic import random_system  # noqa: E402

for n in [int(a) for a in sys.argv[1:]] or [148, 185, 222, 256, 296]:
    s, X = random_system(n, 256, 32, 8, 4, seed=1, points=1, workers=8)
    h = phc.System(s)
    x = torch.from_numpy(X[0]).cuda()
    f = torch.empty((s.n_eq, 2, 4), dtype=torch.float64, device="cuda")
    j = torch.empty((s.n_eq, s.n_var, 2, 4), dtype=torch.float64, device="cuda")
    for _ in range(3):
        h.eval(x, f, j)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        h.eval(x, f, j)
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / 20 * 1e3
    print(json.dumps(dict(n=n, blocks=n * 8, us=round(us, 1), us_per_block_wave=round(us / max(1, -(-n * 8 // 1184)), 1),
                          mode=h.stats.get("layout"))), flush=True)
