"""Accuracy margin of a library build on the seeded fuzz shapes (tests/test_gpu_fuzz.py's
_shape): for every QD (or DD) shape, the normwise errors of F and J at the first and last
point against the 512-bit oracle, printed as the largest error / tolerance ratios.

    PHC_LIB=paper_1109_0545_b200/libphc.so python tools/fuzz_margin.py 4 300
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

import paper_1109_0545_b200 as phc  # noqa: E402
from _parity import TOL, compare_point, oracle_point  # noqa: E402
from test_gpu_fuzz import _shape  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 4
n = int(sys.argv[2]) if len(sys.argv) > 2 else 200
worst = []
for seed in range(n):
    s, X, polys = _shape(seed)
    if s.limbs != L or s.n_terms == 0:
        continue
    h = phc.System(s, device=0)
    Xd = torch.from_numpy(np.ascontiguousarray(X)).cuda()
    F, J = h.eval_batch(Xd) if X.shape[0] > 1 else [t[None] for t in h.eval(Xd[0])]
    F, J = F.cpu().numpy(), J.cpu().numpy()
    for p in sorted({0, X.shape[0] - 1}):
        ar, Fo, Jo = oracle_point(s, X[p], arith="mp")
        ef, ej = compare_point(ar, Fo, Jo, F[p], J[p], L)
        worst.append((max(ef, ej) / TOL[L], seed, p, int(s.kmax) if hasattr(s, "kmax") else -1, X.shape[0]))
worst.sort(reverse=True)
print(json.dumps({"lib": os.environ.get("PHC_LIB", "libphc.so"), "limbs": L, "cases": len(worst),
                  "max_ratio": worst[0][0] if worst else None, "median_ratio": worst[len(worst) // 2][0] if worst else None,
                  "top": worst[:5]}))
