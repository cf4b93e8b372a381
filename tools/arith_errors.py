import os, sys
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
from fractions import Fraction as Fr
import paper_1109_0545_b200 as phc
from test_gpu_arith import run, ex, rand_reals
from synthetic import real_limbs
for L in (2, 4):
    rng = np.random.default_rng(10 + L); n = 2000
    A, B = rand_reals(rng, n, L), rand_reals(rng, n, L)
    a, b = real_limbs(A, L), real_limbs(B, L)
    u = Fr(1, 2 ** (53 * L))
    for op, name, f in ((2, "add", lambda x, y: x + y), (3, "mul", lambda x, y: x * y), (4, "div", lambda x, y: x / y)):
        out = run(phc, op, L, a, b, (n, L)); m = 0
        for i in range(n):
            xa, xb = ex(a[i]), ex(b[i]); ref = f(xa, xb)
            scale = abs(xa) + abs(xb) if name == "add" else abs(ref)
            m = max(m, abs(ex(out[i]) - ref) / (u * scale))
        print(L, name, float(m))
    ac = np.stack([real_limbs(rand_reals(rng, n, L, 4), L), real_limbs(rand_reals(rng, n, L, 4), L)], axis=1)
    bc = np.stack([real_limbs(rand_reals(rng, n, L, 4), L), real_limbs(rand_reals(rng, n, L, 4), L)], axis=1)
    for op in (5, 7, 8):
        out = run(phc, op, L, ac, bc, (n, 2, L)); m = 0
        for i in range(n):
            ar, ai, br, bi = ex(ac[i, 0]), ex(ac[i, 1]), ex(bc[i, 0]), ex(bc[i, 1])
            if op == 8:
                m2 = ar * ar + ai * ai; rr, ri = ar / m2, -ai / m2; sc2 = 1 / m2
            else:
                rr, ri = ar * br - ai * bi, ar * bi + ai * br; sc2 = (ar * ar + ai * ai) * (br * br + bi * bi)
            d2 = (ex(out[i, 0]) - rr) ** 2 + (ex(out[i, 1]) - ri) ** 2
            m = max(m, float((d2 / sc2) ** 0.5 / u) if d2 else 0.0)
        print(L, "cplx op", op, m)
