"""Write tests/golden/large_seed1.npz: the oracle's values for the BASELINE.json "large" config
(n = 256, m = 256, k = 32, D = 8, complex QD, seed 1) — every row of point 0 (F and all 256 x 256
Jacobian entries), and 8 rows at each of 8 points of the 4,096-point batch — so the GPU parity
tests can check the full output of the largest config without ~5 CPU-minutes of mp512 per run.

Imports only ``oracle/`` (the naive evaluator, mpmath at 512 bits: SURVEY.md §8(c) "mp mode")
and ``synthetic/`` (the seeded inputs and the limb split); nothing from the CUDA path.  Each
value is stored as 10 float64 limbs per real part (a greedy round-to-nearest split at 1,100
bits, >= 530 bits kept: the oracle's 512-bit values are stored without loss).  A SHA-256 of the
input arrays (system tables and the points used) is stored beside them; the tests refuse a golden
file whose inputs no longer match the generator.

    python tools/make_golden_large.py            # ~11 min on 8 cores
    python tools/make_golden_large.py --add-newton   # + the Newton step at point 0 (~min)

`--add-newton` adds the oracle's Newton step at point 0 (Alg. 2: dz = J^{-1}(-F) by
mpmath.lu_solve at 512 bits, oracle.solve_step_mp) computed from the stored oracle F and J.
"""
import hashlib
import os
import sys
import time

import mpmath
import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import evaluate_rows, solve_step_mp  # noqa: E402
from synthetic import config_system  # noqa: E402
from synthetic.systems import split_limbs  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "large_seed1.npz")
LIMBS = 10
PREC = 512
# batch sample: both ends of every 8-way shard boundary region plus interior points; 8 rows each
BATCH_POINTS = [1, 511, 512, 1537, 2048, 3071, 3584, 4095]


def batch_rows(p):
    return sorted({(p * 37 + 31 * j) % 256 for j in range(8)})


def input_digest(s, X, points):
    h = hashlib.sha256()
    for a in (s.poly_ptr, s.term_ptr, s.var_idx, s.exponent, s.coeff, X[list(points)]):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def to_limbs(values):
    out = np.zeros((len(values), 2, LIMBS))
    with mpmath.workprec(1100):
        for j, z in enumerate(values):
            z = mpmath.mpc(z)
            out[j, 0] = split_limbs(z.real._mpf_, LIMBS, 1100)
            out[j, 1] = split_limbs(z.imag._mpf_, LIMBS, 1100)
    return out


def from_limbs(limbs):
    out = []
    with mpmath.workprec(1100):
        for v in limbs.reshape(-1, 2, LIMBS):
            out.append(mpmath.mpc(mpmath.fsum(mpmath.mpf(float(d)) for d in v[0]),
                                  mpmath.fsum(mpmath.mpf(float(d)) for d in v[1])))
    return out


def add_newton():
    t0 = time.time()
    g = dict(np.load(OUT))
    s, X = config_system("large", seed=1)
    n = s.n_var
    F = from_limbs(g["F0"])
    Jf = from_limbs(g["J0"])
    J = [Jf[i * n:(i + 1) * n] for i in range(n)]
    with mpmath.workprec(PREC):
        z = [mpmath.mpc(mpmath.fsum(mpmath.mpf(float(d)) for d in X[0, v, 0]),
                        mpmath.fsum(mpmath.mpf(float(d)) for d in X[0, v, 1])) for v in range(n)]
    out = solve_step_mp(F, J, z, PREC)
    assert not out["singular"]
    g["newton_dz0"] = to_limbs(out["dz"])
    g["newton_residual0"] = np.float64(out["residual"])
    np.savez(OUT, **g)
    print(f"Newton step at point 0 added in {time.time() - t0:.0f} s")


def main():
    if "--add-newton" in sys.argv:
        add_newton()
        return
    t0 = time.time()
    s, X = config_system("large_batch", seed=1)
    n = s.n_eq
    F, J = evaluate_rows(s, X[0], None, "mp", PREC)
    f0 = to_limbs(F)
    j0 = to_limbs([v for row in J for v in row]).reshape(n, n, 2, LIMBS)
    print(f"point 0, {n} rows: {time.time() - t0:.0f} s", flush=True)
    rows = np.array([batch_rows(p) for p in BATCH_POINTS], dtype=np.int32)
    fb = np.zeros((len(BATCH_POINTS), rows.shape[1], 2, LIMBS))
    jb = np.zeros((len(BATCH_POINTS), rows.shape[1], n, 2, LIMBS))
    for q, p in enumerate(BATCH_POINTS):
        Fp, Jp = evaluate_rows(s, X[p], rows[q].tolist(), "mp", PREC)
        fb[q] = to_limbs(Fp)
        jb[q] = to_limbs([v for row in Jp for v in row]).reshape(rows.shape[1], n, 2, LIMBS)
        print(f"batch point {p}: {time.time() - t0:.0f} s", flush=True)
    np.savez(OUT, F0=f0, J0=j0, batch_points=np.array(BATCH_POINTS, dtype=np.int32), batch_rows=rows,
             Fb=fb, Jb=jb, prec=np.int32(PREC),
             digest_point0=np.array(input_digest(s, X, [0])),
             digest_batch=np.array(input_digest(s, X, BATCH_POINTS)),
             source=np.array("tools/make_golden_large.py: oracle.evaluate_rows (naive, mpmath 512 bits) on "
                             "synthetic.config_system('large_batch', seed=1); SURVEY.md §8(c) coverage plan"))
    print(f"wrote {OUT} in {time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()
