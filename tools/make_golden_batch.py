"""Write tests/golden/batch_seed1.npz: the oracle's values (exact rational arithmetic) of F and
J at 16 points of the BASELINE.json "batch" config (n = m = 32, k = 16, D = 4, complex DD,
65,536 points, seed 1): the first and last point of every 8-way shard.  bench.py's batch_dd
record checks the GPU's rows at these points against them (every entry), without running the
oracle in the timed process.

Imports only ``oracle/`` (naive evaluator, exact Gaussian dyadic rationals) and ``synthetic/``;
each exact value is stored as 10 float64 limbs per real part (a greedy round-to-nearest split:
>= 530 correct bits, far beyond the 1e-28 tolerance), with a SHA-256 of the inputs.

    python tools/make_golden_batch.py            # ~20 s on 8 cores
"""
import hashlib
import os
import sys
import time
from fractions import Fraction

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import evaluate_rows  # noqa: E402
from synthetic import config_point_rows, config_system  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "batch_seed1.npz")
LIMBS = 10
P = 65536
POINTS = sorted({g * P // 8 for g in range(8)} | {(g + 1) * P // 8 - 1 for g in range(8)})


def to_limbs(values):
    """exact dyadic complex values (re, im, e) -> [N][2][LIMBS] greedy round-to-nearest limbs"""
    out = np.zeros((len(values), 2, LIMBS))
    for j, (a, b, e) in enumerate(values):
        for part, m in enumerate((a, b)):
            r = Fraction(m) * Fraction(2) ** e
            for q in range(LIMBS):
                d = float(r)
                out[j, part, q] = d
                r -= Fraction(d)
    return out


def main():
    t0 = time.time()
    s, _ = config_system("batch", seed=1, points=1)
    X = config_point_rows("batch", 1, POINTS, P)
    n = s.n_eq
    F = np.zeros((len(POINTS), n, 2, LIMBS))
    J = np.zeros((len(POINTS), n, n, 2, LIMBS))
    for q in range(len(POINTS)):
        Fq, Jq = evaluate_rows(s, X[q], None, "exact")
        F[q] = to_limbs(Fq)
        J[q] = to_limbs([v for row in Jq for v in row]).reshape(n, n, 2, LIMBS)
    h = hashlib.sha256()
    for a in (s.poly_ptr, s.term_ptr, s.var_idx, s.exponent, s.coeff, X):
        h.update(np.ascontiguousarray(a).tobytes())
    np.savez(OUT, F=F, J=J, points=np.array(POINTS, dtype=np.int64), digest=np.array(h.hexdigest()),
             source=np.array("tools/make_golden_batch.py: oracle.evaluate_rows (naive, exact rationals) on "
                             "synthetic.config_system('batch', seed=1); SURVEY.md §8(c) coverage plan"))
    print(f"wrote {OUT} in {time.time() - t0:.0f} s")


if __name__ == "__main__":
    main()
