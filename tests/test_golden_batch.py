"""CPU checks of tests/golden/batch_seed1.npz (tools/make_golden_batch.py: exact-rational oracle
values of F and J at 16 points of the BASELINE.json batch config): its inputs are the ones the
generator draws, one point re-evaluated by the oracle matches every stored entry, and
bench.py's batch parity record sees limb rounding as ~u and a perturbed entry as an error."""
import hashlib
import os
from fractions import Fraction

import numpy as np

from oracle import evaluate_rows
from synthetic import config_point_rows, config_system

G = os.path.join(os.path.dirname(__file__), "golden", "batch_seed1.npz")


def test_batch_golden_inputs_and_values():
    g = np.load(G)
    pts = [int(p) for p in g["points"]]
    assert pts[0] == 0 and pts[-1] == 65535 and len(pts) == 16
    s, _ = config_system("batch", seed=1, points=1)
    X = config_point_rows("batch", 1, pts, 65536)
    h = hashlib.sha256()
    for a in (s.poly_ptr, s.term_ptr, s.var_idx, s.exponent, s.coeff, X):
        h.update(np.ascontiguousarray(a).tobytes())
    assert str(g["digest"]) == h.hexdigest()
    q = 9
    F, J = evaluate_rows(s, X[q], None, "exact", workers=1)
    ex = lambda limbs: sum(Fraction(float(d)) for d in limbs)  # noqa: E731

    def close(val, limbs):
        a, b, e = val
        sc = Fraction(2) ** e
        return abs(ex(limbs[0]) - a * sc) <= Fraction(1, 2 ** 500) and abs(ex(limbs[1]) - b * sc) <= Fraction(1, 2 ** 500)

    assert all(close(F[i], g["F"][q, i]) for i in range(32))
    assert all(close(J[i][v], g["J"][q, i, v]) for i in range(32) for v in range(32))


def test_bench_batch_parity_record():
    import bench
    torch = __import__("torch")
    g = np.load(G)
    F = torch.zeros((65536, 32, 2, 2), dtype=torch.float64)
    J = torch.zeros((65536, 32, 32, 2, 2), dtype=torch.float64)
    for q, p in enumerate(g["points"]):
        F[int(p)] = torch.from_numpy(g["F"][q][..., :2].copy())
        J[int(p)] = torch.from_numpy(g["J"][q][..., :2].copy())
    r = bench.parity_batch("batch", F, J)
    assert r["err_F"] < 1e-30 and r["err_J"] < 1e-30 and r["tolerance"] == 1e-28
    J[int(g["points"][3]), 4, 5, 1, 0] += 1e-12
    assert bench.parity_batch("batch", F, J)["err_J"] > 1e-14
