"""CPU checks of the committed large-config golden file (tests/golden/large_seed1.npz, written
by tools/make_golden_large.py from oracle/ and synthetic/ only): its inputs are the ones the
generator draws today, its stored values are the oracle's (one row of point 0 and one row of a
batch point re-evaluated here at 512 bits), and its zero pattern is the system's structure."""
import mpmath
import numpy as np

from _golden import digest, load, to_mpc
from oracle import evaluate_rows
from synthetic import config_point_rows, config_system


def test_golden_inputs_match_generator():
    g = load()
    s, X0 = config_system("large", seed=1)
    assert str(g["digest_point0"]) == digest(s, X0[[0]])
    pts = [int(p) for p in g["batch_points"]]
    Xb = config_point_rows("large_batch", 1, pts)
    assert str(g["digest_batch"]) == digest(s, Xb)


def test_golden_values_are_the_oracles():
    g = load()
    s, X0 = config_system("large", seed=1)
    F, J = evaluate_rows(s, X0[0], [77], "mp", 512, workers=1)
    ref = to_mpc(g["J0"][77])
    with mpmath.workprec(1100):
        assert abs(F[0] - to_mpc(g["F0"][77:78])[0]) < mpmath.mpf(2) ** -500
        assert max(abs(a - b) for a, b in zip(J[0], ref)) < mpmath.mpf(2) ** -500
    q = 5
    p, r = int(g["batch_points"][q]), int(g["batch_rows"][q][3])
    Xp = config_point_rows("large_batch", 1, [p])[0]
    F, J = evaluate_rows(s, Xp, [r], "mp", 512, workers=1)
    with mpmath.workprec(1100):
        assert abs(F[0] - to_mpc(g["Fb"][q, 3:4])[0]) < mpmath.mpf(2) ** -500
        assert max(abs(a - b) for a, b in zip(J[0], to_mpc(g["Jb"][q, 3]))) < mpmath.mpf(2) ** -500


def test_golden_zero_pattern_is_the_structure():
    g = load()
    s, _ = config_system("large", seed=1)
    nz = np.zeros((s.n_eq, s.n_var), bool)
    for i in range(s.n_eq):
        for _, fac in s.terms(i):
            for v, _a in fac:
                nz[i, v] = True
    zero = np.all(g["J0"] == 0, axis=(2, 3))
    assert np.array_equal(zero, ~nz)
    assert np.all(np.abs(g["F0"][:, :, 0]).max(axis=1) > 0)


def test_bench_parity_check_against_golden():
    """bench.py's in-line parity record (exact integer arithmetic on the limbs) sees QD
    rounding of the oracle values as ~1e-65 and a perturbed entry as an error."""
    import bench
    g = load()
    f, j = g["F0"][..., :4].copy(), g["J0"][..., :4].copy()
    r = bench.parity_vs_golden(f, j)
    assert r["err_F"] < 1e-63 and r["err_J"] < 1e-63
    j[7, 9, 1, 1] += 1e-25
    assert bench.parity_vs_golden(f, j)["err_J"] > 1e-30
