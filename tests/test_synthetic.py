"""The seeded input generator (synthetic/): determinism, shapes, normalised limbs, unit modulus."""
import mpmath
import numpy as np

from synthetic import CONFIGS, config_system, random_system


def test_deterministic_and_shapes():
    s1, X1 = config_system("c2", seed=7)
    s2, X2 = config_system("c2", seed=7)
    for a in ("poly_ptr", "term_ptr", "var_idx", "exponent", "coeff"):
        assert np.array_equal(getattr(s1, a), getattr(s2, a))
    assert np.array_equal(X1, X2)
    c = CONFIGS["c2"]
    assert s1.n_terms == c["n"] * c["m"]
    assert s1.coeff.shape == (c["n"] * c["m"], 2, c["limbs"])
    assert X1.shape == (1, c["n"], 2, c["limbs"])
    k = np.diff(s1.term_ptr)
    assert (k == c["k"]).all()
    assert s1.exponent.min() >= 1 and s1.exponent.max() <= c["D"]
    for t in range(s1.n_terms):
        v = s1.var_idx[s1.term_ptr[t]:s1.term_ptr[t + 1]]
        assert (np.diff(v) > 0).all()


def test_batch_point0_is_single_point():
    """Recipe: the single-point config uses X[0] of the batch draw."""
    _, X1 = random_system(6, 3, 2, 3, 4, seed=3, points=1)
    _, X5 = random_system(6, 3, 2, 3, 4, seed=3, points=5)
    assert np.array_equal(X1[0], X5[0])


def test_limbs_normalised_unit_modulus():
    for L in (2, 4):
        s, X = random_system(5, 4, 3, 3, L, seed=11, points=3)
        vals = np.concatenate([s.coeff, X.reshape(-1, 2, L)])
        for z in vals:
            for part in z:
                for l in range(L - 1):  # non-overlapping, round-to-nearest split
                    assert part[l] == 0 or abs(part[l + 1]) <= abs(np.spacing(part[l])) / 2
            with mpmath.workprec(600):
                re = mpmath.fsum([mpmath.mpf(d) for d in z[0]])
                im = mpmath.fsum([mpmath.mpf(d) for d in z[1]])
                assert abs(re * re + im * im - 1) < mpmath.mpf(2) ** (-50 * L)
