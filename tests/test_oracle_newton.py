"""Pins for the Newton-step oracle (NEXT-1; Alg. 2): exact linear solves
checked by multiplying back, the SPEC worked example x^2 - 4 at z = 3, and quadratic
convergence to a known root."""
from fractions import Fraction

import mpmath
import numpy as np
import pytest

from oracle import newton_step, solve_exact
from synthetic import config_system, limbs_from_values, system_from_terms
from synthetic.systems import unit_circle_limbs


def _mat_vec(A, x):
    out = []
    for row in A:
        re = sum(a[0] * v[0] - a[1] * v[1] for a, v in zip(row, x))
        im = sum(a[0] * v[1] + a[1] * v[0] for a, v in zip(row, x))
        out.append((re, im))
    return out


def test_solve_exact_multiplies_back():
    rng = np.random.default_rng(1)
    for n in (1, 2, 5, 9):
        A = [[(Fraction(int(a)), Fraction(int(b))) for a, b in rng.integers(-5, 6, (n, 2))] for _ in range(n)]
        x = [(Fraction(int(a), 7), Fraction(int(b), 3)) for a, b in rng.integers(-9, 10, (n, 2))]
        b = _mat_vec(A, x)
        got = solve_exact(A, b)
        if got is not None:  # random integer matrices are almost surely nonsingular
            assert got == x


def test_solve_exact_needs_pivoting_and_detects_singular():
    # SPEC linsolve example: A = [[0,1],[1,0]], b = (1,2) -> x = (2,1)
    Z, O = (Fraction(0), Fraction(0)), (Fraction(1), Fraction(0))
    assert solve_exact([[Z, O], [O, Z]], [(Fraction(1), 0), (Fraction(2), 0)]) == [(2, 0), (1, 0)]
    assert solve_exact([[O, O], [O, O]], [O, O]) is None


def test_spec_example_x2_minus_4():
    """SPEC corrector example: h = x^2 - 4, z = 3: dz = -5/6, z -> 13/6."""
    s = system_from_terms(1, 1, 2, [[[(0, 2)], []]], limbs_from_values([1, -4], 2))
    out = newton_step(s, limbs_from_values([3], 2), "exact", workers=1)
    assert out["dz"] == [(Fraction(-5, 6), 0)]
    assert out["z_new"] == [(Fraction(13, 6), 0)]
    assert out["residual"] == 5.0


def _root_system(n, seed, L=2):
    """f(x) = g(x) - g(x*) for a random sparse g and a unit-circle root x*: constant terms
    -g_i(x*) are exact rationals rounded to L limbs, so x* is a root up to that rounding."""
    s, X = config_system("tiny", seed=seed)
    return s, X


def test_quadratic_convergence_to_known_root():
    """Newton on f(x) = prod-structure system with root x* = 1 (all ones): f_i(x) = sum_t c_t (m_t(x) - 1),
    a sparse system vanishing at x = (1, ..., 1); from x* + delta the error squares each step."""
    n = 6
    rng = np.random.default_rng(3)
    polys, coeffs = [], []
    for i in range(n):
        terms = []
        for t in range(4):
            vs = sorted(rng.choice(n, 3, replace=False).tolist())
            terms.append([(v, int(rng.integers(1, 4))) for v in vs])
        # the constant term cancels the sum of the coefficients at x = 1
        c = [complex(*rng.integers(-3, 4, 2)) or 1 for _ in terms]
        polys.append(terms + [[]])
        coeffs += c + [-sum(c)]
    s = system_from_terms(n, n, 4, polys, limbs_from_values(coeffs, 4))
    delta = 2.0 ** -12
    x = [1 + delta * complex(*rng.uniform(-1, 1, 2)) for _ in range(n)]
    X = limbs_from_values(x, 4)
    errs = []
    for it in range(3):
        out = newton_step(s, X, "mp", prec=600, workers=1)
        z = out["z_new"]
        errs.append(max(abs(v - 1) for v in z))
        with mpmath.workprec(600):
            X = np.zeros((n, 2, 4))
            for v in range(n):
                for p_, part in enumerate((mpmath.re(z[v]), mpmath.im(z[v]))):
                    r = part
                    for l in range(4):
                        d = float(r)
                        X[v, p_, l] = d
                        r -= d
    assert errs[0] < 1e-5
    assert errs[1] < 50 * errs[0] ** 2
    assert errs[2] < 50 * errs[1] ** 2 + 1e-60


def _row_scaled_solve(A, b):
    """Test-only model of the device eliminations' solve (readings N6/N7 context):
    Gaussian elimination with partial pivoting on [A | b] (largest modulus, ties to the lowest
    row, rows exchanged through a permutation), then the ROW-SCALED back substitution
    c_r = b_r d_r, N_rj = U_rj d_r (d_r = 1 / U_rr), c_r -= N_rj x_j for j = n-1 .. r+1 -- in
    exact Gaussian rationals, so it must reach solve_exact's solution exactly."""
    n = len(A)
    M = [[A[i][j] for j in range(n)] + [b[i]] for i in range(n)]
    perm = list(range(n))
    d = [None] * n
    mod2 = lambda z: z[0] * z[0] + z[1] * z[1]  # noqa: E731
    for k in range(n):
        bi = max(range(k, n), key=lambda i: (mod2(M[perm[i]][k]), -i))
        assert mod2(M[perm[bi]][k]) != 0
        perm[k], perm[bi] = perm[bi], perm[k]
        p = M[perm[k]][k]
        m2 = mod2(p)
        d[k] = (p[0] / m2, -p[1] / m2)
        for i in range(k + 1, n):
            r = perm[i]
            li = (M[r][k][0] * d[k][0] - M[r][k][1] * d[k][1], M[r][k][0] * d[k][1] + M[r][k][1] * d[k][0])
            for j in range(k + 1, n + 1):
                u = M[perm[k]][j]
                M[r][j] = (M[r][j][0] - (li[0] * u[0] - li[1] * u[1]), M[r][j][1] - (li[0] * u[1] + li[1] * u[0]))
    cm = lambda x, y: (x[0] * y[0] - x[1] * y[1], x[0] * y[1] + x[1] * y[0])  # noqa: E731
    c = [cm(M[perm[r]][n], d[r]) for r in range(n)]
    N = [[cm(M[perm[r]][j], d[r]) if j > r else None for j in range(n)] for r in range(n)]
    for j in range(n - 1, 0, -1):
        for r in range(j):
            t = cm(N[r][j], c[j])
            c[r] = (c[r][0] - t[0], c[r][1] - t[1])
    return c


def test_row_scaled_back_substitution_reaches_the_exact_solution():
    """Reading N6: the row-scaled back substitution (scaled rows N = D^-1 U, c = D^-1 b, one
    multiply-subtract per row on the chain) is the same exact solve as the plain definition:
    equal to solve_exact (and to the generating x) in exact rationals, with pivoting exercised
    by small leading entries."""
    rng = np.random.default_rng(6)
    ran = 0
    for n in (1, 2, 3, 6, 9):
        for _ in range(3):
            A = [[(Fraction(int(a), 5), Fraction(int(b), 3)) for a, b in rng.integers(-7, 8, (n, 2))]
                 for _ in range(n)]
            for i in range(n):  # a tiny diagonal forces row exchanges
                A[i][i] = (Fraction(1, 1000), Fraction(0))
            x = [(Fraction(int(a), 7), Fraction(int(b), 11)) for a, b in rng.integers(-9, 10, (n, 2))]
            b = _mat_vec(A, x)
            try:
                ref = solve_exact(A, b)
            except (ZeroDivisionError, AssertionError):
                continue
            got = _row_scaled_solve(A, b)
            assert got == ref == x
            ran += 1
    assert ran >= 12
