"""Pins for the CPU oracle: the oracle is checked against
things other than itself — SPEC/paper worked examples, library routines
(mpmath.power, mpmath.polyval, sympy.diff, numpy matmul), exact finite
differences, the Euler identity, and the paper's AD scheme in exact arithmetic."""
import json
import math
import os
from fractions import Fraction

import mpmath
import numpy as np
import pytest

from oracle import ExactArith, MPArith, evaluate_rows, evaluate_system, rel_errors
from synthetic import (config_system, homogeneous_system, limbs_from_values, random_system,
                       special_gaussian_system, special_linear_system, special_univariate_system,
                       system_from_terms)

from _ad_model import ad_row, omega_products, Counter

GOLD = os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")
EX = ExactArith()


def _cint(p):
    """exact dyadic complex -> (Fraction re, Fraction im)"""
    a, b, e = p
    s = Fraction(2) ** e
    return (a * s, b * s)


def _system_from_gold(g, limbs=2):
    polys = []
    coeffs = []
    for poly in g["polys"]:
        terms = []
        for term in poly:
            terms.append([tuple(f) for f in term["f"]])
            coeffs.append(complex(*term["c"]))
        polys.append(terms)
    n_eq = len(polys)
    sys_ = system_from_terms(n_eq, g["n_var"], limbs, polys, limbs_from_values(coeffs, limbs))
    X = limbs_from_values([complex(*x) for x in g["x"]], limbs)[None]
    return sys_, X


def test_golden_spec_examples():
    gold = json.load(open(GOLD))
    for g in gold["systems"]:
        s, X = _system_from_gold(g)
        F, J = evaluate_system(s, X[0], "exact", workers=1)
        assert [_cint(f) for f in F] == [(Fraction(a), Fraction(b)) for a, b in g["F"]], g["cite"]
        for i in range(s.n_eq):
            assert [_cint(v) for v in J[i]] == [(Fraction(a), Fraction(b)) for a, b in g["J"][i]], g["cite"]


def test_golden_omega_and_3k_minus_6():
    """P:550 '3k-6 multiplications' and SPEC S:209-211 via the paper's scheme (reading C1)."""
    gold = json.load(open(GOLD))
    for g in gold["omega"]:
        cm = Counter(EX)
        om = omega_products(cm, [(v, 0, 0) for v in g["v"]])
        assert [_cint(w) for w in om] == [(Fraction(v), 0) for v in g["omega"]], g["cite"]
        assert cm.mults == g["mults"]
    for k in range(2, 40):
        cm = Counter(EX)
        xs = [(p, 0, 0) for p in range(2, 2 + k)]
        om = omega_products(cm, xs)
        assert cm.mults == 3 * k - 6
        total = math.prod(range(2, 2 + k))
        assert [_cint(w)[0] for w in om] == [Fraction(total, x[0]) for x in xs]


def test_literal_paper_indices_are_wrong():
    """Reading C1: the printed omega_1 = psi_{k-1} is the product WITHOUT x_{i_k}, not without x_{i_1}."""
    cm = Counter(EX)
    om = omega_products(cm, [(2, 0, 0), (3, 0, 0), (5, 0, 0)], literal=True)
    assert _cint(om[0])[0] != 15


@pytest.mark.parametrize("d", [1, 2, 3, 7, 12])
def test_closed_form_power(d):
    """f = c x^d  ->  F = c x^d,  J = c d x^{d-1}, against mpmath.power (binary powering) at 512 bits."""
    sys_, X = special_univariate_system(0, 4, seed=d)  # just to draw a unit-circle c and x
    c = sys_.coeff[0]
    s = system_from_terms(1, 1, 4, [[[(0, d)]]], c[None])
    F, J = evaluate_system(s, X[0], "mp", prec=512, workers=1)
    ar = MPArith(512)
    with mpmath.workprec(512):
        cv = ar.from_limbs(c[0], c[1])
        xv = ar.from_limbs(X[0, 0, 0], X[0, 0, 1])
        fref = cv * mpmath.power(xv, d)
        jref = cv * d * mpmath.power(xv, d - 1)
        assert abs(F[0] - fref) < mpmath.mpf(2) ** -500
        assert abs(J[0][0] - jref) < mpmath.mpf(2) ** -490


@pytest.mark.parametrize("seed", [1, 2])
def test_univariate_vs_mpmath_polyval(seed):
    """n = 1 reduces to a dense univariate polynomial: mpmath.polyval(..., derivative=True) (P4)."""
    deg = 9
    s, X = special_univariate_system(deg, 4, seed)
    F, J = evaluate_system(s, X[0], "mp", prec=512, workers=1)
    ar = MPArith(512)
    with mpmath.workprec(512):
        cs = [ar.from_limbs(s.coeff[t, 0], s.coeff[t, 1]) for t in range(deg + 1)]
        x = ar.from_limbs(X[0, 0, 0], X[0, 0, 1])
        val, der = mpmath.polyval(cs[::-1], x, derivative=True)
        assert abs(F[0] - val) < mpmath.mpf(2) ** -495
        assert abs(J[0][0] - der) < mpmath.mpf(2) ** -490


def test_linear_system_is_matrix():
    """k = 1, a = 1: J equals the coefficient matrix and F = C x (numpy integer matmul) (P4)."""
    s, X, C, x = special_linear_system(7, 2, seed=3)
    F, J = evaluate_system(s, X[0], "exact", workers=1)
    Cc = C[:, :, 0] + 1j * C[:, :, 1]
    xc = x[:, 0] + 1j * x[:, 1]
    Fn = Cc @ xc
    for i in range(7):
        assert _cint(F[i]) == (Fraction(int(Fn[i].real)), Fraction(int(Fn[i].imag)))
        for v in range(7):
            assert _cint(J[i][v]) == (Fraction(int(C[i, v, 0])), Fraction(int(C[i, v, 1])))


def test_gaussian_integer_system_vs_python_complex():
    """Coefficients in Z[i], x in {±1, ±i}: every value is a small Gaussian integer (P5);
    compare with Python's built-in complex power (exact for these small integers)."""
    s, X = special_gaussian_system(6, 5, 3, 4, 2, seed=5)
    F, J = evaluate_system(s, X[0], "exact", workers=1)
    xs = [complex(X[0, v, 0, 0], X[0, v, 1, 0]) for v in range(6)]
    for i in range(6):
        fi = 0j
        ji = [0j] * 6
        for t, factors in s.terms(i):
            c = complex(s.coeff[t, 0, 0], s.coeff[t, 1, 0])
            fi += c * math.prod(xs[v] ** a for v, a in factors)
            for v, a in factors:
                rest = math.prod(xs[u] ** b for u, b in factors if u != v)
                ji[v] += c * a * xs[v] ** (a - 1) * rest
        assert _cint(F[i]) == (Fraction(fi.real), Fraction(fi.imag))
        assert [_cint(z) for z in J[i]] == [(Fraction(z.real), Fraction(z.imag)) for z in ji]


def test_tiny_vs_sympy_diff():
    """Brute force on the tiny config: sympy builds f_i symbolically, sympy.diff differentiates,
    evaluation at the exact rational inputs must equal the exact oracle."""
    sympy = pytest.importorskip("sympy")
    s, X = config_system("tiny", seed=2)
    F, J = evaluate_system(s, X[0], "exact", workers=1)
    xsym = sympy.symbols(f"x0:{s.n_var}")

    def q(limbs):
        return sum((sympy.Rational(*float(d).as_integer_ratio()) for d in limbs), sympy.Integer(0))

    xval = {xsym[v]: q(X[0, v, 0]) + sympy.I * q(X[0, v, 1]) for v in range(s.n_var)}
    for i in range(s.n_eq):
        f = sympy.Integer(0)
        for t, factors in s.terms(i):
            c = q(s.coeff[t, 0]) + sympy.I * q(s.coeff[t, 1])
            f += c * sympy.Mul(*[xsym[v] ** a for v, a in factors])
        fv = sympy.expand(f.subs(xval))
        assert _cint(F[i]) == (Fraction(str(sympy.re(fv))), Fraction(str(sympy.im(fv))))
        for v in range(s.n_var):
            dv = sympy.expand(sympy.diff(f, xsym[v]).subs(xval))
            assert _cint(J[i][v]) == (Fraction(str(sympy.re(dv))), Fraction(str(sympy.im(dv)))), (i, v)


def _fd_weights(r):
    """Central first-derivative weights of order 2r: w_j = (-1)^{j+1} (r!)^2 / (j (r-j)! (r+j)!)."""
    f = math.factorial
    return [Fraction((-1) ** (j + 1) * f(r) ** 2, j * f(r - j) * f(r + j)) for j in range(1, r + 1)]


@pytest.mark.parametrize("name,seed", [("tiny", 1), ("tiny", 3), ("c2", 1)])
def test_exact_finite_differences(name, seed):
    """Along x_v, f_i is a polynomial of degree <= D, so the order-2r central stencil with 2r >= D
    is exact: in exact arithmetic  sum_j w_j (f(x+jh e_v) - f(x-jh e_v)) = h J_{i,v}  (P6)."""
    s, X = config_system(name, seed=seed)
    D = int(s.exponent.max())
    r = (D + 1) // 2
    w = _fd_weights(r)
    den = math.lcm(*[x.denominator for x in w])
    wi = [int(x * den) for x in w]
    h_exp = -7  # h = 2^-7
    F0, J = evaluate_system(s, X[0], "exact", workers=1)
    vs = range(s.n_var) if name == "tiny" else [0, 7, 19]
    for v in vs:
        acc = [EX.zero() for _ in range(s.n_eq)]
        for j, wj in zip(range(1, r + 1), wi):
            for sign, mult in ((1, wj), (-1, -wj)):
                Xs = X[0].copy()
                Xp = [list(Xs[u, 0]) + [0.0] for u in range(s.n_var)]
                # x_v + sign*j*h exactly: append the shift as an extra real limb
                Xe = np.zeros((s.n_var, 2, s.limbs + 1))
                Xe[:, :, : s.limbs] = Xs
                Xe[v, 0, s.limbs] = sign * j * 2.0 ** h_exp
                se = system_from_terms(s.n_eq, s.n_var, s.limbs, [[f for _, f in s.terms(i)] for i in range(s.n_eq)], s.coeff)
                se.limbs = s.limbs + 1
                se.coeff = np.concatenate([s.coeff, np.zeros((s.n_terms, 2, 1))], axis=2)
                Fs, _ = evaluate_system(se, Xe, "exact", workers=1)
                for i in range(s.n_eq):
                    acc[i] = EX.add(acc[i], EX.scale_int(Fs[i], mult))
        for i in range(s.n_eq):
            lhs = _cint(acc[i])
            rhs = _cint(EX.scale_int(J[i][v], den))
            hj = Fraction(2) ** h_exp
            assert lhs == (rhs[0] * hj, rhs[1] * hj), (name, i, v)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_ad_scheme_equals_naive_exactly(seed):
    """P7: the §6 scheme (reading C1, exponent factor C3) equals the naive oracle EXACTLY in exact
    arithmetic, and spends exactly 3k-6 multiplications on omega per term."""
    s, X = config_system("c2", seed=seed)
    F, J = evaluate_system(s, X[0], "exact", workers=1)
    xs = [EX.from_limbs(X[0, v, 0], X[0, v, 1]) for v in range(s.n_var)]
    for i in range(s.n_eq):
        terms, coeffs = [], []
        for t, factors in s.terms(i):
            terms.append(factors)
            coeffs.append(EX.from_limbs(s.coeff[t, 0], s.coeff[t, 1]))
        f, jrow, om = ad_row(EX, xs, terms, coeffs, s.n_var)
        assert _cint(f) == _cint(F[i])
        assert [_cint(z) for z in jrow] == [_cint(z) for z in J[i]]
        assert all(cnt == 3 * k - 6 for k, cnt in om)


@pytest.mark.parametrize("seed", [4, 5])
def test_euler_identity_homogeneous(seed):
    """P8: every term of f_i has total degree d_i  ->  sum_v x_v J_{i,v} = d_i f_i, exactly."""
    s, X, degs = homogeneous_system(9, 7, 4, 6, 2, seed)
    F, J = evaluate_system(s, X[0], "exact", workers=1)
    xs = [EX.from_limbs(X[0, v, 0], X[0, v, 1]) for v in range(s.n_var)]
    for i in range(s.n_eq):
        acc = EX.zero()
        for v in range(s.n_var):
            acc = EX.add(acc, EX.mul(xs[v], J[i][v]))
        assert _cint(acc) == _cint(EX.scale_int(F[i], degs[i]))


def test_zero_coordinates():
    """Reading C5: x_v = 0 needs no special case. x1^1 x2^2 x3^1 at x = (0, 2, 3):
    F = 0, J = (x2^2 x3, 0, 0) = (12, 0, 0); and with a_1 = 2: all zero."""
    s = system_from_terms(1, 3, 2, [[[(0, 1), (1, 2), (2, 1)]]], limbs_from_values([1], 2))
    X = limbs_from_values([0, 2, 3], 2)
    F, J = evaluate_system(s, X, "exact", workers=1)
    assert _cint(F[0]) == (0, 0)
    assert [_cint(z) for z in J[0]] == [(12, 0), (0, 0), (0, 0)]
    s = system_from_terms(1, 3, 2, [[[(0, 2), (1, 2), (2, 1)]]], limbs_from_values([1], 2))
    F, J = evaluate_system(s, X, "exact", workers=1)
    assert [_cint(z) for z in J[0]] == [(0, 0)] * 3


def test_mp512_matches_exact_c2():
    """P2: the 512-bit mode agrees with the exact mode to ~1e-140 (it is used where exact is slow)."""
    s, X = config_system("c2", seed=1)
    Fe, Je = evaluate_system(s, X[0], "exact")
    Fm, Jm = evaluate_system(s, X[0], "mp", prec=512)
    ef, _, _ = rel_errors(EX, Fe, _to_limbs(Fm))
    assert ef < 1e-140


def _to_limbs(vals, L=10):
    out = np.zeros((len(vals), 2, L))
    with mpmath.workprec(1200):
        for j, z in enumerate(vals):
            for p, part in enumerate((mpmath.re(z), mpmath.im(z))):
                r = part
                for l in range(L):
                    d = float(r)
                    out[j, p, l] = d
                    r = r - d
    return out


def test_mp_precision_doubling_large_rows():
    """P2 for the mp mode on the large config: 512 vs 1024 bits agree far below 1e-60 on sampled rows."""
    s, X = config_system("large", seed=1)
    F5, J5 = evaluate_rows(s, X[0], [0], "mp", prec=512)
    F1, J1 = evaluate_rows(s, X[0], [0], "mp", prec=1024)
    with mpmath.workprec(1100):
        assert abs(F5[0] - F1[0]) < mpmath.mpf(10) ** -140
        assert max(abs(a - b) for a, b in zip(J5[0], J1[0])) < mpmath.mpf(10) ** -140


def test_error_metric_detects_a_lost_limb():
    """The comparator sees a dropped DD low limb (~1e-17) and passes exact limbs (0)."""
    s, X = config_system("tiny", seed=1)
    F, J = evaluate_system(s, X[0], "exact", workers=1)
    lim = _to_limbs([EX.to_mpc(f) for f in F], 2)
    err, _, _ = rel_errors(EX, F, lim)
    assert err < 1e-30
    lim[3, 0, 1] = 0.0
    err, _, _ = rel_errors(EX, F, lim)
    assert err > 1e-20


# ---------------------------------------------------------------------------
# the comparators themselves (oracle/compare.py): exact_equal_limbs decides every bitwise
# P4/P5 GPU test, rel_errors every tolerance test; pin both against values built here
# from Python Fractions (independent of ExactArith.from_limbs)
# ---------------------------------------------------------------------------

def _fraction_to_exact(fr):
    """Fraction with a power-of-two denominator -> ExactArith real (m, e)."""
    num, den = fr.numerator, fr.denominator
    assert den & (den - 1) == 0
    return num, -(den.bit_length() - 1)


def _exact_from_fractions(re, im):
    (a, ea), (b, eb) = _fraction_to_exact(re), _fraction_to_exact(im)
    e = min(ea, eb)
    return (a << (ea - e), b << (eb - e), e)


def _random_limbs(rng, N, L):
    """N normalised complex values of L limbs each (leading limb ~U(-1, 1), each next limb
    below half an ulp of the previous one)."""
    out = np.zeros((N, 2, L))
    for j in range(N):
        for p in range(2):
            h = rng.uniform(-1, 1)
            for l in range(L):
                out[j, p, l] = h
                h = rng.uniform(-0.5, 0.5) * np.spacing(abs(h))
    return out


@pytest.mark.parametrize("L", [2, 4])
def test_exact_equal_limbs_pinned(L):
    from oracle import exact_equal_limbs
    rng = np.random.default_rng(11 + L)
    lim = _random_limbs(rng, 6, L)
    refs = [_exact_from_fractions(sum(Fraction(float(d)) for d in lim[j, 0]),
                                  sum(Fraction(float(d)) for d in lim[j, 1])) for j in range(6)]
    assert exact_equal_limbs(EX, refs, lim)
    # a one-ulp change of ANY limb of either part of any value is seen
    for j in (0, 5):
        for p in (0, 1):
            for l in range(L):
                bad = lim.copy()
                bad[j, p, l] = np.nextafter(bad[j, p, l], np.inf)
                assert not exact_equal_limbs(EX, refs, bad), (j, p, l)
    # conjugation (imaginary part negated) and swapped parts are seen
    bad = lim.copy()
    bad[2, 1] = -bad[2, 1]
    assert not exact_equal_limbs(EX, refs, bad)
    bad = lim.copy()
    bad[3] = bad[3, ::-1]
    assert not exact_equal_limbs(EX, refs, bad)
    # the same VALUE in a different (non-normalised) limb split is equal: values, not bits
    alt = lim.copy()
    h = alt[1, 0, 0]
    u = np.spacing(abs(h))
    alt[1, 0, 0] = h + u
    alt[1, 0, 1] = alt[1, 0, 1] - u
    assert Fraction(float(alt[1, 0, 1])) == Fraction(float(lim[1, 0, 1])) - Fraction(float(u))
    assert exact_equal_limbs(EX, refs, alt)


@pytest.mark.parametrize("fn", ["exact", "rel"])
def test_comparators_reject_length_and_shape_mismatch(fn):
    """A truncated or over-long GPU array, or one in the wrong layout, is an error: zip() would
    otherwise compare only the common prefix and pass."""
    from oracle import exact_equal_limbs
    rng = np.random.default_rng(3)
    lim = _random_limbs(rng, 5, 4)
    refs = [_exact_from_fractions(sum(Fraction(float(d)) for d in lim[j, 0]),
                                  sum(Fraction(float(d)) for d in lim[j, 1])) for j in range(5)]
    call = (lambda r, g: exact_equal_limbs(EX, r, g)) if fn == "exact" else (lambda r, g: rel_errors(EX, r, g))
    call(refs, lim)
    with pytest.raises(ValueError):
        call(refs, lim[:4])          # GPU side truncated
    with pytest.raises(ValueError):
        call(refs[:4], lim)          # oracle side truncated
    with pytest.raises(ValueError):
        call(refs, lim.transpose(0, 2, 1))  # [N][L][2] instead of [N][2][L]
    with pytest.raises(ValueError):
        call(refs, lim.reshape(5, -1))


def test_rel_errors_pinned_values():
    """rel_errors against hand-computed norms: one entry off by exactly 2^-60 in a vector whose
    largest modulus is 2 (and Frobenius norm sqrt(1 + 4 + 4)) gives max(2^-60 / 2, 2^-60 / 3)."""
    vals = [(1, 0, 0), (0, 2, 0), (2, 0, 0)]
    lim = np.zeros((3, 2, 2))
    lim[0, 0, 0], lim[1, 1, 0], lim[2, 0, 0] = 1.0, 2.0, 2.0
    assert rel_errors(EX, vals, lim)[0] == 0.0
    lim[1, 0, 1] = 2.0 ** -60           # real part of entry 1 gains 2^-60
    err, dmax, rmax = rel_errors(EX, vals, lim)
    assert dmax == 2.0 ** -60 and rmax == 2.0
    assert err == pytest.approx(2.0 ** -61, rel=1e-12)  # inf-norm ratio 2^-61 > Frobenius 2^-60/3
