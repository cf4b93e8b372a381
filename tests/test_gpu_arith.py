"""GPU unit tests of the DD/QD arithmetic core (pin P12; SPEC S:90-91,
S:616-617): the error-free transformations are exact (checked in rationals), the DD/QD
operations are accurate to their normwise bounds, outputs are normalised.  The device side
runs through the phc_arith_test hook; every expected value is an exact rational."""
from fractions import Fraction as Fr

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from _parity import limbs_normalised  # noqa: E402
from synthetic import real_limbs  # noqa: E402


@pytest.fixture(scope="module")
def phc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1109_0545_b200 as m
    return m


def run(phc, op, L, a, b, out_shape):
    from paper_1109_0545_b200.system import _ptr
    ad, bd = torch.from_numpy(np.ascontiguousarray(a)).cuda(), torch.from_numpy(np.ascontiguousarray(b)).cuda()
    out = torch.empty(out_shape, dtype=torch.float64, device="cuda")
    phc.phc_arith_test(op, L, int(a.shape[0]), _ptr(ad), _ptr(bd), _ptr(out), None)
    torch.cuda.synchronize()
    return out.cpu().numpy()


def ex(limbs):
    return sum((Fr(float(d)) for d in limbs), Fr(0))


def rand_reals(rng, n, L, spread=20):
    """n random reals with full L-limb precision and exponents in [-spread, spread]."""
    vals = []
    for _ in range(n):
        m = 1
        for _c in range(L):  # every bit of the 62 L-bit mantissa random
            m = (m << 62) | int(rng.integers(1 << 62))
        sgn = -1 if rng.random() < 0.5 else 1
        v = Fr(sgn * m, 1 << (62 * L)) * Fr(2) ** int(rng.integers(-spread, spread))
        vals.append(v)
    return vals


def test_two_sum_two_prod_exact(phc):
    rng = np.random.default_rng(1)
    n = 1 << 18
    a = rng.standard_normal(n) * 2.0 ** rng.integers(-60, 60, n)
    b = rng.standard_normal(n) * 2.0 ** rng.integers(-60, 60, n)
    s = run(phc, 0, 2, a, b, (n, 2))
    assert np.array_equal(s[:, 0], a + b)  # s = fl(a + b)
    p = run(phc, 1, 2, a, b, (n, 2))
    assert np.array_equal(p[:, 0], a * b)  # p = fl(a b)
    for i in rng.choice(n, 4000, replace=False):
        assert Fr(s[i, 0]) + Fr(s[i, 1]) == Fr(a[i]) + Fr(b[i])
        assert Fr(p[i, 0]) + Fr(p[i, 1]) == Fr(a[i]) * Fr(b[i])


@pytest.mark.parametrize("L", [2, 4])
def test_real_ops_accuracy(phc, L):
    rng = np.random.default_rng(10 + L)
    n = 3000
    A, B = rand_reals(rng, n, L), rand_reals(rng, n, L)
    a, b = real_limbs(A, L), real_limbs(B, L)
    u = Fr(1, 2 ** (53 * L))
    # measured maxima over these samples (tools/arith_errors.py), in u = 2^(-53 L):
    # DD add 1.47, mul 2.05, div 1.91; QD add 0.11, mul 1.35, div 0.82 -> bounds ~2x above
    bound = {"add": 4 * u, "mul": 5 * u, "div": 5 * u}
    for op, name, f in ((2, "add", lambda x, y: x + y), (3, "mul", lambda x, y: x * y), (4, "div", lambda x, y: x / y)):
        out = run(phc, op, L, a, b, (n, L))
        assert limbs_normalised(out[:, None, :])
        for i in range(n):
            xa, xb = ex(a[i]), ex(b[i])
            ref = f(xa, xb)
            scale = abs(xa) + abs(xb) if name == "add" else abs(ref)
            assert abs(ex(out[i]) - ref) <= bound[name] * scale, (name, i)
    # times a double
    d = rng.standard_normal(n)
    bd = np.zeros((n, L))
    bd[:, 0] = d
    out = run(phc, 9, L, a, bd, (n, L))
    for i in range(n):
        ref = ex(a[i]) * Fr(d[i])
        assert abs(ex(out[i]) - ref) <= 4 * u * abs(ref)


@pytest.mark.parametrize("L", [2, 4])
def test_complex_ops_accuracy(phc, L):
    rng = np.random.default_rng(20 + L)
    n = 2000
    a = np.stack([real_limbs(rand_reals(rng, n, L, 4), L), real_limbs(rand_reals(rng, n, L, 4), L)], axis=1)
    b = np.stack([real_limbs(rand_reals(rng, n, L, 4), L), real_limbs(rand_reals(rng, n, L, 4), L)], axis=1)
    u = Fr(1, 2 ** (53 * L))
    mods = lambda z: (z[0] * z[0] + z[1] * z[1])  # noqa: E731  (|z|^2, exact)
    for op in (5, 7):  # product (normalised), lazy product + renormalisation (the hot path's)
        out = run(phc, op, L, a, b, (n, 2, L))
        assert limbs_normalised(out)
        for i in range(n):
            ar, ai, br, bi = ex(a[i, 0]), ex(a[i, 1]), ex(b[i, 0]), ex(b[i, 1])
            rr, ri = ar * br - ai * bi, ar * bi + ai * br
            d2 = (ex(out[i, 0]) - rr) ** 2 + (ex(out[i, 1]) - ri) ** 2
            # measured max 4.59 u (DD), 1.54 u (QD), normwise
            assert d2 <= (10 * u) ** 2 * mods((ar, ai)) * mods((br, bi)), (op, i)
    out = run(phc, 6, L, a, b, (n, 2, L))
    for i in range(n):
        for c in (0, 1):
            xa, xb = ex(a[i, c]), ex(b[i, c])
            assert abs(ex(out[i, c]) - (xa + xb)) <= 4 * u * (abs(xa) + abs(xb))
    out = run(phc, 8, L, a, b, (n, 2, L))
    for i in range(n):
        ar, ai = ex(a[i, 0]), ex(a[i, 1])
        m2 = mods((ar, ai))
        rr, ri = ar / m2, -ai / m2
        d2 = (ex(out[i, 0]) - rr) ** 2 + (ex(out[i, 1]) - ri) ** 2
        assert d2 <= (8 * u) ** 2 / m2, i  # measured max 2.99 u (DD), 2.42 u (QD)


def test_signed_zero_and_exact_cases(phc):
    """Exactly representable products and sums come out exact and normalised (P5)."""
    for L in (2, 4):
        a = np.zeros((4, 2, L))
        b = np.zeros((4, 2, L))
        a[:, 0, 0] = [3, -2, 0, 1.5]
        a[:, 1, 0] = [1, 0.5, -4, 0]
        b[:, 0, 0] = [2, 8, 1, -0.25]
        b[:, 1, 0] = [-1, 0, 2, 0.75]
        out = run(phc, 5, L, a, b, (4, 2, L))
        za = a[:, 0, 0] + 1j * a[:, 1, 0]
        zb = b[:, 0, 0] + 1j * b[:, 1, 0]
        z = za * zb
        assert np.array_equal(out[:, 0, 0], z.real) and np.array_equal(out[:, 1, 0], z.imag)
        assert (out[:, :, 1:] == 0).all()


@pytest.mark.parametrize("L", [2, 4])
def test_warp_reciprocal_equals_reciprocal(phc, L):
    """The eliminations' pivot reciprocal (recip_warp: the two long divisions on two lanes)
    is P::recip bitwise, including signed zeros and tiny/huge moduli."""
    rng = np.random.default_rng(40 + L)
    n = 4000
    a = np.stack([real_limbs(rand_reals(rng, n, L, 30), L), real_limbs(rand_reals(rng, n, L, 30), L)], axis=1)
    a[:5, 1] = 0.0                       # real operands
    a[5:10, 0] = 0.0                     # imaginary operands
    a[10:15, 1] = -0.0
    r8 = run(phc, 8, L, a, a, (n, 2, L))
    r10 = run(phc, 10, L, a, a, (n, 2, L))
    assert np.array_equal(r8.view(np.uint64), r10.view(np.uint64))
