"""GPU parity for NEXT-2, common-support systems and the two-stage evaluation (Alg. 2
V -> Y; Table 1 system shape P:355-358): the CUDA path through
phc_system_create_common against the oracle on the expanded system (the plain definition),
against the per-term path on the same polynomials, sharding, structural zeros, Newton."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from _parity import TOL, compare_point, limbs_normalised, oracle_point  # noqa: E402
from synthetic import common_config, common_support_system, expand_common  # noqa: E402


@pytest.fixture(scope="module")
def phc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1109_0545_b200 as m
    return m


def _eval(h, X, devices=None):
    F, J = h.eval_batch(torch.from_numpy(np.ascontiguousarray(X)).cuda(), devices=devices)
    torch.cuda.synchronize()
    return F.cpu().numpy(), J.cpu().numpy()


@pytest.mark.parametrize("L,seed", [(2, 1), (2, 2), (4, 1)])
def test_small_common_vs_exact_oracle(phc, L, seed):
    c, X = common_support_system(8, 12, 1, 6, 3, L, seed=seed, points=3)
    h = phc.System(c)
    F, J = _eval(h, X)
    e = expand_common(c)
    for p in range(3):
        ar, Fr, Jr = oracle_point(e, X[p], arith="exact")
        ef, ej = compare_point(ar, Fr, Jr, F[p], J[p], L)
        assert ef <= TOL[L] and ej <= TOL[L], (p, ef, ej)
    assert limbs_normalised(F) and limbs_normalised(J)


@pytest.mark.parametrize("name", ["common_dd", "common"])
def test_table1_shape_sampled_rows(phc, name):
    """n = 40, M = 200 shared monomials, k in 10..30, exponents 1..3 (average degree 40)."""
    c, X = common_config(name, seed=1, points=2)
    h = phc.System(c)
    F, J = _eval(h, X)
    e = expand_common(c)
    rows = [0, 23, 39]
    ar, Fr, Jr = oracle_point(e, X[1], rows=rows, arith="exact" if c.limbs == 2 else "mp")
    ef, ej = compare_point(ar, Fr, Jr, F[1], J[1], c.limbs, rows)
    assert ef <= TOL[c.limbs] and ej <= TOL[c.limbs], (ef, ej)


def test_common_matches_per_term_path(phc):
    """Same polynomials through the per-term path (expanded system): equal within tolerance
    (different summation order, so not bitwise)."""
    c, X = common_config("common_dd", seed=2, points=4)
    F1, J1 = _eval(phc.System(c), X)
    F2, J2 = _eval(phc.System(expand_common(c)), X)
    import mpmath
    with mpmath.workprec(300):
        for a, b in ((F1, F2), (J1, J2)):
            va = a[..., 0] + a[..., 1]
            vb = b[..., 0] + b[..., 1]
            assert np.max(np.abs(va - vb)) <= 1e-26 * max(1.0, np.max(np.abs(vb)))


def test_common_sharded_bitwise_and_unused_variable(phc):
    c, X = common_support_system(10, 30, 1, 4, 3, 2, seed=4, points=21)
    # drop every factor on x_7: its Jacobian column must then be exactly zero
    keep = c.var_idx != 7
    counts = np.add.reduceat(keep.astype(np.int64), c.mono_ptr[:-1]) if keep.size else np.zeros(c.n_mono, np.int64)
    counts[np.diff(c.mono_ptr) == 0] = 0
    c.mono_ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    c.var_idx, c.exponent = c.var_idx[keep].copy(), c.exponent[keep].copy()
    h = phc.System(c)
    F1, J1 = _eval(h, X)
    F4, J4 = _eval(h, X, devices=[0, 0, 0, 0])
    assert np.array_equal(F1, F4) and np.array_equal(J1, J4)
    assert (J1[:, :, 7] == 0).all()


def test_newton_on_common_system_converges(phc):
    """Quadratic convergence to a constructed root: shift the constant column so that a chosen
    point z is a root (f_i(z) = 0), start near z, watch the residual fall to the floor."""
    c, X = common_support_system(12, 40, 1, 3, 2, 2, seed=5, points=1)
    # append the constant monomial and set its coefficients to -sum_j C[i][j] z^{a_j} (host,
    # via the GPU evaluator of the system without it: F(z) then C0 = -F(z))
    c.mono_ptr = np.append(c.mono_ptr, c.mono_ptr[-1])
    c.coeff = np.concatenate([c.coeff, np.zeros((12, 1, 2, 2))], axis=1)
    h0 = phc.System(c)
    z = X[0]
    F0, _ = _eval(h0, z[None])
    c.coeff[:, -1] = -F0[0]
    h = phc.System(c)
    x = torch.from_numpy((z * (1 + 1e-3))[None].copy()).cuda()
    res = []
    for _ in range(7):
        x, r, st = h.newton_step(x)
        torch.cuda.synchronize()
        assert int(st[0]) == 0
        res.append(float(r[0]))
    assert res[0] > 1e-5 and res[-1] < 1e-28, res


@pytest.mark.parametrize("L", [2, 4])
def test_common_homotopy_vs_oracle_and_endpoints(phc, L):
    """Homotopy coefficients on a common-support handle: h(x, t) with the dense start and
    target matrices blended per entry, against the homotopy oracle on the expanded system;
    t = 0 / 1 bitwise the plain start / target evaluations."""
    from oracle.homotopy import evaluate_homotopy_rows
    from synthetic import random_t, real_limbs
    c, X = common_support_system(9, 14, 1, 5, 3, L, seed=7, points=3)
    from synthetic.systems import unit_circle_limbs
    ct = unit_circle_limbs(np.random.default_rng(3).uniform(0, 6.283, (9, 14)), L, 1)
    h = phc.System(c, coeff_target=ct)
    T = random_t(3, L, seed=8)
    F, J = h.eval_homotopy_batch(torch.from_numpy(X).cuda(), torch.from_numpy(T).cuda())
    torch.cuda.synchronize()
    e = expand_common(c)
    for p in range(3):
        ar, Fr, Jr = evaluate_homotopy_rows(e, ct.reshape(-1, 2, L), X[p], T[p], arith="exact" if L == 2 else "mp")
        ef, ej = compare_point(ar, Fr, Jr, F[p].cpu().numpy(), J[p].cpu().numpy(), L)
        assert ef <= TOL[L] and ej <= TOL[L], (p, ef, ej)
    T01 = torch.from_numpy(real_limbs([0, 1, 0], L)).cuda()
    F01, J01 = h.eval_homotopy_batch(torch.from_numpy(X).cuda(), T01)
    Fs, Js = phc.System(c).eval_batch(torch.from_numpy(X).cuda())
    c2 = type(c)(c.n_eq, c.n_var, L, c.mono_ptr, c.var_idx, c.exponent, ct)
    Ft, Jt = phc.System(c2).eval_batch(torch.from_numpy(X).cuda())
    torch.cuda.synchronize()
    assert torch.equal(F01[0], Fs[0]) and torch.equal(J01[0], Js[0])
    assert torch.equal(F01[1], Ft[1]) and torch.equal(J01[1], Jt[1])


def test_track_on_common_support_handle(phc):
    """The total-degree homotopy shares one support across its polynomials: tracked through a
    common-support handle (two-stage evaluation) the 8 paths reach the same end points as
    through the per-term handle (within the tolerance)."""
    from synthetic import as_common, total_degree_homotopy
    s, cf, X0 = total_degree_homotopy(3, 2, seed=7)
    c, cft = as_common(s, cf)
    X = torch.from_numpy(X0).cuda()
    Xa, sa, _ = phc.System(s, coeff_target=cf).track(X)
    Xb, sb, _ = phc.System(c, coeff_target=cft).track(X)
    assert (sa == 1).all() and (sb == 1).all()
    za = Xa.cpu().numpy()
    zb = Xb.cpu().numpy()
    d = np.abs((za[..., 0] + za[..., 1]) - (zb[..., 0] + zb[..., 1])).max()
    assert d <= 1e-25, d
