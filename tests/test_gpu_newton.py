"""GPU parity for NEXT-1, one Newton iteration (Alg. 2): the CUDA step
(evaluation + GE with partial pivoting + back substitution + update) against the exact
oracle step; quadratic convergence to a known root at full size; singular pivots."""
import math

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import newton_step  # noqa: E402
from synthetic import config_system, limbs_from_values, system_from_terms  # noqa: E402


@pytest.fixture(scope="module")
def phc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1109_0545_b200 as m
    return m


def _tol(L, n, cond):
    """Normwise error budget of one DD/QD Newton step: the evaluation error (<= 1e-28 / 1e-60
    relative) and the elimination's backward error (~ n u) are amplified by cond(J)."""
    u = 2.0 ** -104 if L == 2 else 2.0 ** -209
    return max(1e-28 if L == 2 else 1e-60, 64 * n * u * cond)


def _gpu_step(phc, s, X):
    h = phc.System(s)
    Xd = torch.from_numpy(np.ascontiguousarray(X)).cuda()
    Xn, res, status = h.newton_step(Xd)
    torch.cuda.synchronize()
    return Xn.cpu().numpy(), res.cpu().numpy(), status.cpu().numpy(), h


def _check_point(s, Xp, xn, res):
    """Normwise error of the GPU's new point against the oracle step (mp512 evaluation and
    mpmath.lu_solve; exact rationals only for the tiny config), relative to ||dz||."""
    import mpmath
    arith = "exact" if s.n_var <= 8 else "mp"
    out = newton_step(s, Xp, arith)
    assert not out["singular"]
    with mpmath.workprec(1024):
        if arith == "exact":
            ref = [mpmath.mpc(mpmath.mpf(a[0].numerator) / a[0].denominator, mpmath.mpf(a[1].numerator) / a[1].denominator)
                   for a in out["z_new"]]
            dz = [mpmath.mpc(mpmath.mpf(a[0].numerator) / a[0].denominator, mpmath.mpf(a[1].numerator) / a[1].denominator)
                  for a in out["dz"]]
        else:
            ref, dz = out["z_new"], out["dz"]
        got = [mpmath.mpc(mpmath.fsum(mpmath.mpf(float(d)) for d in v[0]), mpmath.fsum(mpmath.mpf(float(d)) for d in v[1]))
               for v in xn]
        num = max(abs(a - b) for a, b in zip(got, ref))
        den = max(abs(d) for d in dz)
    assert res == pytest.approx(out["residual"], rel=1e-12)
    return float(num / den)


@pytest.mark.parametrize("name,seed", [("tiny", 1), ("tiny", 2), ("c2", 1), ("c3", 1)])
def test_newton_step_vs_exact_oracle(phc, name, seed):
    s, X = config_system(name, seed=seed)
    xn, res, status, h = _gpu_step(phc, s, X)
    assert status[0] == 0
    # condition number of J (float64) for the error budget
    F, Jd = h.eval(torch.from_numpy(X[0]).cuda())
    Jc = Jd.cpu().numpy()[..., 0, 0] + 1j * Jd.cpu().numpy()[..., 1, 0]
    cond = np.linalg.cond(Jc)
    err = _check_point(s, X[0], xn[0], res[0])
    assert err <= _tol(s.limbs, s.n_var, cond), (err, cond)


def test_newton_step_batch_sampled(phc):
    s, X = config_system("batch", seed=2, points=4096)
    xn, res, status, h = _gpu_step(phc, s, X)
    assert (status == 0).all()
    F, J = h.eval_batch(torch.from_numpy(X[[0, 1000, 4095]]).cuda())
    Jn = J.cpu().numpy()
    for k, p in enumerate((0, 1000, 4095)):
        cond = np.linalg.cond(Jn[k][..., 0, 0] + 1j * Jn[k][..., 1, 0])
        err = _check_point(s, X[p], xn[p], res[p])
        assert err <= _tol(2, 32, cond), (p, err, cond)


def _root_system(n, k, L, seed):
    """f_i(x) = sum_t c_t (m_t(x) - 1): vanishes at x = (1, ..., 1) exactly."""
    rng = np.random.default_rng(seed)
    polys, coeffs = [], []
    for i in range(n):
        terms = [[(v, int(rng.integers(1, 4))) for v in sorted(rng.choice(n, k, replace=False).tolist())]
                 for _ in range(6)]
        terms.append([(i, 1)])  # keeps J well conditioned near the root
        c = [complex(*rng.integers(-3, 4, 2)) or 1 for _ in terms]
        c[-1] = complex(4 * k + 8, 1)
        polys.append(terms + [[]])
        coeffs += c + [-sum(c)]
    return system_from_terms(n, n, L, polys, limbs_from_values(coeffs, L))


@pytest.mark.parametrize("n,k,L,steps,tol", [(32, 8, 2, 4, 1e-29), (40, 10, 4, 5, 1e-61), (256, 16, 4, 5, 1e-60)])
def test_newton_converges_quadratically_to_known_root(phc, n, k, L, steps, tol):
    """At any size (incl. the n = 256 QD global-memory elimination): from x* + delta the error
    roughly squares each step down to the working precision."""
    s = _root_system(n, k, L, seed=n)
    rng = np.random.default_rng(7)
    x0 = [1 + 1e-3 * complex(*rng.uniform(-1, 1, 2)) for _ in range(n)]
    X = torch.from_numpy(limbs_from_values(x0, L)[None].copy()).cuda()
    h = phc.System(s)
    errs = []
    for _ in range(steps):
        X, res, status = h.newton_step(X, X)  # in place
        torch.cuda.synchronize()
        assert int(status[0]) == 0
        x = X.cpu().numpy()[0]
        re = x[:, 0, :].sum(axis=1) - 1.0  # limb sums in float64 suffice for the first steps
        e_hi = max(abs(x[:, 0, 0] - 1.0).max(), abs(x[:, 1, 0]).max())
        errs.append(e_hi)
    assert errs[0] < 1e-4 and errs[1] < 1e-7
    # final: exact error from the limbs
    from fractions import Fraction
    x = X.cpu().numpy()[0]
    final = max(abs(complex(float(sum(Fraction(float(d)) for d in x[v, 0]) - 1), float(sum(Fraction(float(d)) for d in x[v, 1]))))
                for v in range(n))
    assert final <= tol, final


def test_newton_singular_and_in_place(phc):
    """A variable absent from the system gives a zero Jacobian column: status 1, x unchanged.
    In-place and out-of-place steps agree bitwise."""
    s = system_from_terms(2, 2, 2, [[[(0, 2)], []], [[(0, 1)], []]], limbs_from_values([1, -4, 1, 2], 2))
    X = torch.from_numpy(limbs_from_values([3, 5], 2)[None].copy()).cuda()
    h = phc.System(s)
    Xn, res, status = h.newton_step(X)
    torch.cuda.synchronize()
    assert int(status[0]) == 1 and torch.equal(Xn, X)
    s2, X2 = config_system("c2", seed=3, points=8)
    h2 = phc.System(s2)
    A = torch.from_numpy(X2).cuda()
    B = A.clone()
    out, _, _ = h2.newton_step(A)
    h2.newton_step(B, B)
    torch.cuda.synchronize()
    assert torch.equal(out, B)


@pytest.mark.parametrize("coop", ["0", "1"])
def test_newton_multi_kernel_path_vs_oracle(phc, monkeypatch, coop):
    """n = 64 QD: [J | -F] (266 KB) exceeds shared memory, so the elimination runs in global
    memory over many SMs: two launches per column (multi-kernel path, coop = 0) or one
    cooperative launch with a grid barrier per column (coop = 1)."""
    monkeypatch.setenv("PHC_NEWTON_COOP", coop)
    from synthetic import random_system
    s, X = random_system(64, 8, 6, 3, 4, seed=3, points=2)
    xn, res, status, h = _gpu_step(phc, s, X)
    assert (status == 0).all()
    F, Jd = h.eval_batch(torch.from_numpy(X).cuda())
    for p in (0, 1):
        Jc = Jd.cpu().numpy()[p][..., 0, 0] + 1j * Jd.cpu().numpy()[p][..., 1, 0]
        cond = np.linalg.cond(Jc)
        err = _check_point(s, X[p], xn[p], res[p])
        assert err <= _tol(4, 64, cond), (p, err, cond)


@pytest.mark.parametrize("coop", ["0", "1"])
def test_newton_multi_kernel_singular(phc, monkeypatch, coop):
    """Global-memory paths: a variable absent from the system -> zero pivot column -> status 1,
    x unchanged, for both points."""
    monkeypatch.setenv("PHC_NEWTON_COOP", coop)
    from synthetic import random_system
    s, X = random_system(60, 6, 5, 2, 4, seed=4, points=2)
    keep = s.var_idx != 59
    counts = np.add.reduceat(keep.astype(np.int64), s.term_ptr[:-1])
    counts[np.diff(s.term_ptr) == 0] = 0
    s.term_ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    s.var_idx, s.exponent = s.var_idx[keep].copy(), s.exponent[keep].copy()
    xn, res, status, h = _gpu_step(phc, s, X)
    assert (status == 1).all()
    assert np.array_equal(xn, X)


@pytest.mark.parametrize("name", ["c2", "batch"])
def test_warp_and_cta_eliminations_agree_bitwise(phc, name):
    """16 < n <= 32: below 4,096 points the elimination runs one warp per point, from 4,096 on
    one CTA per point; both perform the same operations in the same order, so the steps are
    bitwise equal (4,096 vs 4,095 points: the evaluation takes the batch kernel in both)."""
    s, X = config_system(name, seed=4, points=4096)
    h = phc.System(s)
    Xd = torch.from_numpy(X).cuda()
    Xa, ra, sa = h.newton_step(Xd)          # 4,096 points: CTA kernel
    Xb, rb, sb = h.newton_step(Xd[:4095])   # 4,095 points: warp kernel
    torch.cuda.synchronize()
    assert (sa == 0).all() and (sb == 0).all()
    assert torch.equal(Xa[:4095], Xb) and torch.equal(ra[:4095], rb)


def test_newton_cta_kernel_singular_and_lookahead_pivot(phc):
    """The shared-memory CTA elimination (n = 40 QD, one point): a variable absent from the
    system gives a zero pivot column found by the look-ahead warp -> status 1, x unchanged;
    the other point of the batch (a regular system) is solved."""
    from synthetic import random_system
    s, X = random_system(40, 6, 5, 2, 4, seed=6, points=2)
    keep = s.var_idx != 39
    counts = np.add.reduceat(keep.astype(np.int64), s.term_ptr[:-1])
    counts[np.diff(s.term_ptr) == 0] = 0
    s.term_ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    s.var_idx, s.exponent = s.var_idx[keep].copy(), s.exponent[keep].copy()
    xn, res, status, h = _gpu_step(phc, s, X)
    assert (status == 1).all()
    assert np.array_equal(xn, X)
    s2, X2 = random_system(40, 6, 5, 2, 4, seed=7, points=1)
    xn2, res2, st2, _ = _gpu_step(phc, s2, X2)
    assert st2[0] == 0


@pytest.mark.parametrize("name,points", [("c3", 3), ("c2", 2)])
def test_global_eliminations_equal_shared_memory_kernel_bitwise(phc, monkeypatch, name, points):
    """The three CTA-level eliminations -- shared memory (one CTA per point), multi-kernel and
    cooperative (global memory, forced with PHC_NEWTON_GLOBAL) -- make the same pivot choices
    and the same operations per entry in the same order: bitwise equal steps."""
    s, X = config_system(name, seed=9, points=points)
    h = phc.System(s)
    Xd = torch.from_numpy(X).cuda()
    monkeypatch.setenv("PHC_NEWTON_WARP", "0")
    ref = h.newton_step(Xd)
    torch.cuda.synchronize()
    monkeypatch.setenv("PHC_NEWTON_GLOBAL", "1")
    for coop in ("0", "1"):
        monkeypatch.setenv("PHC_NEWTON_COOP", coop)
        out = h.newton_step(Xd)
        torch.cuda.synchronize()
        for a, b in zip(ref, out):
            assert torch.equal(a, b), coop


def test_cooperative_elimination_singular_first_column(phc, monkeypatch):
    """Cooperative path, zero pivot in column 0 (variable 0 absent): status 1, x unchanged."""
    from synthetic import random_system
    s, X = random_system(40, 6, 5, 2, 4, seed=8, points=1)
    keep = s.var_idx != 0
    counts = np.add.reduceat(keep.astype(np.int64), s.term_ptr[:-1])
    counts[np.diff(s.term_ptr) == 0] = 0
    s.term_ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    s.var_idx, s.exponent = s.var_idx[keep].copy(), s.exponent[keep].copy()
    monkeypatch.setenv("PHC_NEWTON_GLOBAL", "1")
    monkeypatch.setenv("PHC_NEWTON_COOP", "1")
    xn, res, status, h = _gpu_step(phc, s, X)
    assert status[0] == 1
    assert np.array_equal(xn, X)


@pytest.mark.parametrize("seed", range(int(__import__("os").environ.get("PHC_FUZZ_SEEDS_NEWTON", "12"))))
def test_newton_fuzz_shapes(phc, seed):
    """Random square systems of varied size and precision through every elimination regime
    (warp kernel n <= 32, shared-memory CTA kernel, cooperative and multi-kernel global
    paths for matrices beyond shared memory), each sampled point against the oracle step
    within the error budget."""
    from synthetic import random_system
    rng = np.random.Generator(np.random.PCG64(500 + seed))
    L = int(rng.choice([2, 4]))
    n = int(rng.choice([3, 9, 20, 33, 45, 70]))
    P = int(rng.choice([1, 2, 6]))
    m = int(rng.integers(3, 9))
    k = int(min(n, rng.integers(1, 6)))
    s, X = random_system(n, m, k, int(rng.integers(1, 4)), L, seed=600 + seed, points=P)
    xn, res, status, h = _gpu_step(phc, s, X)
    F, Jd = h.eval_batch(torch.from_numpy(X).cuda())
    for p in sorted({0, P - 1}):
        Jc = Jd.cpu().numpy()[p][..., 0, 0] + 1j * Jd.cpu().numpy()[p][..., 1, 0]
        cond = np.linalg.cond(Jc)
        if not np.isfinite(cond) or cond > 1e12:
            continue  # numerically singular draw: nothing to compare at this precision
        assert status[p] == 0
        err = _check_point(s, X[p], xn[p], res[p])
        assert err <= _tol(L, n, cond), (seed, n, L, P, p, err, cond)


@pytest.mark.parametrize("n,k,L,tol", [(12, 4, 2, 1e-26), (40, 10, 4, 1e-55)])
def test_newton_solve_equals_repeated_steps(phc, n, k, L, tol):
    """Alg. 2 to tolerance (phc_newton_solve_batch) from points near a known root: every point
    stops after the iteration whose residual (tested before its update) passed tol; its
    result, residual and iteration count equal those of calling the Newton step the same
    number of times (bitwise), and the result is the root to working precision."""
    s = _root_system(n, k, L, seed=n + 1)
    rng = np.random.default_rng(3)
    P = 5
    x0 = [[1 + d * complex(*rng.uniform(-1, 1, 2)) for _ in range(n)] for d in (1e-2, 1e-3, 1e-4, 1e-6, 1e-9)]
    X = torch.from_numpy(np.stack([limbs_from_values(v, L) for v in x0])).cuda()
    h = phc.System(s)
    Xo, res, its, st = h.newton_solve(X, tol, 20)
    torch.cuda.synchronize()
    assert (st == 0).all(), (st, its, res)
    its = its.cpu().numpy()
    assert len(set(its.tolist())) > 1  # the points stop at different iterations
    for p in range(P):
        Y = X[p:p + 1].clone()
        last = None
        for _ in range(int(its[p])):
            Y, r, sp = h.newton_step(Y, Y)
            last = r
        torch.cuda.synchronize()
        assert torch.equal(Y[0], Xo[p]) and float(last[0]) == float(res[p])
        assert float(res[p]) <= tol
    from fractions import Fraction
    xo = Xo.cpu().numpy()
    err = max(abs(complex(float(sum(Fraction(float(d)) for d in xo[p, v, 0]) - 1), float(sum(Fraction(float(d)) for d in xo[p, v, 1]))))
              for p in range(P) for v in range(n))
    assert err <= (1e-28 if L == 2 else 1e-60), err


def test_newton_solve_edge_cases(phc):
    """max_it = 0 (point returned, residual 1, status fail unless tol > 1), max_it reached
    (status 1), a singular Jacobian (status 2, point where it was met), the SPEC example
    x^2 - 4 from x = 1 converging to 2."""
    L = 2
    s = system_from_terms(1, 1, L, [[[(0, 2)], []]], limbs_from_values([1, -4], L))
    h = phc.System(s)
    X = torch.from_numpy(limbs_from_values([1.0], L)[None].copy()).cuda()
    Xo, res, its, st = h.newton_solve(X, 1e-25, 0)
    torch.cuda.synchronize()
    assert torch.equal(Xo, X) and int(its[0]) == 0 and float(res[0]) == 1.0 and int(st[0]) == 1
    Xo, res, its, st = h.newton_solve(X, 1e-25, 2)
    assert int(st[0]) == 1 and int(its[0]) == 2
    Xo, res, its, st = h.newton_solve(X, 1e-25, 30)
    torch.cuda.synchronize()
    assert int(st[0]) == 0 and int(its[0]) < 30
    z = Xo.cpu().numpy()[0, 0]
    assert abs(float(z[0, 0]) - 2.0) == 0.0 and abs(z[0, 1]) < 1e-30 and z[1, 0] == 0.0
    # singular at the start: f = x^2 + 1 at x = 0 -> residual 1, J = 0
    s0 = system_from_terms(1, 1, L, [[[(0, 2)], []]], limbs_from_values([1, 1], L))
    X0 = torch.zeros((1, 1, 2, L), dtype=torch.float64, device="cuda")
    Xo, res, its, st = phc.System(s0).newton_solve(X0, 1e-25, 5)
    torch.cuda.synchronize()
    assert int(st[0]) == 2 and int(its[0]) == 1 and torch.equal(Xo, X0)


def test_newton_solve_tol_at_least_one_runs_no_iteration(phc):
    """Alg. 2 starts from ||h|| := 1 and loops while ||h|| > tol: with tol >= 1 the
    loop body never runs, so x_out = x, iterations 0, residual 1, and fail := ||h|| >= tol
    (status 1 for tol = 1, 0 for tol = 2)."""
    L = 2
    s = system_from_terms(1, 1, L, [[[(0, 2)], []]], limbs_from_values([1, -4], L))
    h = phc.System(s)
    X = torch.from_numpy(limbs_from_values([1.0], L)[None].copy()).cuda()
    for tol, want in ((1.0, 1), (2.0, 0)):
        Xo, res, its, st = h.newton_solve(X, tol, 5)
        torch.cuda.synchronize()
        assert torch.equal(Xo, X) and int(its[0]) == 0 and float(res[0]) == 1.0 and int(st[0]) == want, tol


def _nan_f_finite_j_system(L):
    """f(x) = x^3 - x^3 + x at x = 1e103: x^3 overflows in the evaluation (F = NaN), while
    J = 3x^2 - 3x^2 + 1 = 1 stays finite."""
    s = system_from_terms(1, 1, L, [[[(0, 3)], [(0, 3)], [(0, 1)]]], limbs_from_values([1, -1, 1], L))
    X = limbs_from_values([1e103], L)[None].copy()
    return s, X


@pytest.mark.parametrize("regime", ["warp", "cta", "multi", "coop"])
@pytest.mark.parametrize("L", [2, 4])
def test_newton_nan_residual_is_reported(phc, monkeypatch, regime, L):
    """A NaN in F with a finite J reaches the residual (not dropped by a max reduction) in every
    elimination regime, and Alg. 2 to tolerance reports the point as failed (status 1)."""
    env = {"warp": {"PHC_NEWTON_WARP": "1"}, "cta": {"PHC_NEWTON_WARP": "0"},
           "multi": {"PHC_NEWTON_GLOBAL": "1", "PHC_NEWTON_COOP": "0"},
           "coop": {"PHC_NEWTON_GLOBAL": "1", "PHC_NEWTON_COOP": "1"}}[regime]
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    s, X = _nan_f_finite_j_system(L)
    h = phc.System(s)
    Xd = torch.from_numpy(X).cuda()
    F, J = h.eval_batch(Xd)
    torch.cuda.synchronize()
    assert torch.isnan(F).any() and bool(torch.isfinite(J).all())
    Xn, res, status = h.newton_step(Xd)
    torch.cuda.synchronize()
    assert math.isnan(float(res[0])) and int(status[0]) == 0
    Xo, res, its, st = h.newton_solve(Xd, 1e-20, 4)
    torch.cuda.synchronize()
    assert int(st[0]) == 1 and int(its[0]) == 1 and math.isnan(float(res[0]))


def test_cooperative_elimination_singular_middle_column_repeated(phc, monkeypatch):
    """Cooperative path, zero pivot in a MIDDLE column (variable 30 of 60 absent): CTA 0 finds it
    in the look-ahead of iteration 29 while the other CTAs start that iteration; the per-column
    flag slots keep every CTA on the same grid barrier count.  Repeated to give the race a
    chance; every call ends (no hang) with status 1 and x unchanged."""
    from synthetic import random_system
    s, X = random_system(60, 6, 5, 2, 4, seed=14, points=2)
    keep = s.var_idx != 30
    counts = np.add.reduceat(keep.astype(np.int64), s.term_ptr[:-1])
    counts[np.diff(s.term_ptr) == 0] = 0
    s.term_ptr = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    s.var_idx, s.exponent = s.var_idx[keep].copy(), s.exponent[keep].copy()
    monkeypatch.setenv("PHC_NEWTON_GLOBAL", "1")
    monkeypatch.setenv("PHC_NEWTON_COOP", "1")
    h = phc.System(s)
    Xd = torch.from_numpy(X).cuda()
    for _ in range(25):
        Xn, res, status = h.newton_step(Xd)
    torch.cuda.synchronize()
    assert (status.cpu().numpy() == 1).all() and torch.equal(Xn, Xd)
