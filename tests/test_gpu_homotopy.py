"""GPU parity for NEXT-3, homotopy coefficients (§7, reading H1): the CUDA
evaluation of h(x, t) = sum ((1-t) c_s + t c_f) x^a with a per-point t against the homotopy
oracle; reductions to the plain evaluator at t = 0 and t = 1; the "old" t-as-variable
evaluator (phc_homotopy_old_create) against the new one and against the oracle's dh/dt;
sharding; Newton on h(., t)."""
from dataclasses import replace

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from _parity import TOL, compare_point, limbs_normalised  # noqa: E402
from oracle import rel_errors  # noqa: E402
from oracle.homotopy import evaluate_homotopy_dt, evaluate_homotopy_rows  # noqa: E402
from synthetic import (config_system, homotopy_target, limbs_from_values, random_t, real_limbs,  # noqa: E402
                       system_from_terms)


@pytest.fixture(scope="module")
def phc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1109_0545_b200 as m
    return m


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _hom_eval(h, X, T, devices=None):
    F, J = h.eval_homotopy_batch(_cuda(X), _cuda(T), devices=devices)
    torch.cuda.synchronize()
    return F.cpu().numpy(), J.cpu().numpy()


@pytest.mark.parametrize("name,seed", [("tiny", 1), ("tiny", 2), ("c2", 1), ("c3", 1)])
def test_homotopy_vs_oracle(phc, name, seed):
    s, X = config_system(name, seed=seed, points=3)
    cf = homotopy_target(s, seed=100 + seed)
    T = random_t(3, s.limbs, seed=200 + seed)
    h = phc.System(s, coeff_target=cf)
    F, J = _hom_eval(h, X, T)
    arith = "exact" if s.limbs == 2 else "mp"
    for p in range(3):
        ar, Fr, Jr = evaluate_homotopy_rows(s, cf, X[p], T[p], arith=arith)
        ef, ej = compare_point(ar, Fr, Jr, F[p], J[p], s.limbs)
        assert ef <= TOL[s.limbs] and ej <= TOL[s.limbs], (p, ef, ej)
    assert limbs_normalised(F) and limbs_normalised(J)


@pytest.mark.parametrize("name", ["c2", "c3", "batch", "large"])
def test_t0_t1_equal_plain_evaluations(phc, name):
    """c(0) = c_s and c(1) = c_f exactly in the blend ((1 - t) and t are exactly 1 and 0),
    so the homotopy at t = 0 / 1 is bitwise the plain evaluation of the start / target system."""
    s, X = config_system(name, seed=3, points=2)
    cf = homotopy_target(s, seed=5)
    h = phc.System(s, coeff_target=cf)
    T = real_limbs([0, 1], s.limbs)
    F, J = _hom_eval(h, X, T)
    Fs, Js = phc.System(s).eval_batch(_cuda(X))
    Ft, Jt = phc.System(replace(s, coeff=cf)).eval_batch(_cuda(X))
    torch.cuda.synchronize()
    assert np.array_equal(F[0], Fs.cpu().numpy()[0]) and np.array_equal(J[0], Js.cpu().numpy()[0])
    assert np.array_equal(F[1], Ft.cpu().numpy()[1]) and np.array_equal(J[1], Jt.cpu().numpy()[1])


def test_plain_eval_unchanged_by_target(phc):
    """Attaching a target does not change the plain evaluation (start coefficients)."""
    s, X = config_system("c2", seed=2, points=2)
    a = phc.System(s)
    b = phc.System(s, coeff_target=homotopy_target(s, seed=1))
    Fa, Ja = a.eval_batch(_cuda(X))
    Fb, Jb = b.eval_batch(_cuda(X))
    torch.cuda.synchronize()
    assert torch.equal(Fa, Fb) and torch.equal(Ja, Jb)


@pytest.mark.parametrize("name", ["tiny", "c2", "c3"])
def test_old_t_as_variable_evaluator(phc, name):
    """The "old" evaluator (t as variable n+1) at (x, t): F and J[:, :n] equal the
    new evaluator's within tolerance, J[:, n] = dh/dt against the oracle."""
    s, X = config_system(name, seed=1, points=2)
    cf = homotopy_target(s, seed=11)
    T = random_t(2, s.limbs, seed=12)
    new = phc.System(s, coeff_target=cf)
    old = phc.System(s, coeff_target=cf, old_homotopy=True)
    assert old.n_var == s.n_var + 1
    F, J = _hom_eval(new, X, T)
    Xe = np.zeros((2, s.n_var + 1, 2, s.limbs))
    Xe[:, :s.n_var] = X
    Xe[:, s.n_var, 0, :] = T
    Fo, Jo = old.eval_batch(_cuda(Xe))
    torch.cuda.synchronize()
    Fo, Jo = Fo.cpu().numpy(), Jo.cpu().numpy()
    arith = "exact" if s.limbs == 2 else "mp"
    for p in range(2):
        ar, Fr, Jr = evaluate_homotopy_rows(s, cf, X[p], T[p], arith=arith)
        ef, ej = compare_point(ar, Fr, Jr, Fo[p], np.ascontiguousarray(Jo[p][:, :s.n_var]), s.limbs)
        assert ef <= TOL[s.limbs] and ej <= TOL[s.limbs], (p, ef, ej)
        ar, D = evaluate_homotopy_dt(s, cf, X[p], arith=arith)
        ed, _, _ = rel_errors(ar, D, Jo[p][:, s.n_var])
        assert ed <= TOL[s.limbs], ed


def test_homotopy_sharded_bitwise(phc):
    s, X = config_system("c2", seed=4, points=37)
    cf = homotopy_target(s, seed=3)
    T = random_t(37, 2, seed=4)
    h = phc.System(s, coeff_target=cf)
    F1, J1 = _hom_eval(h, X, T)
    F3, J3 = _hom_eval(h, X, T, devices=[0, 0, 0])
    assert np.array_equal(F1, F3) and np.array_equal(J1, J3)


def test_homotopy_large_sampled_rows(phc):
    """large (n = 256, k = 32, QD): the block path's layout 0 with the blend; mp512 rows."""
    s, X = config_system("large", seed=1, points=1)
    cf = homotopy_target(s, seed=2)
    T = random_t(1, 4, seed=3)
    h = phc.System(s, coeff_target=cf)
    F, J = _hom_eval(h, X, T)
    rows = [0, 200]
    ar, Fr, Jr = evaluate_homotopy_rows(s, cf, X[0], T[0], rows=rows, arith="mp")
    ef, ej = compare_point(ar, Fr, Jr, F[0], J[0], 4, rows)
    assert ef <= TOL[4] and ej <= TOL[4], (ef, ej)


def test_homotopy_generic_path(phc):
    """k > 32 runs the generic (three-kernel) path; its blend against the oracle."""
    rng = np.random.Generator(np.random.PCG64(5))
    n, m, k = 40, 3, 36
    polys = [[[(int(v), int(a)) for v, a in zip(sorted(rng.choice(n, k, replace=False)), rng.integers(1, 3, k))]
              for _ in range(m)] for _ in range(n)]
    s0, X = config_system("c3", seed=1, points=2)
    s = system_from_terms(n, n, 4, polys, s0.coeff[: n * m])
    cf = homotopy_target(s, seed=6)
    T = random_t(2, 4, seed=7)
    h = phc.System(s, coeff_target=cf)
    assert h.stats["path"] == 0
    F, J = _hom_eval(h, X, T)
    ar, Fr, Jr = evaluate_homotopy_rows(s, cf, X[1], T[1], rows=[0, 39], arith="mp")
    ef, ej = compare_point(ar, Fr, Jr, F[1], J[1], 4, [0, 39])
    assert ef <= TOL[4] and ej <= TOL[4], (ef, ej)


@pytest.mark.parametrize("L", [2, 4])
def test_newton_on_homotopy_spec_path(phc, L):
    """h = x^2 - (1+3t) (start x^2 - 1, target x^2 - 4).  Newton at
    t = 1/2 from x = 1.5 converges quadratically to sqrt(5/2); the residual reaches the
    precision's floor."""
    s = system_from_terms(1, 1, L, [[[(0, 2)], []]], limbs_from_values([1, -1], L))
    cf = limbs_from_values([1, -4], L)
    h = phc.System(s, coeff_target=cf)
    X = _cuda(limbs_from_values([1.5], L)[None])
    T = _cuda(real_limbs([0.5], L))
    res = []
    for _ in range(8):
        X, r, st = h.newton_step_homotopy(X, T)
        torch.cuda.synchronize()
        assert int(st[0]) == 0
        res.append(float(r[0]))
    x = X.cpu().numpy()[0, 0]
    import mpmath
    with mpmath.workprec(600):
        got = mpmath.fsum(mpmath.mpf(float(d)) for d in x[0])
        err = abs(got - mpmath.sqrt(mpmath.mpf(5) / 2))
    assert float(err) < (1e-30 if L == 2 else 1e-62), float(err)
    assert res[0] > 1e-3 and res[4] < 1e-20  # quadratic: 0.25 -> ~7e-3 -> ~5e-6 -> ~3e-12 -> ~6e-25
