"""GPU parity for NEXT-4: the predictor kernel (phc_predict_batch, §5)
against the Lagrange oracle, bitwise on exactly representable quadratic paths; the path
tracker (phc_track_paths, Alg. 1) on SPEC's analytic path and on a total-degree
homotopy whose end points are checked by the exact oracle."""
from fractions import Fraction as Fr

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import ExactArith, evaluate_system  # noqa: E402
from oracle.predictor import predict_point  # noqa: E402
from synthetic import limbs_from_values, real_limbs, system_from_terms, total_degree_homotopy  # noqa: E402


@pytest.fixture(scope="module")
def phc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1109_0545_b200 as m
    return m


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def _mp(limbs):
    return sum(Fr(float(d)) for d in limbs)


@pytest.mark.parametrize("L", [2, 4])
def test_predictor_vs_oracle(phc, L):
    rng = np.random.Generator(np.random.PCG64(10 + L))
    P, n = 48, 5
    nh = rng.integers(1, 4, P).astype(np.int32)
    t0 = rng.uniform(0.2, 0.9, P)
    gaps = rng.uniform(0.001, 0.05, (P, 2))
    th = np.zeros((P, 3, L))
    xh = np.zeros((P, 3, n, 2, L))
    tn = np.zeros((P, L))
    for p in range(P):
        ts = [Fr(t0[p]), Fr(t0[p]) - Fr(gaps[p, 0]), Fr(t0[p]) - Fr(gaps[p, 0]) - Fr(gaps[p, 1])]
        th[p] = real_limbs(ts, L)
        tn[p] = real_limbs([Fr(t0[p]) + Fr(float(rng.uniform(0.001, 0.05)))], L)[0]
        vals = rng.uniform(-1, 1, (3, n, 2))
        for s in range(3):
            xh[p, s] = limbs_from_values([complex(*v) for v in vals[s]], L)
    tol = 1e-27 if L == 2 else 1e-59
    for order in (0, 1, 2):
        out = phc.predict_batch(order, _cuda(nh), _cuda(th), _cuda(xh), _cuda(tn)).cpu().numpy()
        for p in range(P):
            h = min(int(nh[p]), order + 1)
            ref = predict_point(th[p], xh[p], h, tn[p])
            for i in range(n):
                d = abs(complex(float(_mp(out[p, i, 0]) - ref[i][0]), float(_mp(out[p, i, 1]) - ref[i][1])))
                assert d <= tol * max(1.0, abs(complex(float(ref[i][0]), float(ref[i][1])))), (order, p, i, d)


@pytest.mark.parametrize("L", [2, 4])
def test_predictor_exact_on_dyadic_parabola(phc, L):
    """x(t) = a + b t + c t^2 with dyadic a, b, c and t in {1/2, 1/4, 0} -> 3/4: every step is
    exact, so the quadratic prediction is bitwise x(3/4)."""
    a, b, c = complex(0.75, -1.5), complex(2.0, 0.25), complex(-3.0, 1.0)
    ts = [0.5, 0.25, 0.0]
    x = lambda t: a + b * t + c * t * t  # noqa: E731
    th = real_limbs(ts, L)[None]
    xh = np.stack([limbs_from_values([x(t), 2 * x(t)], L) for t in ts])[None]
    out = phc.predict_batch(2, _cuda(np.array([3], np.int32)), _cuda(th), _cuda(xh),
                            _cuda(real_limbs([0.75], L))).cpu().numpy()
    want = limbs_from_values([x(0.75), 2 * x(0.75)], L)
    assert np.array_equal(out[0], want)


@pytest.mark.parametrize("L", [2, 4])
def test_track_spec_analytic_path(phc, L):
    """h = x^2 - (1+3t) from z0 = 1 reaches z = 2 (analytic path sqrt(1+3t))."""
    s = system_from_terms(1, 1, L, [[[(0, 2)], []]], limbs_from_values([1, -1], L))
    h = phc.System(s, coeff_target=limbs_from_values([1, -4], L))
    X0 = _cuda(limbs_from_values([1.0], L)[None])
    Xe, status, stats = h.track(X0)
    assert status[0] == 1, stats
    z = Xe.cpu().numpy()[0, 0]
    err = abs(_mp(z[0]) - 2) + abs(_mp(z[1]))
    assert float(err) <= (1e-30 if L == 2 else 1e-62), float(err)
    assert stats[0, 0] >= 10 and stats[0, 3] > 0


def test_track_total_degree_homotopy(phc):
    """n = 3 quadratic target system, total-degree start system gamma (x_i^2 - 1): the 8 paths
    all arrive; the exact oracle evaluates the target system at each end point (residual at
    the precision floor) and the 8 end points are distinct (a generic system has 8 roots)."""
    s, cf, X0 = total_degree_homotopy(3, 2, seed=7)
    h = phc.System(s, coeff_target=cf)
    Xe, status, stats = h.track(_cuda(X0))
    assert (status == 1).all(), (status, stats)
    ends = Xe.cpu().numpy()
    from dataclasses import replace
    target = replace(s, coeff=cf)
    ar = ExactArith()
    for p in range(8):
        F, _ = evaluate_system(target, ends[p], arith="exact", workers=1)
        res = max(float(abs(ar.to_mpc(f, 300))) for f in F)
        assert res <= 1e-26, (p, res)
    z = ends[:, :, 0, 0] + 1j * ends[:, :, 1, 0]
    d = min(np.linalg.norm(z[a] - z[b]) for a in range(8) for b in range(a))
    assert d > 1e-6, d


def test_track_quadratic_needs_no_more_steps_than_secant(phc):
    """§5: the quadratic predictor brings a gain in the number of corrections over the
    secant predictor (here: total predictor-corrector steps over the 8 paths, same settings)."""
    s, cf, X0 = total_degree_homotopy(3, 2, seed=7)
    h = phc.System(s, coeff_target=cf)
    _, st2, stats2 = h.track(_cuda(X0), predictor=2)
    _, st1, stats1 = h.track(_cuda(X0), predictor=1)
    assert (st2 == 1).all() and (st1 == 1).all()
    assert stats2[:, 1].sum() <= stats1[:, 1].sum(), (stats2[:, 1].sum(), stats1[:, 1].sum())


def test_track_rejects_bad_parameters(phc):
    s = system_from_terms(1, 1, 2, [[[(0, 2)], []]], limbs_from_values([1, -1], 2))
    h = phc.System(s, coeff_target=limbs_from_values([1, -4], 2))
    with pytest.raises(phc.PhcError):
        h.track(_cuda(limbs_from_values([1.0], 2)[None]), step_init=2.0)
    plain = phc.System(s)
    with pytest.raises(phc.PhcError):
        plain.track(_cuda(limbs_from_values([1.0], 2)[None]))


def test_track_window_changes_no_decision(phc, monkeypatch):
    """The device-side step control runs W steps between host checks (phc_track_paths); a
    path that stops inside a window is frozen by the control kernel, so every window size
    gives bitwise the same end points, statuses and per-path statistics as W = 1."""
    s, cf, X0 = total_degree_homotopy(4, 2, seed=3)
    h = phc.System(s, coeff_target=cf)
    out = {}
    for w in (1, 3, 8, 64):
        monkeypatch.setenv("PHC_TRACK_WINDOW", str(w))
        Xe, status, stats, te = h.track(_cuda(X0), t_end=True)
        out[w] = (Xe.cpu().numpy(), status, stats, te.cpu().numpy())
    for w in (3, 8, 64):
        for a, b in zip(out[1], out[w]):
            assert np.array_equal(a, b), w
    assert (out[1][1] == 1).all()


def test_track_max_steps_inside_window(phc, monkeypatch):
    """max_steps smaller than the window: every path stops at exactly max_steps steps."""
    s, cf, X0 = total_degree_homotopy(3, 2, seed=7)
    h = phc.System(s, coeff_target=cf)
    monkeypatch.setenv("PHC_TRACK_WINDOW", "16")
    _, status, stats = h.track(_cuda(X0), max_steps=5)
    assert (status == 2).all() and (stats[:, 1] == 5).all(), (status, stats[:, 1])


def test_track_graph_equals_plain_launches(phc, monkeypatch):
    """Windows replayed as CUDA graphs (re-captured or updated whenever the number of active
    paths changes) give bitwise the results of plain launches (PHC_TRACK_GRAPH=0)."""
    s, cf, X0 = total_degree_homotopy(4, 2, seed=11)
    h = phc.System(s, coeff_target=cf)
    out = {}
    for g in ("0", "1"):
        monkeypatch.setenv("PHC_TRACK_GRAPH", g)
        Xe, status, stats, te = h.track(_cuda(X0), t_end=True)
        out[g] = (Xe.cpu().numpy(), status, stats, te.cpu().numpy())
    for a, b in zip(out["0"], out["1"]):
        assert np.array_equal(a, b)
    assert (out["1"][1] == 1).all()
    assert len(set(out["1"][2][:, 1].tolist())) > 1  # paths stop at different steps: A changes


def test_track_graph_fallback_when_regime_changes(phc, monkeypatch):
    """A k = 12 monomial in every polynomial makes few-path corrector calls take the latency
    path, whose workspace is first allocated when the active paths drop -- inside a window
    capture.  The tracker must fall back to plain launches there and still give bitwise the
    results of a run without graphs."""
    n, L = 12, 2
    s, cf, X0 = total_degree_homotopy(n, L, seed=13)
    big = [(v, 1) for v in range(n)]
    polys = [[list(fac) for _, fac in s.terms(i)] + [big] for i in range(n)]
    M = len(polys[0]) - 1
    start = np.zeros((n * (M + 1), 2, L))
    target = np.zeros((n * (M + 1), 2, L))
    for i in range(n):
        start[i * (M + 1):i * (M + 1) + M] = s.coeff[i * M:(i + 1) * M]
        target[i * (M + 1):i * (M + 1) + M] = cf[i * M:(i + 1) * M]
        target[i * (M + 1) + M, 0, 0] = 1e-3  # small k = 12 term in the target only
    s2 = system_from_terms(n, n, L, polys, start)
    h = phc.System(s2, coeff_target=target)
    assert h.stats["kmax"] == 12
    X = _cuda(X0[[0, 5, 17, 99, 1000, 2047, 3000, 4095]])
    out = {}
    for g in ("0", "1"):
        monkeypatch.setenv("PHC_TRACK_GRAPH", g)
        Xe, status, stats = h.track(X.clone(), max_steps=3000)
        out[g] = (Xe.cpu().numpy(), status, stats)
    for a, b in zip(out["0"], out["1"]):
        assert np.array_equal(a, b)
