"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Element-by-element comparison on seeded BASELINE.json configs (tiny, c2, c3 full;
batch and large on sampled points/rows at full size in the bench launch
configuration), special systems with exactly representable results (bitwise),
edge cases, metamorphic and determinism properties."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from _parity import TOL, compare_point, limbs_normalised, oracle_point  # noqa: E402
from oracle import ExactArith, evaluate_system, rel_errors  # noqa: E402
from synthetic import (config_system, limbs_from_values, special_gaussian_system,  # noqa: E402
                       special_linear_system, system_from_terms, random_system, homogeneous_system)


@pytest.fixture(scope="module")
def phc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1109_0545_b200 as m
    return m


def gpu_eval(phc, s, X, devices=None):
    h = phc.System(s, device=0)
    Xd = torch.from_numpy(np.ascontiguousarray(X)).cuda()
    if X.shape[0] == 1 and devices is None:
        f, j = h.eval(Xd[0])
        torch.cuda.synchronize()
        return f.cpu().numpy()[None], j.cpu().numpy()[None], h
    F, J = h.eval_batch(Xd, devices=devices)
    torch.cuda.synchronize()
    return F.cpu().numpy(), J.cpu().numpy(), h


@pytest.mark.parametrize("name,seed", [("tiny", 1), ("tiny", 2), ("tiny", 3), ("c2", 1), ("c2", 2), ("c2", 3),
                                       ("c3", 1), ("c3", 2)])
def test_config_full_exact(phc, name, seed):
    s, X = config_system(name, seed=seed)
    f, j, _ = gpu_eval(phc, s, X)
    ar, F, J = oracle_point(s, X[0], arith="exact")
    ef, ej = compare_point(ar, F, J, f[0], j[0], s.limbs)
    assert ef <= TOL[s.limbs] and ej <= TOL[s.limbs], (ef, ej)
    assert limbs_normalised(f) and limbs_normalised(j)
    # structural zeros are exact zeros
    nz = np.zeros((s.n_eq, s.n_var), bool)
    for i in range(s.n_eq):
        for _, fac in s.terms(i):
            for v, _a in fac:
                nz[i, v] = True
    assert (j[0][~nz] == 0).all()


def test_batch_config_sampled(phc):
    """batch: n=32, m=32, k=16, 65,536 points, DD; exact oracle on sampled points including
    the first and last point of every 8-way shard."""
    s, X = config_system("batch", seed=1)
    F, J, _ = gpu_eval(phc, s, X)
    P = X.shape[0]
    pts = sorted({0, P - 1, 12345, 40000} | {g * P // 8 for g in range(8)} | {(g + 1) * P // 8 - 1 for g in range(8)})
    for p in pts:
        ar, Fr, Jr = oracle_point(s, X[p], arith="exact")
        ef, ej = compare_point(ar, Fr, Jr, F[p], J[p], 2)
        assert ef <= TOL[2] and ej <= TOL[2], (p, ef, ej)


# The large config (configs[4]) is checked entry by entry against committed oracle values in
# tests/test_gpu_large.py (every F and J entry of the single point; 8 x 8 batch point-rows;
# batch point == single call for all 4,096 points).


@pytest.mark.parametrize("L", [2, 4])
def test_gaussian_integer_bitwise(phc, L):
    """P5: Z[i] coefficients, x in {±1, ±i}: exact result, GPU must match bitwise."""
    s, X = special_gaussian_system(12, 9, 5, 4, L, seed=7)
    f, j, _ = gpu_eval(phc, s, X)
    F, J = evaluate_system(s, X[0], "exact", workers=1)
    ar = ExactArith()
    from oracle import exact_equal_limbs
    assert exact_equal_limbs(ar, F, f[0])
    assert exact_equal_limbs(ar, [v for row in J for v in row], j[0].reshape(-1, 2, L))


@pytest.mark.parametrize("L", [2, 4])
def test_linear_system_J_is_C(phc, L):
    """P4: k = 1, a = 1 -> J equals the coefficient matrix bitwise."""
    s, X, C, x = special_linear_system(33, L, seed=2)
    f, j, _ = gpu_eval(phc, s, X)
    assert np.array_equal(j[0][:, :, :, 0], C.astype(np.float64))
    assert (j[0][:, :, :, 1:] == 0).all()
    Cc = C[:, :, 0] + 1j * C[:, :, 1]
    Fn = Cc @ (x[:, 0] + 1j * x[:, 1])
    assert np.array_equal(f[0][:, 0, 0], Fn.real) and np.array_equal(f[0][:, 1, 0], Fn.imag)


@pytest.mark.parametrize("L", [2, 4])
def test_edge_cases_mixed_k(phc, L):
    """Constant terms (k=0), k=1, duplicate terms, an empty polynomial, zero coordinates,
    a term in every variable, mixed k within a polynomial."""
    n = 9
    polys = [
        [[], [(0, 1)], [(0, 1)], [(1, 3), (4, 1)]],            # constant, duplicates
        [],                                                     # empty polynomial: F = 0, J row = 0
        [[(v, 1 + v % 3) for v in range(n)]],                   # every variable (k = n)
        [[(2, 2)], [(2, 2), (3, 1)], [(0, 1), (5, 7), (8, 2)]],  # mixed k
        [[(3, 1)], [(3, 2), (6, 1)]],                           # x_3 = 0 below
    ] + [[[(v, 2), ((v + 1) % n, 1)] if v + 1 < n else [(0, 1), (v, 2)]] for v in range(4)]
    T = sum(len(p) for p in polys)
    rng = np.random.default_rng(5)
    vals = [complex(a, b) for a, b in rng.uniform(-1, 1, (T, 2))]
    coeff = limbs_from_values(vals, L)
    s = system_from_terms(len(polys), n, L, polys, coeff)
    xv = [complex(a, b) for a, b in rng.uniform(-1, 1, (n, 2))]
    xv[3] = 0
    X = limbs_from_values(xv, L)[None]
    f, j, _ = gpu_eval(phc, s, X)
    ar, F, J = oracle_point(s, X[0], arith="exact")
    ef, ej = compare_point(ar, F, J, f[0], j[0], L)
    assert ef <= TOL[L] and ej <= TOL[L], (ef, ej)
    assert (f[0][1] == 0).all() and (j[0][1] == 0).all()


@pytest.mark.parametrize("L", [2, 4])
def test_ragged_and_many_points(phc, L):
    """A ragged system (k varying 0..12, m not a multiple of 32) over 37 points."""
    rng = np.random.default_rng(11)
    n = 23
    polys = []
    for i in range(n):
        terms = []
        for t in range(int(rng.integers(1, 45))):
            k = int(rng.integers(0, 13))
            vs = sorted(rng.choice(n, k, replace=False).tolist())
            terms.append([(v, int(rng.integers(1, 6))) for v in vs])
        polys.append(terms)
    T = sum(len(p) for p in polys)
    s0, _ = random_system(2, 1, 1, 1, L, seed=1)  # unit-circle helpers
    from synthetic.systems import unit_circle_limbs
    coeff = unit_circle_limbs(rng.uniform(0, 6.283, T), L, 1)
    s = system_from_terms(n, n, L, polys, coeff)
    X = unit_circle_limbs(rng.uniform(0, 6.283, (37, n)), L, 1)
    F, J, h = gpu_eval(phc, s, X)
    for p in (0, 17, 36):
        ar, Fr, Jr = oracle_point(s, X[p], arith="exact")
        ef, ej = compare_point(ar, Fr, Jr, F[p], J[p], L)
        assert ef <= TOL[L] and ej <= TOL[L], (p, ef, ej)
        # the same point alone takes the latency path (one warp per term)
        f1, j1 = h.eval(torch.from_numpy(X[p]).cuda())
        torch.cuda.synchronize()
        ef, ej = compare_point(ar, Fr, Jr, f1.cpu().numpy(), j1.cpu().numpy(), L)
        assert ef <= TOL[L] and ej <= TOL[L], (p, "latency", ef, ej)


def test_euler_identity_full_batch(phc):
    """P8 at size: homogeneous system over 2,048 points, sum_v x_v J_iv = d_i f_i checked in
    float64 on every point (a property that needs no oracle)."""
    s, X, degs = homogeneous_system(24, 20, 6, 9, 2, seed=9, points=2048)
    F, J, _ = gpu_eval(phc, s, X)
    f = F[:, :, 0, 0] + 1j * F[:, :, 1, 0]
    jj = J[..., 0, 0] + 1j * J[..., 1, 0]
    x = X[..., 0, 0] + 1j * X[..., 1, 0]
    lhs = np.einsum("piv,pv->pi", jj, x)
    rhs = f * np.asarray(degs)[None, :]
    assert np.max(np.abs(lhs - rhs)) <= 1e-12 * np.max(np.abs(rhs))


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_conjugation_and_scaling_bitwise(phc, name):
    """P9: conj(inputs) -> conj(outputs) bitwise; coefficients * 2^s -> outputs * 2^s bitwise."""
    s, X = config_system(name, seed=2, points=64)
    F, J, _ = gpu_eval(phc, s, X)
    sc = s.__class__(**{**s.__dict__})
    sc.coeff = s.coeff.copy()
    sc.coeff[:, 1, :] *= -1
    Xc = X.copy()
    Xc[:, :, 1, :] *= -1
    Fc, Jc, _ = gpu_eval(phc, sc, Xc)
    assert np.array_equal(Fc[:, :, 0], F[:, :, 0]) and np.array_equal(Fc[:, :, 1], -F[:, :, 1])
    assert np.array_equal(Jc[..., 0, :], J[..., 0, :]) and np.array_equal(Jc[..., 1, :], -J[..., 1, :])
    ss = s.__class__(**{**s.__dict__})
    ss.coeff = s.coeff * 2.0 ** -7
    Fs, Js, _ = gpu_eval(phc, ss, X)
    assert np.array_equal(Fs, F * 2.0 ** -7) and np.array_equal(Js, J * 2.0 ** -7)


def test_determinism_and_device_lists(phc):
    """P10: repeated runs and device lists with repeats are bitwise equal; host API equals device API."""
    s, X = config_system("batch", seed=3, points=1000)
    F1, J1, h = gpu_eval(phc, s, X)
    F2, J2, _ = gpu_eval(phc, s, X, devices=[0, 0, 0])
    F3, J3, _ = gpu_eval(phc, s, X, devices=[0, 0, 0, 0, 0, 0, 0, 0])
    assert np.array_equal(F1, F2) and np.array_equal(J1, J2)
    assert np.array_equal(F1, F3) and np.array_equal(J1, J3)
    Fh, Jh = h.eval_batch_host(np.ascontiguousarray(X))
    assert np.array_equal(F1, Fh) and np.array_equal(J1, Jh)
    # a single-point call takes the latency path (one warp per term, warp scans; DESIGN.md
    # reading N2-2): deterministic, equal to the batch kernel within the tolerance
    Xd = torch.from_numpy(X[513]).cuda()
    f, j = h.eval(Xd)
    f2, j2 = h.eval(Xd)
    torch.cuda.synchronize()
    assert torch.equal(f, f2) and torch.equal(j, j2)
    assert _limb_rel_diff(F1[513], f.cpu().numpy()) <= TOL[2] and _limb_rel_diff(J1[513], j.cpu().numpy()) <= TOL[2]


def _limb_rel_diff(a, b):
    """max |a - b| / max |a| over entries, from the exact limb sums (Fractions)."""
    from fractions import Fraction
    a = np.asarray(a).reshape(-1, a.shape[-1])
    b = np.asarray(b).reshape(-1, b.shape[-1])
    ex = lambda r: sum(Fraction(float(d)) for d in r)  # noqa: E731
    num = max(abs(ex(x) - ex(y)) for x, y in zip(a, b))
    den = max(abs(ex(x)) for x in a)
    return float(num / den) if den else float(num)


@pytest.mark.parametrize("name", ["tiny", "c2", "c3", "batch"])
def test_latency_path_vs_batch_path(phc, name):
    """The same point through the latency path (1 point) and the batch kernel (many points):
    both within tolerance of the exact oracle (checked above per config) and of each other."""
    s, X = config_system(name, seed=5, points=400 if name != "c3" else 8)
    F, J, h = gpu_eval(phc, s, X)
    for p in (0, X.shape[0] - 1):
        f, j = h.eval(torch.from_numpy(X[p]).cuda())
        torch.cuda.synchronize()
        assert _limb_rel_diff(F[p], f.cpu().numpy()) <= TOL[s.limbs]
        assert _limb_rel_diff(J[p], j.cpu().numpy()) <= TOL[s.limbs]
        assert limbs_normalised(f.cpu().numpy()) and limbs_normalised(j.cpu().numpy())


def test_host_pipeline_equals_device_call(phc):
    """phc_eval_jacobian_batch_host pipelines chunks of ~128 MiB of output (output copies
    overlapping the next chunk's evaluation; 2 chunks here): bitwise the device call's results."""
    s, X = config_system("batch", seed=6, points=8200)
    F, J, h = gpu_eval(phc, s, X)
    Fh = torch.empty((X.shape[0], s.n_eq, 2, 2), dtype=torch.float64).pin_memory()
    Jh = torch.empty((X.shape[0], s.n_eq, s.n_var, 2, 2), dtype=torch.float64).pin_memory()
    Xh = torch.from_numpy(X).pin_memory()
    h.eval_batch_host(Xh.numpy(), Fh.numpy(), Jh.numpy())
    assert np.array_equal(F, Fh.numpy()) and np.array_equal(J, Jh.numpy())


@pytest.mark.parametrize("L", [2, 4])
def test_compiled_maxima(phc, L):
    """The compiled limits of include/phc.h: a term with k = PHC_MAX_K = 64 factors (generic
    path), an exponent of PHC_MAX_EXP = 255, and n_var = PHC_MAX_VARS = 65534 (a sparse
    system touching the last variable); against the mp512 oracle."""
    from synthetic.systems import unit_circle_limbs
    rng = np.random.default_rng(21)
    n = 64
    polys = [[[(v, int(rng.integers(1, 4))) for v in range(n)], [(5, 255)]],
             [[(0, 255), (63, 1)], []],
             [[(v, 1) for v in range(0, n, 2)]]]
    T = sum(len(p) for p in polys)
    coeff = unit_circle_limbs(rng.uniform(0, 6.283, T), L, 1)
    s = system_from_terms(3, n, L, polys, coeff)
    X = unit_circle_limbs(rng.uniform(0, 6.283, (1, n)), L, 1)
    f, j, h = gpu_eval(phc, s, X)
    assert h.stats["kmax"] == 64 and h.stats["D"] == 255 and h.stats["path"] == 0
    ar, F, J = oracle_point(s, X[0], arith="mp")
    ef, ej = compare_point(ar, F, J, f[0], j[0], L)
    assert ef <= TOL[L] and ej <= TOL[L], (ef, ej)
    # n_var at the limit, two sparse polynomials
    nv = 65534
    polys = [[[(0, 2), (nv - 1, 3)], [(nv // 2, 1)]], [[(nv - 1, 1)], []]]
    coeff = unit_circle_limbs(rng.uniform(0, 6.283, 4), L, 1)
    s2 = system_from_terms(2, nv, L, polys, coeff)
    X2 = np.zeros((1, nv, 2, L))
    X2[0, :, 0, 0] = 1.0
    X2[0, [0, nv // 2, nv - 1]] = unit_circle_limbs(rng.uniform(0, 6.283, 3), L, 1)
    f2, j2, _ = gpu_eval(phc, s2, X2)
    ar, F2, J2 = oracle_point(s2, X2[0], arith="mp")
    cols = [0, nv // 2, nv - 1, 1, 77]
    ef = rel_errors(ar, F2, f2[0])[0]
    ej = rel_errors(ar, [J2[i][c] for i in range(2) for c in cols], np.stack([j2[0][i, c] for i in range(2) for c in cols]))[0]
    assert ef <= TOL[L] and ej <= TOL[L], (ef, ej)
    assert np.count_nonzero(j2[0][..., 0, 0]) == 4


@pytest.mark.parametrize("L", [2, 4])
def test_empty_inputs(phc, L):
    """Zero points: every batch call is a no-op returning PHC_OK; a system without any term
    (n_terms = 0): F = 0 and J = 0 exactly, through the latency path and the batch kernels."""
    s, X = config_system("tiny" if L == 2 else "c3", seed=1, points=1)
    h = phc.System(s)
    X0 = torch.empty((0, s.n_var, 2, L), dtype=torch.float64, device="cuda")
    F0, J0 = h.eval_batch(X0)
    Xn, r, st = h.newton_step(X0)
    torch.cuda.synchronize()
    assert F0.shape[0] == 0 and J0.shape[0] == 0 and Xn.shape[0] == 0
    empty = system_from_terms(3, 4, L, [[], [], []], np.zeros((0, 2, L)))
    he = phc.System(empty)
    Xe = torch.from_numpy(np.ones((5000, 4, 2, L))).cuda()
    for pts in (1, 5000):
        F, J = he.eval_batch(Xe[:pts])
        torch.cuda.synchronize()
        assert (F == 0).all() and (J == 0).all()


def test_generic_path_beyond_65535_points(phc):
    """The generic path (k > 32) puts the point on gridDim.y: calls with more than 65,535
    points are chunked (point 70,000 checked against the exact oracle)."""
    from synthetic.systems import unit_circle_limbs
    rng = np.random.default_rng(9)
    n = 34
    polys = [[[(v, 1) for v in range(33)]], [[(0, 2), (33, 1)], []]]
    coeff = unit_circle_limbs(rng.uniform(0, 6.283, 3), 2, 1)
    s = system_from_terms(2, n, 2, polys, coeff)
    P = 70001
    X = unit_circle_limbs(rng.uniform(0, 6.283, (P, n)), 2, 8)
    F, J, h = gpu_eval(phc, s, X)
    assert h.stats["path"] == 0
    for p in (0, 65535, 70000):
        ar, Fr, Jr = oracle_point(s, X[p], arith="exact")
        ef, ej = compare_point(ar, Fr, Jr, F[p], J[p], 2)
        assert ef <= TOL[2] and ej <= TOL[2], (p, ef, ej)


@pytest.mark.parametrize("mode", ["staged", "fused"])
def test_remote_shard_branches_on_one_gpu(phc, mode, monkeypatch):
    """PHC_DEBUG_REMOTE sends the home device's shards through the remote-device branches of
    phc_eval_jacobian_batch (staged: peer copies of chunked shards on a second stream, with a
    device listed several times; fused: kernels storing into the home buffers): bitwise the
    unsharded results, plain and homotopy."""
    from synthetic import homotopy_target, random_t
    s, X = config_system("batch", seed=8, points=3 * 8200)
    cf = homotopy_target(s, seed=9)
    T = random_t(X.shape[0], 2, seed=10)
    h = phc.System(s, coeff_target=cf)
    Xd, Td = torch.from_numpy(X).cuda(), torch.from_numpy(T).cuda()
    F1, J1 = h.eval_batch(Xd)
    H1, K1 = h.eval_homotopy_batch(Xd, Td)
    torch.cuda.synchronize()
    monkeypatch.setenv("PHC_DEBUG_REMOTE", mode)
    F2, J2 = h.eval_batch(Xd, devices=[0, 0, 0])
    H2, K2 = h.eval_homotopy_batch(Xd, Td, devices=[0, 0, 0])
    torch.cuda.synchronize()
    assert torch.equal(F1, F2) and torch.equal(J1, J2)
    assert torch.equal(H1, H2) and torch.equal(K1, K2)


def _quadratic_system(n, terms_per_poly, seed, hub=False):
    """k <= 2 DD system: every polynomial has `terms_per_poly` random monomials of degree <= 2
    (hub: every term of polynomial i contains x_0, so a block cannot spread (class, x_0) over
    2 lanes per class and the planner must keep K = 4)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    polys = []
    for _ in range(n):
        terms = []
        for _t in range(terms_per_poly):
            if hub:
                b = int(rng.integers(1, n))
                terms.append([(0, 1), (b, int(rng.integers(1, 3)))])
            else:
                k = int(rng.integers(0, 3))
                vs = sorted(rng.choice(n, size=k, replace=False).tolist())
                terms.append([(v, int(rng.integers(1, 3))) for v in vs])
        polys.append(terms)
    T = n * terms_per_poly
    vals = np.exp(2j * np.pi * rng.random(T)) * rng.uniform(0.5, 2.0, T)
    s = system_from_terms(n, n, 2, polys, limbs_from_values(vals, 2))
    X = np.stack([limbs_from_values(np.exp(2j * np.pi * rng.random(n)), 2) for _ in range(3)])
    return s, X


@pytest.mark.parametrize("hub,K", [(False, 2), (True, 4)])
def test_low_degree_lane_placement(phc, hub, K):
    """k <= 2 systems: the planner places each block's terms on lanes so that no (class, var)
    accumulator is shared by more than two lanes and colours with K = 2 slots; a system whose
    blocks cannot be balanced (one variable in every term) keeps K = 4.  Both match the exact
    oracle (3 points, batch kernel), structural zeros exact."""
    s, X = _quadratic_system(12, 70, seed=5 if not hub else 6, hub=hub)
    F, J, h = gpu_eval(phc, s, X, devices=[0])
    st = h.stats
    assert st["layout"] == 2 and st["K"] == K, st
    for p in range(X.shape[0]):
        ar, Fo, Jo = oracle_point(s, X[p], arith="exact")
        ef, ej = compare_point(ar, Fo, Jo, F[p], J[p], 2)
        assert ef <= TOL[2] and ej <= TOL[2], (p, ef, ej)
