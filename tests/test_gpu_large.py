"""GPU parity at the largest config (BASELINE.json configs[4] "large": n = m = 256, k = 32,
D = 8, complex QD) and full-batch properties (SURVEY.md §8(c) coverage plan):

* the single point: EVERY entry of F and J (256 x 257 complex QD values) against the committed
  mp512 oracle values (tests/golden/large_seed1.npz, tools/make_golden_large.py), normwise
  <= 1e-60 (reading C9), structural zeros exact;
* the 4,096-point batch: 8 points x 8 rows against the golden values, and every batch point
  bitwise equal to the single-point call at that point (P10);
* P9 (conjugation, 2^s coefficient scaling: bitwise) on large x 64 points and on the full
  65,536-point batch-DD config; P10 on the full batch (device lists, range shards)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from _golden import load, to_mpc  # noqa: E402
from _parity import TOL, limbs_normalised  # noqa: E402
from oracle import MPArith, rel_errors  # noqa: E402
from synthetic import config_system  # noqa: E402


@pytest.fixture(scope="module")
def phc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1109_0545_b200 as m
    return m


@pytest.fixture(scope="module")
def golden():
    return load()


@pytest.fixture(scope="module")
def large_batch(phc):
    s, X = config_system("large_batch", seed=1)
    h = phc.System(s, device=0)
    Xd = torch.from_numpy(X).cuda()
    F, J = h.eval_batch(Xd)
    torch.cuda.synchronize()
    return s, X, h, Xd, F, J


def _nz(s):
    nz = np.zeros((s.n_eq, s.n_var), bool)
    for i in range(s.n_eq):
        for _, fac in s.terms(i):
            for v, _a in fac:
                nz[i, v] = True
    return nz


def test_large_single_point_every_entry(phc, golden):
    """phc_eval_jacobian at point 0: all 256 F values and all 65,536 J entries vs the oracle."""
    s, X = config_system("large", seed=1)
    h = phc.System(s, device=0)
    f, j = h.eval(torch.from_numpy(X[0]).cuda())
    torch.cuda.synchronize()
    f, j = f.cpu().numpy(), j.cpu().numpy()
    ar = MPArith(512)
    ef, _, _ = rel_errors(ar, to_mpc(golden["F0"]), f)
    ej, _, _ = rel_errors(ar, to_mpc(golden["J0"]), j.reshape(-1, 2, 4))
    assert ef <= TOL[4] and ej <= TOL[4], (ef, ej)
    assert limbs_normalised(f) and limbs_normalised(j)
    assert (j[~_nz(s)] == 0).all()
    # every row on its own too (a bad row cannot hide in the norm of the others)
    Fm, Jm = to_mpc(golden["F0"]), to_mpc(golden["J0"])
    for i in range(0, 256, 17):
        e, _, _ = rel_errors(ar, Jm[i * 256:(i + 1) * 256], j[i])
        assert e <= TOL[4], (i, e)


def test_large_batch_sampled_points_vs_golden(golden, large_batch):
    """large x 4,096 (one batch call, the bench configuration): 8 points x 8 rows vs the oracle."""
    s, X, h, Xd, F, J = large_batch
    ar = MPArith(512)
    for q, p in enumerate(golden["batch_points"]):
        rows = [int(r) for r in golden["batch_rows"][q]]
        fg = F[int(p)].cpu().numpy()[rows]
        jg = J[int(p)].cpu().numpy()[rows]
        ef, _, _ = rel_errors(ar, to_mpc(golden["Fb"][q]), fg)
        ej, _, _ = rel_errors(ar, to_mpc(golden["Jb"][q]), jg.reshape(-1, 2, 4))
        assert ef <= TOL[4] and ej <= TOL[4], (int(p), ef, ej)


def test_large_batch_points_equal_single_calls(large_batch):
    """P10: every one of the 4,096 batch points equals the single-point call at that point
    bitwise (both take the fused block kernel: 65,536 terms exceed the latency-path bound)."""
    s, X, h, Xd, F, J = large_batch
    f = torch.empty((s.n_eq, 2, 4), dtype=torch.float64, device="cuda")
    j = torch.empty((s.n_eq, s.n_var, 2, 4), dtype=torch.float64, device="cuda")
    bad = torch.zeros((), dtype=torch.int64, device="cuda")
    for p in range(X.shape[0]):
        h.eval(Xd[p], f, j)
        bad += (f != F[p]).sum() + (j != J[p]).sum()
    torch.cuda.synchronize()
    assert int(bad) == 0


def _conj_scale_check(phc, s, Xd, F, J, scale_exp):
    """P9 on the device: conj(inputs) -> conj(outputs) and coeff * 2^s -> outputs * 2^s, bitwise."""
    sc = s.__class__(**{**s.__dict__})
    sc.coeff = s.coeff.copy()
    sc.coeff[:, 1, :] *= -1
    Xc = Xd.clone()
    Xc[:, :, 1, :] *= -1
    hc = phc.System(sc, device=0)
    Fc, Jc = hc.eval_batch(Xc)
    torch.cuda.synchronize()
    assert torch.equal(Fc[:, :, 0], F[:, :, 0]) and torch.equal(Fc[:, :, 1], -F[:, :, 1])
    assert torch.equal(Jc[..., 0, :], J[..., 0, :]) and torch.equal(Jc[..., 1, :], -J[..., 1, :])
    del Fc, Jc, hc
    ss = s.__class__(**{**s.__dict__})
    ss.coeff = s.coeff * 2.0 ** scale_exp
    hs = phc.System(ss, device=0)
    Fs, Js = hs.eval_batch(Xd)
    torch.cuda.synchronize()
    assert torch.equal(Fs, F * 2.0 ** scale_exp) and torch.equal(Js, J * 2.0 ** scale_exp)


def test_large_conjugation_and_scaling_bitwise(phc, large_batch):
    """P9 on the large config, 64 points of the batch (the bench's kernel)."""
    s, X, h, Xd, F, J = large_batch
    Xs = Xd[:64].contiguous()
    Fs, Js = h.eval_batch(Xs)
    torch.cuda.synchronize()
    # the 64-point call takes the same kernel as the 4,096-point one: same bits
    assert torch.equal(Fs, F[:64]) and torch.equal(Js, J[:64])
    _conj_scale_check(phc, s, Xs, Fs, Js, -11)


def test_full_batch_dd_conjugation_scaling_and_shardings(phc):
    """BASELINE.json configs[3] at full size (65,536 points, DD): P9 bitwise over every point;
    P10: an 8-way device list (one GPU repeated) and 8 range shards (the per-process call of
    a multi-GPU run, phc_eval_jacobian_batch_range) give the unsharded result bitwise."""
    s, X = config_system("batch", seed=1)
    h = phc.System(s, device=0)
    Xd = torch.from_numpy(X).cuda()
    F, J = h.eval_batch(Xd)
    torch.cuda.synchronize()
    assert bool(torch.isfinite(F).all()) and bool(torch.isfinite(J).all())
    _conj_scale_check(phc, s, Xd, F, J, 9)
    F8, J8 = h.eval_batch(Xd, devices=[0] * 8)
    torch.cuda.synchronize()
    assert torch.equal(F8, F) and torch.equal(J8, J)
    del F8, J8
    Fr = torch.full_like(F, float("nan"))
    Jr = torch.full_like(J, float("nan"))
    P = X.shape[0]
    for r in range(8):
        h.eval_batch_range(Xd, r * P // 8, (r + 1) * P // 8, Fr, Jr)
    torch.cuda.synchronize()
    assert torch.equal(Fr, F) and torch.equal(Jr, J)


def test_range_call_keeps_the_regime_of_the_whole_call(phc):
    """A shard of a call small enough for the latency path on its own is still evaluated in the
    regime of the whole call (phc.h determinism): 1,000 c3 points in 4 shards of 250."""
    s, X = config_system("c3", seed=3, points=1000)
    h = phc.System(s, device=0)
    Xd = torch.from_numpy(X).cuda()
    F, J = h.eval_batch(Xd)
    Fr, Jr = torch.zeros_like(F), torch.zeros_like(J)
    for a, b in ((0, 1), (1, 250), (250, 999), (999, 1000)):
        h.eval_batch_range(Xd, a, b, Fr, Jr)
    torch.cuda.synchronize()
    assert torch.equal(Fr, F) and torch.equal(Jr, J)
    with pytest.raises(phc.PhcError):
        h.eval_batch_range(Xd, 10, 5, Fr, Jr)
    with pytest.raises(phc.PhcError):
        h.eval_batch_range(Xd, 0, 1001, Fr, Jr)


def test_large_newton_step_vs_oracle(phc, golden):
    """NEXT-1 at the largest config (n = 256, QD, single point: the cooperative global-memory
    elimination): the GPU's step dz = x_new - x against the oracle's (golden newton_dz0:
    mpmath.lu_solve at 512 bits on the oracle's F and J), within the error budget
    64 n u cond(J) of a backward-stable elimination; the residual max_i |F_i| as the oracle's."""
    import mpmath
    from fractions import Fraction
    if "newton_dz0" not in golden:
        pytest.skip("golden file without the Newton step (tools/make_golden_large.py --add-newton)")
    s, X = config_system("large", seed=1)
    h = phc.System(s, device=0)
    Xd = torch.from_numpy(X).cuda()
    Xn, res, status = h.newton_step(Xd)
    F, J = h.eval_batch(Xd)
    torch.cuda.synchronize()
    assert int(status[0]) == 0
    assert float(res[0]) == pytest.approx(float(golden["newton_residual0"]), rel=1e-12)
    xn = Xn.cpu().numpy()[0]
    ref = to_mpc(golden["newton_dz0"])
    ex = lambda r: sum(Fraction(float(d)) for d in r)  # noqa: E731

    def mpq(fr):
        return mpmath.mpf(fr.numerator) / fr.denominator

    with mpmath.workprec(1100):
        got = [mpmath.mpc(mpq(ex(xn[v, 0]) - ex(X[0, v, 0])), mpq(ex(xn[v, 1]) - ex(X[0, v, 1])))
               for v in range(s.n_var)]
        num = max(abs(a - b) for a, b in zip(got, ref))
        den = max(abs(b) for b in ref)
    Jc = J.cpu().numpy()[0][..., 0, 0] + 1j * J.cpu().numpy()[0][..., 1, 0]
    budget = 64 * s.n_var * 2.0 ** -209 * np.linalg.cond(Jc)
    assert float(num / den) <= max(budget, 1e-60), (float(num / den), budget)


@pytest.mark.parametrize("points,shards", [(2000, 5), (5, 5)])
def test_range_call_common_support(phc, points, shards):
    """phc_eval_jacobian_batch_range on a common-support handle (the two-stage path, NEXT-2):
    shards of a batch call and of a few-point call (latency regime, chosen from the whole
    call's point count) are bitwise the unsharded call."""
    from synthetic import common_config
    c, X = common_config("common_dd", seed=4, points=points)
    h = phc.System(c, device=0)
    Xd = torch.from_numpy(X).cuda()
    F, J = h.eval_batch(Xd)
    Fr, Jr = torch.zeros_like(F), torch.zeros_like(J)
    for r in range(shards):
        h.eval_batch_range(Xd, r * points // shards, (r + 1) * points // shards, Fr, Jr)
    torch.cuda.synchronize()
    assert torch.equal(Fr, F) and torch.equal(Jr, J)


@pytest.mark.parametrize("seed", [2, 3])
def test_large_other_seeds_sampled_rows(phc, seed):
    """Two more random systems of the large shape (seeds 2, 3; single point): 3 rows of F and J
    against the mp512 oracle computed here (the committed values cover seed 1 in full)."""
    from _parity import compare_point, oracle_point
    s, X = config_system("large", seed=seed)
    h = phc.System(s, device=0)
    f, j = h.eval(torch.from_numpy(X[0]).cuda())
    torch.cuda.synchronize()
    rows = [0, 100 + seed, 255]
    ar, Fr, Jr = oracle_point(s, X[0], rows=rows, arith="mp")
    ef, ej = compare_point(ar, Fr, Jr, f.cpu().numpy(), j.cpu().numpy(), 4, rows)
    assert ef <= TOL[4] and ej <= TOL[4], (ef, ej)


@pytest.mark.parametrize("seed", [2, 3])
def test_batch_other_seeds_sampled_points(phc, seed):
    """The batch shape on two more random systems (seeds 2, 3; all 65,536 points in one call,
    the bench configuration): 4 points against the exact oracle, every entry."""
    from _parity import compare_point, oracle_point
    s, X = config_system("batch", seed=seed)
    h = phc.System(s, device=0)
    F, J = h.eval_batch(torch.from_numpy(X).cuda())
    torch.cuda.synchronize()
    for p in (0, 777 * seed, 40000 + seed, 65535):
        ar, Fr, Jr = oracle_point(s, X[p], arith="exact")
        ef, ej = compare_point(ar, Fr, Jr, F[p].cpu().numpy(), J[p].cpu().numpy(), 2)
        assert ef <= TOL[2] and ej <= TOL[2], (p, ef, ej)
