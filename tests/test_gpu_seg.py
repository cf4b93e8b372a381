"""Segmented latency path (kernels_scan.cuh poly_seg_kernel): QD single-point
calls with 12 <= k <= 32 take it (G lanes per term, two factors per lane).  Parity against the
exact oracle for every compiled segment width on a ragged system (k = 0..12, terms not a
multiple of the slots), with several splits and with several terms per warp (the add branch
of the slot rows), the c3 config against the warp-scan kernel, and reproducibility."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from _parity import TOL, compare_point, oracle_point  # noqa: E402
from synthetic import config_system, system_from_terms  # noqa: E402
from synthetic.systems import unit_circle_limbs  # noqa: E402


@pytest.fixture(scope="module")
def phc():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1109_0545_b200 as m
    return m


def ragged_qd(seed=11, n=23, points=3):
    rng = np.random.default_rng(seed)
    polys = []
    for _ in range(n):
        terms = []
        for _ in range(int(rng.integers(1, 45))):
            k = int(rng.integers(0, 13))
            vs = sorted(rng.choice(n, k, replace=False).tolist())
            terms.append([(v, int(rng.integers(1, 6))) for v in vs])
        polys.append(terms)
    T = sum(len(p) for p in polys)
    coeff = unit_circle_limbs(rng.uniform(0, 6.283, T), 4, 1)
    s = system_from_terms(n, n, 4, polys, coeff)
    X = unit_circle_limbs(rng.uniform(0, 6.283, (points, n)), 4, 1)
    return s, X


def with_env(env, fn):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        return fn()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("env", [{"PHC_SEG": "8"}, {"PHC_SEG": "10"}, {"PHC_SEG": "12"}, {"PHC_SEG": "16"},
                                 {"PHC_SEG": "10", "PHC_SEG_S": "1"}, {"PHC_SEG": "8", "PHC_SEG_W": "1", "PHC_SEG_S": "2"}])
def test_seg_widths_ragged_vs_oracle(phc, env):
    s, X = ragged_qd()
    h = with_env(env, lambda: phc.System(s))
    st = h.stats
    assert st["latency_kernel"] == 2 and st["latency_G"] == int(env["PHC_SEG"]), st
    for p in range(len(X)):
        ar, Fr, Jr = oracle_point(s, X[p], arith="exact")
        f, j = h.eval(torch.from_numpy(X[p]).cuda())
        ef, ej = compare_point(ar, Fr, Jr, f.cpu().numpy(), j.cpu().numpy(), 4)
        assert ef <= TOL[4] and ej <= TOL[4], (env, p, ef, ej)


def test_c3_segmented_vs_warp_scan(phc):
    s, X = config_system("c3", seed=1)
    h = phc.System(s)
    st = h.stats
    assert st["latency_kernel"] == 2 and st["latency_G"] == 10 and st["latency_launches"] == 2, st
    h0 = with_env({"PHC_SEG": "0"}, lambda: phc.System(s))
    assert h0.stats["latency_kernel"] == 1
    x = torch.from_numpy(X[0]).cuda()
    f, j = h.eval(x)
    f0, j0 = h0.eval(x)
    a, b = f.cpu().numpy(), f0.cpu().numpy()
    scale = np.abs(b[..., 0]).max()
    assert np.abs((a - b).sum(-1)).max() <= 1e-60 * scale
    a, b = j.cpu().numpy(), j0.cpu().numpy()
    scale = np.abs(b[..., 0]).max()
    assert np.abs((a - b).sum(-1)).max() <= 1e-60 * scale
    # bitwise reproducible call to call
    for _ in range(3):
        f2, j2 = h.eval(x)
        assert torch.equal(f2, f) and torch.equal(j2, j)
