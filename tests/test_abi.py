"""The C-ABI library loads and exports every symbol include/phc.h declares; validation
errors are reported (no GPU needed: validation precedes any device call)."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_header_symbols():
    import paper_1109_0545_b200._lib as L
    hdr = open(os.path.join(ROOT, "include", "phc.h")).read()
    names = set(re.findall(r"\b(phc_\w+)\s*\(", hdr))
    assert names == set(L.EXPORTED)
    for n in names:
        assert hasattr(L.lib, n), n
    assert L.phc_version().startswith("phc-b200")


def _arrays(**over):
    from synthetic import config_system
    s, _ = config_system("tiny", seed=1)
    for k, v in over.items():
        setattr(s, k, v)
    return s


@pytest.mark.parametrize("mut,code", [
    (lambda s: setattr(s, "limbs", 3), -4),
    (lambda s: setattr(s, "n_eq", 0), -1),
    (lambda s: s.var_idx.__setitem__(5, s.var_idx[4]), -1),   # not strictly increasing
    (lambda s: s.var_idx.__setitem__(0, 99), -1),             # out of range
    (lambda s: s.exponent.__setitem__(3, 0), -1),             # exponent < 1
    (lambda s: s.exponent.__setitem__(3, 300), -4),           # beyond compiled limit
    (lambda s: s.coeff.__setitem__((2, 0, 1), np.nan), -1),   # non-finite coefficient
    (lambda s: s.poly_ptr.__setitem__(8, 63), -1),            # wrong end value
])
def test_validation_errors(mut, code):
    import paper_1109_0545_b200 as phc
    s = _arrays()
    s.var_idx = s.var_idx.copy()
    s.exponent = s.exponent.copy()
    s.coeff = s.coeff.copy()
    s.poly_ptr = s.poly_ptr.copy()
    mut(s)
    with pytest.raises(phc.PhcError) as ei:
        phc.System(s)
    assert ei.value.code == code, str(ei.value)


def test_no_fallback_without_library(tmp_path, monkeypatch):
    """The binding refuses to import without libphc.so (no CPU fallback)."""
    import importlib.util
    src = os.path.join(ROOT, "paper_1109_0545_b200", "_lib.py")
    spec = importlib.util.spec_from_file_location("phc_lib_copy", src)
    mod = importlib.util.module_from_spec(spec)
    monkeypatch.setattr(os.path, "exists", lambda p: False)
    with pytest.raises(ImportError):
        spec.loader.exec_module(mod)


@pytest.mark.parametrize("mut,code", [
    (lambda c: setattr(c, "limbs", 3), -4),
    (lambda c: setattr(c, "mono_ptr", np.zeros(1, np.int64)), -1),            # no monomials
    (lambda c: c.coeff.__setitem__((1, 2, 0, 0), np.inf), -1),                # non-finite coefficient
    (lambda c: c.var_idx.__setitem__(0, 40), -1),                             # variable out of range
])
def test_common_validation_errors(mut, code):
    """phc_system_create_common (NEXT-2) validates before touching a device."""
    import paper_1109_0545_b200 as phc
    from synthetic import common_support_system
    c, _ = common_support_system(8, 12, 2, 5, 3, 2, seed=1)
    c.coeff = c.coeff.copy()
    c.var_idx = c.var_idx.copy()
    mut(c)
    with pytest.raises(phc.PhcError) as ei:
        phc.System(c)
    assert ei.value.code == code, str(ei.value)


def test_expand_common_structure():
    """The expansion used by the oracle keeps every (polynomial, monomial) pair in order."""
    from synthetic import common_support_system, expand_common
    c, _ = common_support_system(6, 9, 1, 4, 2, 4, seed=3)
    e = expand_common(c)
    assert e.n_terms == 6 * 9
    for i in range(6):
        for j, (t, fac) in enumerate(e.terms(i)):
            a, b = int(c.mono_ptr[j]), int(c.mono_ptr[j + 1])
            assert fac == list(zip(c.var_idx[a:b].tolist(), c.exponent[a:b].tolist()))
            assert np.array_equal(e.coeff[t], c.coeff[i, j])


def test_next_row_entry_points_validate_without_device():
    """The NEXT-row entry points reject bad arguments before touching a device."""
    import ctypes
    import paper_1109_0545_b200._lib as L
    lib = L.lib
    P = ctypes.c_void_p
    # predictor: bad limbs / order / NULL pointers
    assert lib.phc_predict_batch(3, 4, 1, 2, None, None, None, None, None, None) == L.PHC_EUNSUPPORTED
    assert lib.phc_predict_batch(2, 4, 1, 3, None, None, None, None, None, None) == L.PHC_EINVAL
    assert lib.phc_predict_batch(2, 4, 1, 2, None, None, None, None, None, None) == L.PHC_EINVAL
    assert lib.phc_predict_batch(2, 4, 0, 2, None, None, None, None, None, None) == L.PHC_OK  # no paths: no-op
    # arithmetic self-test hook
    assert lib.phc_arith_test(11, 2, 4, None, None, None, None) == L.PHC_EINVAL
    assert lib.phc_arith_test(0, 3, 4, None, None, None, None) == L.PHC_EUNSUPPORTED
    assert lib.phc_arith_test(0, 2, 0, None, None, None, None) == L.PHC_OK
    # NULL handles
    prm = L.TrackParams(step_init=0.01, step_min=1e-8, step_max=0.1, expand=2.0, contract=0.5, tol=1e-20,
                        max_newton=4, max_steps=10, end_newton=0, predictor=2)
    assert lib.phc_track_paths(None, 1, None, ctypes.byref(prm), None, None, None, None) == L.PHC_EINVAL
    assert lib.phc_system_set_target(None, None) == L.PHC_EINVAL
    assert lib.phc_eval_homotopy_batch(None, 1, None, None, None, None, None, 0, None) == L.PHC_EINVAL
    assert lib.phc_newton_step_homotopy_batch(None, 1, None, None, None, None, None, None) == L.PHC_EINVAL
    assert lib.phc_newton_solve_batch(None, 1, None, None, 1e-20, 4, None, None, None, None, None) == L.PHC_EINVAL
    h = P()
    assert lib.phc_homotopy_old_create(ctypes.byref(h), 0, 1, 2, 0, None, None, None, None, None, None, 0) == L.PHC_EINVAL
    assert lib.phc_system_create_common(ctypes.byref(h), 2, 2, 2, 0, None, None, None, None, 0) == L.PHC_EINVAL
    assert "NULL" in L.phc_last_error() or L.phc_last_error() != ""


def test_range_and_ipc_entry_points_validate_without_device():
    """The multi-process entry points reject bad arguments before touching a device."""
    import ctypes
    import paper_1109_0545_b200._lib as L
    lib = L.lib
    P = ctypes.c_void_p
    assert lib.phc_eval_jacobian_batch_range(None, 10, 0, 5, None, None, None, None) == L.PHC_EINVAL
    off = ctypes.c_int64()
    assert lib.phc_ipc_get_handle(None, None, ctypes.byref(off)) == L.PHC_EINVAL
    base = P()
    assert lib.phc_ipc_open(None, 0, ctypes.byref(base)) == L.PHC_EINVAL
    assert lib.phc_ipc_close(None, 0) == L.PHC_OK  # NULL mapping: no-op
    assert "NULL" in L.phc_last_error() or L.phc_last_error() == ""
