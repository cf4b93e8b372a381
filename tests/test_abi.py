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
