"""Shared helpers for parity tests: run the GPU path through the C ABI, compare with the oracle."""
import numpy as np

from oracle import ExactArith, MPArith, evaluate_rows, rel_errors

TOL = {2: 1e-28, 4: 1e-60}  # BASELINE.json north_star: <=1e-28 (DD), <=1e-60 (QD), in norm (reading C9)


def oracle_point(s, Xp, rows=None, arith=None, prec=512):
    """Oracle F/J rows at one point: exact arithmetic by default, mp512 when arith='mp'."""
    arith = arith or "exact"
    F, J = evaluate_rows(s, Xp, rows, arith, prec)
    ar = ExactArith() if arith == "exact" else MPArith(prec)
    return ar, F, J


def compare_point(ar, F, J, f_gpu, j_gpu, L, rows=None):
    """Normwise relative errors (reading C9) of the GPU rows vs the oracle rows."""
    rows = list(range(f_gpu.shape[0])) if rows is None else list(rows)
    fg = np.asarray(f_gpu)[rows]
    jg = np.asarray(j_gpu)[rows].reshape(-1, 2, L)
    ef, _, _ = rel_errors(ar, F, fg)
    ej, _, _ = rel_errors(ar, [v for row in J for v in row], jg)
    return ef, ej


def limbs_normalised(a):
    """hi == fl(hi + lo) for DD; |x_{l+1}| <= ulp(x_l) for QD (non-overlapping)."""
    a = np.asarray(a)
    L = a.shape[-1]
    x = a.reshape(-1, L)
    for l in range(L - 1):
        hi, lo = x[:, l], x[:, l + 1]
        ok = (hi == 0) & (lo == 0) | (np.abs(lo) <= np.spacing(np.abs(hi)))
        if not ok.all():
            return False
    return True
