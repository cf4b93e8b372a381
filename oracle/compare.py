"""ORACLE — test infrastructure only (see oracle/__init__.py).  Error metric.

Tolerance reading C9 (SURVEY.md §8(c) "Tolerance"): per point,
separately for F and for J, entries taken as complex moduli and the difference
Delta computed at >= 1024 bits from the GPU's limbs,

    err = max( ||Delta||_inf / ||ref||_inf ,  ||Delta||_F / ||ref||_F ).
"""
from __future__ import annotations

import mpmath
import numpy as np


def _limbs_to_mpc(re_limbs, im_limbs):
    return mpmath.mpc(mpmath.fsum([mpmath.mpf(float(d)) for d in re_limbs]),
                      mpmath.fsum([mpmath.mpf(float(d)) for d in im_limbs]))


def _check_shapes(ref_values, gpu_limbs):
    """The two sides must describe the same N complex values: ``gpu_limbs`` is [N][2][L]
    (real limbs, imaginary limbs) and ``ref_values`` has exactly N entries.  A mismatch is an
    error, never a silent truncation (``zip`` would compare only the common prefix)."""
    ref_values = list(ref_values)
    gpu_limbs = np.asarray(gpu_limbs)
    if gpu_limbs.ndim != 3 or gpu_limbs.shape[1] != 2 or gpu_limbs.shape[2] < 1:
        raise ValueError(f"gpu limbs must be [N][2][L], got shape {gpu_limbs.shape}")
    if len(ref_values) != gpu_limbs.shape[0]:
        raise ValueError(f"{len(ref_values)} oracle values against {gpu_limbs.shape[0]} GPU values")
    return ref_values, gpu_limbs


def rel_errors(ar, ref_values, gpu_limbs, prec=1024):
    """Normwise relative error of ``gpu_limbs`` (float64 [N][2][L]) against the
    oracle values ``ref_values`` (N values of arithmetic ``ar``).  Returns
    (err, max_abs_delta, max_abs_ref) as floats.  Raises ValueError when the two
    sides do not hold the same number of values."""
    ref_values, gpu_limbs = _check_shapes(ref_values, gpu_limbs)
    with mpmath.workprec(prec):
        inf_d = mpmath.mpf(0)
        inf_r = mpmath.mpf(0)
        fro_d = mpmath.mpf(0)
        fro_r = mpmath.mpf(0)
        for ref, g in zip(ref_values, gpu_limbs):
            r = ar.to_mpc(ref, prec)
            gv = _limbs_to_mpc(g[0], g[1])
            d = abs(gv - r)
            a = abs(r)
            inf_d = max(inf_d, d)
            inf_r = max(inf_r, a)
            fro_d += d * d
            fro_r += a * a
        if inf_r == 0:
            err = mpmath.mpf(0) if inf_d == 0 else mpmath.inf
        else:
            err = max(inf_d / inf_r, mpmath.sqrt(fro_d) / mpmath.sqrt(fro_r))
        return float(err), float(inf_d), float(inf_r)


def exact_equal_limbs(ar, ref_values, gpu_limbs):
    """True iff every GPU value equals the exact oracle value exactly (bitwise for
    exactly representable results, P5).  Raises ValueError when the two sides do not
    hold the same number of values."""
    ref_values, gpu_limbs = _check_shapes(ref_values, gpu_limbs)
    for ref, g in zip(ref_values, gpu_limbs):
        gv = ar.from_limbs(g[0], g[1])
        a, b, e = ar.add(gv, ar.scale_int(ref, -1))
        if a != 0 or b != 0:
            return False
    return True
