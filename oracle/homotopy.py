"""ORACLE — test infrastructure only (see oracle/__init__.py).  Homotopy evaluator (NEXT-3).

The paper's "new" evaluation handles the continuation parameter t through the
coefficients instead of treating it "as just another variable" (§7,
P:647-649, Table 6).  The homotopy is

    h_i(x, t) = sum_{t' in T_i} c_{t'}(t) * x^{a_{t'}},
    c(t)      = (1 - t) * c_start + t * c_target            (reading H1, DESIGN.md;
                                                             SPEC S:233 "c_ij(t)")

with start and target coefficients on one shared support.  Its Jacobian in x is the
plain definition (oracle/naive.py) with the blended coefficients, and

    dh_i/dt   = sum_{t' in T_i} (c_target - c_start) * x^{a_{t'}}

is the extra column the "old" t-as-variable evaluator produces.

Every step is the plain definition: the blended coefficient is formed first, then the
monomial and every derivative monomial by repeated multiplication (``naive._row``).
t is real, given as limbs (exact in ``ExactArith``).
"""
from __future__ import annotations

import mpmath

from .naive import ExactArith, MPArith, _row, monomial


def _arith(arith, prec):
    return ExactArith() if arith == "exact" else MPArith(prec)


def _real(ar, t_limbs):
    return ar.from_limbs(list(t_limbs), [0.0] * len(t_limbs))


def blended_coefficient(ar, cs, cf, t):
    """c(t) = (1 - t) * c_start + t * c_target (reading H1)."""
    one_minus_t = ar.add(ar.one(), ar.scale_int(t, -1))
    return ar.add(ar.mul(one_minus_t, cs), ar.mul(t, cf))


def evaluate_homotopy_rows(system, coeff_target, X_point, t_limbs, rows=None, arith="exact", prec=512):
    """(F, J) of h(., t) at one point for ``rows``: F[r], J[r][v] (values of the arithmetic)."""
    ar = _arith(arith, prec)
    rows = list(range(system.n_eq)) if rows is None else list(rows)
    old = mpmath.mp.prec
    mpmath.mp.prec = prec
    try:
        L = system.limbs
        xs = [ar.from_limbs(X_point[v, 0, :L], X_point[v, 1, :L]) for v in range(system.n_var)]
        t = _real(ar, t_limbs)
        F, J = [], []
        for i in rows:
            terms, coeffs = [], []
            for tt, factors in system.terms(i):
                cs = ar.from_limbs(system.coeff[tt, 0], system.coeff[tt, 1])
                cf = ar.from_limbs(coeff_target[tt, 0], coeff_target[tt, 1])
                terms.append(factors)
                coeffs.append(blended_coefficient(ar, cs, cf, t))
            f, jrow = _row(ar, terms, coeffs, xs, system.n_var)
            F.append(f)
            J.append(jrow)
    finally:
        mpmath.mp.prec = old
    return ar, F, J


def evaluate_homotopy_dt(system, coeff_target, X_point, rows=None, arith="exact", prec=512):
    """dh_i/dt = sum (c_target - c_start) x^a for ``rows`` (independent of t)."""
    ar = _arith(arith, prec)
    rows = list(range(system.n_eq)) if rows is None else list(rows)
    old = mpmath.mp.prec
    mpmath.mp.prec = prec
    try:
        L = system.limbs
        xs = [ar.from_limbs(X_point[v, 0, :L], X_point[v, 1, :L]) for v in range(system.n_var)]
        out = []
        for i in rows:
            acc = ar.zero()
            for tt, factors in system.terms(i):
                cs = ar.from_limbs(system.coeff[tt, 0], system.coeff[tt, 1])
                cf = ar.from_limbs(coeff_target[tt, 0], coeff_target[tt, 1])
                acc = ar.add(acc, ar.mul(ar.add(cf, ar.scale_int(cs, -1)), monomial(ar, xs, factors)))
            out.append(acc)
    finally:
        mpmath.mp.prec = old
    return ar, out
