"""ORACLE — test infrastructure only (see oracle/__init__.py).  One Newton step.

Algorithm 2, one iteration, with the paper's stages:
  Y := evaluated polynomials and Jacobian at z
  ||h(z)|| := Residual(Y)                                  (reading N1: max_i |F_i|)
  Ab := GE([J | -F]) with partial pivoting
  dz := Back_Subs(Ab)
  z := z + dz
The linear system is J dz = -F (reading N2: Alg. 2 writes "A x = b" without signs).

The oracle solves J dz = -F EXACTLY (rational arithmetic, Gaussian elimination taking the
first nonzero pivot: in exact arithmetic the solution does not depend on the pivot order,
so the paper's "largest number in the current column" rule matters only for
rounding and is the GPU's business) or at 512 bits with mpmath.lu_solve.  Exact rational
elimination grows its numbers quickly (a 20 x 20 step takes minutes): use it for n <= 8
and the mp mode above that.
"""
from __future__ import annotations

from fractions import Fraction

import mpmath

from .naive import ExactArith, MPArith, evaluate_system


def _cf(p):
    """exact dyadic complex (re, im, e) -> (Fraction, Fraction)"""
    a, b, e = p
    s = Fraction(2) ** e
    return (a * s, b * s)


def _cmul(x, y):
    return (x[0] * y[0] - x[1] * y[1], x[0] * y[1] + x[1] * y[0])


def _csub(x, y):
    return (x[0] - y[0], x[1] - y[1])


def _cdiv(x, y):
    d = y[0] * y[0] + y[1] * y[1]
    return ((x[0] * y[0] + x[1] * y[1]) / d, (x[1] * y[0] - x[0] * y[1]) / d)


def solve_exact(A, b):
    """Exact solution of A x = b over Q(i) by Gaussian elimination (first nonzero pivot).
    A: n x n list of (Fraction, Fraction); b: n list.  Returns x or None if singular."""
    n = len(A)
    M = [list(A[i]) + [b[i]] for i in range(n)]
    for k in range(n):
        p = next((i for i in range(k, n) if M[i][k] != (0, 0)), None)
        if p is None:
            return None
        M[k], M[p] = M[p], M[k]
        for i in range(k + 1, n):
            if M[i][k] == (0, 0):
                continue
            l = _cdiv(M[i][k], M[k][k])
            for j in range(k, n + 1):
                M[i][j] = _csub(M[i][j], _cmul(l, M[k][j]))
    x = [None] * n
    for i in range(n - 1, -1, -1):
        acc = M[i][n]
        for j in range(i + 1, n):
            acc = _csub(acc, _cmul(M[i][j], x[j]))
        x[i] = _cdiv(acc, M[i][i])
    return x


def newton_step(system, X_point, arith="exact", prec=512, workers=None):
    """One Newton step at the point X_point ([n][2][L] limbs).

    Returns dict(residual, dz, z_new, singular) with
      residual = max_i |F_i| (float),
      dz, z_new: exact mode -> lists of (Fraction, Fraction); mp mode -> lists of mpc."""
    assert system.n_eq == system.n_var, "Newton needs a square system"
    F, J = evaluate_system(system, X_point, arith, prec, workers)
    n = system.n_eq
    if arith == "exact":
        ar = ExactArith()
        Fq = [_cf(f) for f in F]
        Jq = [[_cf(v) for v in row] for row in J]
        zq = [_cf(ar.from_limbs(X_point[v, 0], X_point[v, 1])) for v in range(n)]
        res = max(abs(complex(float(f[0]), float(f[1]))) for f in Fq) if n else 0.0
        dz = solve_exact(Jq, [(-f[0], -f[1]) for f in Fq])
        if dz is None:
            return dict(residual=res, dz=None, z_new=None, singular=True)
        z_new = [(a[0] + d[0], a[1] + d[1]) for a, d in zip(zq, dz)]
        return dict(residual=res, dz=dz, z_new=z_new, singular=False)
    ar = MPArith(prec)
    with mpmath.workprec(prec):
        z = [ar.from_limbs(X_point[v, 0], X_point[v, 1]) for v in range(n)]
    return solve_step_mp(F, J, z, prec)


def solve_step_mp(F, J, z, prec=512):
    """The solve and update of one Newton step from evaluated F [n] and J [n][n]
    (mpmath complex values) at the point z [n]: residual max_i |F_i|, dz = J^{-1} (-F) by
    mpmath.lu_solve at `prec` bits, z_new = z + dz.  (newton_step's mp mode after the
    evaluation; separate so stored oracle values of F and J can be reused.)"""
    n = len(F)
    with mpmath.workprec(prec):
        res = float(max(abs(f) for f in F))
        A = mpmath.matrix([[J[i][v] for v in range(n)] for i in range(n)])
        b = mpmath.matrix([-F[i] for i in range(n)])
        try:
            dzm = mpmath.lu_solve(A, b)
        except ZeroDivisionError:
            return dict(residual=res, dz=None, z_new=None, singular=True)
        dz = [dzm[i] for i in range(n)]
        return dict(residual=res, dz=dz, z_new=[a + d for a, d in zip(z, dz)], singular=False)
