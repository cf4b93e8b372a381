"""ORACLE — test infrastructure only (see oracle/__init__.py).  Predictor (NEXT-4).

PAPER.md §5: for each coordinate i independently, "interpolate points
(t_prev1, x*_prev1[i]), (t_prev, x*_prev[i]), and (t, x*[i]) by a parabola"; the new guess
is "the value of this parabola at the point (t + current step size)".  With fewer accepted
points the interpolant has lower degree (reading T2: 2 points = secant line, 1 point =
constant).  This is the plain Lagrange form

    p(tau) = sum_j x_j prod_{m != j} (tau - t_m) / (t_j - t_m)

in exact rationals (inputs are limbs, hence dyadic), one coordinate at a time; the CUDA
kernel uses Newton divided differences, so the two share no arithmetic.
"""
from __future__ import annotations

from fractions import Fraction


def real_from_limbs(limbs) -> Fraction:
    return sum((Fraction(float(d)) for d in limbs), Fraction(0))


def complex_from_limbs(re_limbs, im_limbs):
    return real_from_limbs(re_limbs), real_from_limbs(im_limbs)


def lagrange_value(ts, xs, tau):
    """Value at tau of the interpolant through (ts[j], xs[j]); xs complex as (re, im) Fractions."""
    re, im = Fraction(0), Fraction(0)
    for j, (tj, xj) in enumerate(zip(ts, xs)):
        w = Fraction(1)
        for m, tm in enumerate(ts):
            if m != j:
                w *= (tau - tm) / (tj - tm)
        re += w * xj[0]
        im += w * xj[1]
    return re, im


def predict_point(t_hist, x_hist, h, t_new):
    """One path: t_hist [3][L] limbs (slot 0 newest), x_hist [3][n][2][L], h valid slots used,
    t_new [L] -> list of n exact complex predictions."""
    ts = [real_from_limbs(t_hist[s]) for s in range(h)]
    tau = real_from_limbs(t_new)
    n = len(x_hist[0])
    out = []
    for i in range(n):
        xs = [complex_from_limbs(x_hist[s][i][0], x_hist[s][i][1]) for s in range(h)]
        out.append(lagrange_value(ts, xs, tau))
    return out
