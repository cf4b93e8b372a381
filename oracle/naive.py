"""ORACLE — test infrastructure only (see oracle/__init__.py).  Naive evaluator.

What it computes (the plain definition; SURVEY.md §8(c) "Definition"):

    f_i(x)     = sum_{t in T_i} c_t * prod_{j=1..k_t} x_{i_{t,j}}^{a_{t,j}}
    J_{i,v}(x) = df_i/dx_v
               = sum_{t in T_i, v in vars(t)} c_t * a_{t,v} * x_v^{a_{t,v}-1}
                                              * prod_{j: i_{t,j} != v} x_{i_{t,j}}^{a_{t,j}}

* Monomials are normalised, 0 <= i_1 < ... < i_k < n, a_j >= 1
  (§6).
* Y = "the evaluated polynomials ... along with all partial derivatives as needed
  in the Jacobian matrix" (Alg. 2 discussion): F and the full J.
* The exponent factor a_m multiplies the shifted monomial x^{a-e_m}
  (reading C3; the paper's P:524-531 omits it in words).
* Every monomial, and separately every derivative monomial, is evaluated by
  repeated multiplication of its factors (no Speelpenning sharing, no power
  table): this is the naive evaluator north_star asks for, and it shares no
  code with the GPU path.
* J_{i,v} = 0 exactly when no term of f_i contains x_v.

Arithmetic is pluggable:
* ``ExactArith`` — exact Gaussian dyadic rationals (a + b i) * 2^e with Python
  ints.  Every input limb is a double, hence a dyadic rational, so this is the
  exact value of the GPU's own inputs (SURVEY.md §8(c) pin P1).
* ``MPArith(prec)`` — mpmath complex at ``prec`` bits (default 512), inputs
  converted exactly from the limbs.
"""
from __future__ import annotations

import os
from multiprocessing import get_context

import mpmath


# ---------------------------------------------------------------------------
# arithmetics
# ---------------------------------------------------------------------------

class ExactArith:
    """Exact complex dyadic rationals, value = (re + i*im) * 2**e, re/im/e Python ints."""

    name = "exact"

    @staticmethod
    def real_from_double(d: float):
        num, den = float(d).as_integer_ratio()  # den is a power of two
        return num, -(den.bit_length() - 1)

    def from_limbs(self, re_limbs, im_limbs):
        acc = (0, 0, 0)
        for d in re_limbs:
            m, e = self.real_from_double(d)
            acc = self.add(acc, (m, 0, e))
        for d in im_limbs:
            m, e = self.real_from_double(d)
            acc = self.add(acc, (0, m, e))
        return acc

    def zero(self):
        return (0, 0, 0)

    def one(self):
        return (1, 0, 0)

    @staticmethod
    def mul(p, q):
        a, b, e = p
        c, d, f = q
        return (a * c - b * d, a * d + b * c, e + f)

    @staticmethod
    def add(p, q):
        a, b, e = p
        c, d, f = q
        if e > f:
            s = e - f
            return ((a << s) + c, (b << s) + d, f)
        s = f - e
        return (a + (c << s), b + (d << s), e)

    @staticmethod
    def scale_int(p, s: int):
        return (p[0] * s, p[1] * s, p[2])

    @staticmethod
    def to_mpc(p, prec=1024):
        a, b, e = p
        with mpmath.workprec(prec):
            return mpmath.mpc(mpmath.ldexp(mpmath.mpf(a), e), mpmath.ldexp(mpmath.mpf(b), e))


class MPArith:
    """mpmath complex at ``prec`` bits."""

    name = "mp"

    def __init__(self, prec: int = 512):
        self.prec = prec

    def from_limbs(self, re_limbs, im_limbs):
        with mpmath.workprec(self.prec + 1024):  # exact sum of the limbs
            re = mpmath.fsum([mpmath.mpf(float(d)) for d in re_limbs])
            im = mpmath.fsum([mpmath.mpf(float(d)) for d in im_limbs])
        return mpmath.mpc(re, im)

    def zero(self):
        return mpmath.mpc(0)

    def one(self):
        return mpmath.mpc(1)

    def mul(self, p, q):
        return p * q

    def add(self, p, q):
        return p + q

    def scale_int(self, p, s: int):
        return p * s

    @staticmethod
    def to_mpc(p, prec=1024):
        return p


# ---------------------------------------------------------------------------
# the definition
# ---------------------------------------------------------------------------

def monomial(ar, xs, factors):
    """prod_j x_{v_j}^{a_j} by repeated multiplication (factors = [(v, a), ...])."""
    r = ar.one()
    for v, a in factors:
        for _ in range(a):
            r = ar.mul(r, xs[v])
    return r


def derivative_monomial(ar, xs, factors, v_d):
    """d/dx_{v_d} of prod_j x_{v_j}^{a_j} = a_d * x_{v_d}^{a_d-1} * prod_{j != d} x_{v_j}^{a_j},
    evaluated by repeated multiplication, separately from the monomial itself."""
    r = ar.one()
    a_d = None
    for v, a in factors:
        if v == v_d:
            a_d = a
            for _ in range(a - 1):
                r = ar.mul(r, xs[v])
        else:
            for _ in range(a):
                r = ar.mul(r, xs[v])
    assert a_d is not None
    return ar.scale_int(r, a_d)


def _row(ar, sys_terms, coeffs, xs, n_var):
    """F_i and the dense J row i for one polynomial, accumulating terms in index order."""
    f = ar.zero()
    jrow = [ar.zero() for _ in range(n_var)]
    for factors, c in zip(sys_terms, coeffs):
        f = ar.add(f, ar.mul(c, monomial(ar, xs, factors)))
        for v, _a in factors:
            jrow[v] = ar.add(jrow[v], ar.mul(c, derivative_monomial(ar, xs, factors, v)))
    return f, jrow


def _unpack(system, X_point, ar, rows):
    L = system.limbs
    xs = [ar.from_limbs(X_point[v, 0, :L], X_point[v, 1, :L]) for v in range(system.n_var)]
    jobs = []
    for i in rows:
        terms, coeffs = [], []
        for t, factors in system.terms(i):
            terms.append(factors)
            coeffs.append(ar.from_limbs(system.coeff[t, 0], system.coeff[t, 1]))
        jobs.append((terms, coeffs))
    return xs, jobs


def _worker(args):
    arname, prec, terms, coeffs, xs, n_var = args
    ar = ExactArith() if arname == "exact" else MPArith(prec)
    if arname == "mp":
        mpmath.mp.prec = prec
    return _row(ar, terms, coeffs, xs, n_var)


def _procs():
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def evaluate_rows(system, X_point, rows=None, arith="mp", prec=512, workers=None):
    """Evaluate F_i and J row i for ``rows`` (default all) at one point.

    ``X_point`` is float64 [n_var][2][limbs].  Returns (F, J) as lists of values
    of the chosen arithmetic: F[r] and J[r][v] for r indexing ``rows``.
    Rows are spread over a process pool when ``workers`` > 1.
    """
    rows = list(range(system.n_eq)) if rows is None else list(rows)
    ar = ExactArith() if arith == "exact" else MPArith(prec)
    old = mpmath.mp.prec
    mpmath.mp.prec = prec
    try:
        xs, jobs = _unpack(system, X_point, ar, rows)
        workers = _procs() if workers is None else workers
        args = [(arith, prec, terms, coeffs, xs, system.n_var) for terms, coeffs in jobs]
        if workers > 1 and len(rows) > 1:
            with get_context("fork").Pool(min(workers, len(rows))) as pool:
                res = pool.map(_worker, args, chunksize=1)
        else:
            res = [_worker(a) for a in args]
    finally:
        mpmath.mp.prec = old
    return [r[0] for r in res], [r[1] for r in res]


def evaluate_system(system, X_point, arith="mp", prec=512, workers=None):
    """All rows: (F [n_eq], J [n_eq][n_var])."""
    return evaluate_rows(system, X_point, None, arith, prec, workers)
