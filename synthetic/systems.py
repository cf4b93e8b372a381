"""Seeded generators for sparse polynomial systems and evaluation points.

Recipe (SURVEY.md §8(d) "Synthetic inputs", readings C7 and C11 in DESIGN.md):

* ``rng = numpy.random.Generator(numpy.random.PCG64(seed))``.
* For each polynomial i = 0..n-1 and term t = 0..m-1 (independent supports per
  polynomial, reading C7): ``vars = sorted(rng.choice(n, k, replace=False))``,
  ``exps = rng.integers(1, D+1, k)``, ``theta_c = rng.uniform(0, 2*pi)``.
* Then point angles ``rng.uniform(0, 2*pi, size=(P, n))``.
* Each real cos/sin of an angle (the double theta, taken exactly) is evaluated
  in mpmath at 64*L+64 bits and split greedily into L round-to-nearest doubles,
  giving normalised DD (L=2) or QD (L=4) limbs.

Array layout is the one ``include/phc.h`` declares: ``coeff`` and points are
``[..][2][L]`` float64 with the real limbs first, then the imaginary limbs.

This module holds none of the evaluation method's arithmetic; the limb split
below is input preparation (round a high-precision real to a limb vector).
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass
from multiprocessing import get_context

import numpy as np
from mpmath.libmp import from_float, from_int, from_rational, mpf_cos_sin, mpf_sub, round_nearest, to_float

# BASELINE.json configs[0..4] (n, m, k, D, limbs, points)
CONFIGS = {
    "tiny": dict(n=8, m=8, k=4, D=3, limbs=2, points=1),
    "c2": dict(n=20, m=20, k=10, D=4, limbs=2, points=1),
    "c3": dict(n=40, m=40, k=20, D=5, limbs=4, points=1),
    "batch": dict(n=32, m=32, k=16, D=4, limbs=2, points=65536),
    "large": dict(n=256, m=256, k=32, D=8, limbs=4, points=1),
    "large_batch": dict(n=256, m=256, k=32, D=8, limbs=4, points=4096),
}


@dataclass
class SystemArrays:
    """A sparse polynomial system in the C-ABI's CSR layout (include/phc.h)."""

    n_eq: int
    n_var: int
    limbs: int
    poly_ptr: np.ndarray  # int64 [n_eq+1]
    term_ptr: np.ndarray  # int64 [n_terms+1]
    var_idx: np.ndarray  # int32 [n_factors], 0-based, strictly increasing per term
    exponent: np.ndarray  # int32 [n_factors], >= 1
    coeff: np.ndarray  # float64 [n_terms][2][limbs]

    @property
    def n_terms(self) -> int:
        return int(self.term_ptr.shape[0] - 1)

    def terms(self, i):
        """Yield (t, [(var, exp), ...]) for the terms of polynomial i (host helper)."""
        for t in range(int(self.poly_ptr[i]), int(self.poly_ptr[i + 1])):
            a, b = int(self.term_ptr[t]), int(self.term_ptr[t + 1])
            yield t, list(zip(self.var_idx[a:b].tolist(), self.exponent[a:b].tolist()))


def split_limbs(v, limbs: int, prec: int) -> list[float]:
    """Greedy round-to-nearest split of an mpmath mpf tuple into ``limbs`` doubles."""
    out = []
    r = v
    for _ in range(limbs):
        h = to_float(r, False, round_nearest)  # round to nearest (mpmath's default truncates)
        out.append(h)
        r = mpf_sub(r, from_float(h), prec)
    return out


def _cos_sin_limbs(args):
    thetas, limbs = args
    prec = 64 * limbs + 64
    out = np.empty((len(thetas), 2, limbs), dtype=np.float64)
    for j, th in enumerate(thetas):
        c, s = mpf_cos_sin(from_float(float(th)), prec)
        out[j, 0, :] = split_limbs(c, limbs, prec)
        out[j, 1, :] = split_limbs(s, limbs, prec)
    return out


def _procs() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def unit_circle_limbs(thetas: np.ndarray, limbs: int, workers: int | None = None) -> np.ndarray:
    """e^{i theta} for every double theta, as [..., 2, limbs] float64 limbs."""
    flat = np.ascontiguousarray(thetas, dtype=np.float64).reshape(-1)
    if flat.size == 0:
        return np.empty(thetas.shape + (2, limbs))
    workers = workers or _procs()
    if flat.size < 4096 or workers == 1:
        res = _cos_sin_limbs((flat, limbs))
    else:
        chunks = np.array_split(flat, workers * 4)
        with get_context("fork").Pool(workers) as pool:
            res = np.concatenate(pool.map(_cos_sin_limbs, [(c, limbs) for c in chunks]))
    return res.reshape(thetas.shape + (2, limbs))


def system_from_terms(n_eq, n_var, limbs, polys, coeff_limbs) -> SystemArrays:
    """Build CSR arrays from ``polys[i] = [[(var, exp), ...] per term]`` and coefficient limbs [T][2][L]."""
    poly_ptr = [0]
    term_ptr = [0]
    vi, ex = [], []
    for terms in polys:
        for term in terms:
            for v, a in term:
                vi.append(v)
                ex.append(a)
            term_ptr.append(len(vi))
        poly_ptr.append(len(term_ptr) - 1)
    coeff = np.asarray(coeff_limbs, dtype=np.float64).reshape(len(term_ptr) - 1, 2, limbs)
    return SystemArrays(
        n_eq=n_eq,
        n_var=n_var,
        limbs=limbs,
        poly_ptr=np.asarray(poly_ptr, dtype=np.int64),
        term_ptr=np.asarray(term_ptr, dtype=np.int64),
        var_idx=np.asarray(vi, dtype=np.int32),
        exponent=np.asarray(ex, dtype=np.int32),
        coeff=np.ascontiguousarray(coeff),
    )


def random_system(n, m, k, D, limbs, seed, points=1, workers=None):
    """The BASELINE.json system family: n polynomials, m terms each, k distinct variables
    per term, exponents iid uniform in 1..D, unit-circle coefficients and points.

    Returns (SystemArrays, X) with X float64 [points][n][2][limbs].
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    polys = []
    thetas_c = np.empty(n * m)
    for i in range(n):
        terms = []
        for t in range(m):
            vars_ = sorted(rng.choice(n, k, replace=False).tolist())
            exps = rng.integers(1, D + 1, k).tolist()
            thetas_c[i * m + t] = rng.uniform(0.0, 2.0 * math.pi)
            terms.append(list(zip(vars_, exps)))
        polys.append(terms)
    thetas_x = rng.uniform(0.0, 2.0 * math.pi, size=(points, n))
    coeff = unit_circle_limbs(thetas_c, limbs, workers)
    X = unit_circle_limbs(thetas_x, limbs, workers)
    return system_from_terms(n, n, limbs, polys, coeff), X


def config_system(name: str, seed: int = 1, points: int | None = None, workers=None):
    """System + points for a BASELINE.json config name (see CONFIGS)."""
    c = CONFIGS[name]
    P = c["points"] if points is None else points
    return random_system(c["n"], c["m"], c["k"], c["D"], c["limbs"], seed, P, workers)


def config_point_rows(name: str, seed: int, rows, points: int | None = None):
    """Rows ``rows`` of the point batch ``config_system(name, seed, points)`` draws, without
    converting the other points' angles (the same generator stream: the system's draws, then
    the (points, n) angle matrix).  Returns float64 [len(rows)][n][2][limbs]."""
    c = CONFIGS[name]
    P = c["points"] if points is None else points
    n, m, k, D, limbs = c["n"], c["m"], c["k"], c["D"], c["limbs"]
    rng = np.random.Generator(np.random.PCG64(seed))
    for _ in range(n * m):
        rng.choice(n, k, replace=False)
        rng.integers(1, D + 1, k)
        rng.uniform(0.0, 2.0 * math.pi)
    thetas_x = rng.uniform(0.0, 2.0 * math.pi, size=(P, n))
    return unit_circle_limbs(thetas_x[list(rows)], limbs)


def limbs_from_values(values, limbs: int) -> np.ndarray:
    """Exact small complex values (Python complex / int / Fraction pairs) → [..][2][limbs] limbs.

    Each real part is split greedily; for values that are doubles the tail limbs are 0.
    """
    arr = []
    prec = 64 * limbs + 64
    for z in values:
        if isinstance(z, tuple):
            re, im = z
        else:
            re, im = complex(z).real, complex(z).imag
        row = []
        for part in (re, im):
            if hasattr(part, "numerator") and not isinstance(part, (int, float)):
                mp = from_rational(part.numerator, part.denominator, prec)
            elif isinstance(part, int):
                mp = from_int(part)
            else:
                mp = from_float(float(part))
            row.append(split_limbs(mp, limbs, prec))
        arr.append(row)
    return np.asarray(arr, dtype=np.float64).reshape(len(values), 2, limbs)


# ---------------------------------------------------------------------------
# Special systems whose results are known without the oracle
# ---------------------------------------------------------------------------

def special_linear_system(n, limbs, seed):
    """k = 1, a = 1, each (i, v) once: F = C x and J = C exactly (P4).

    Coefficients are small Gaussian integers, points small Gaussian integers, so
    every intermediate result is an exact double.  Returns (system, X, C) with C
    an int64 [n][n][2] array of Gaussian-integer coefficients.
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    C = rng.integers(-9, 10, size=(n, n, 2))
    polys = [[[(v, 1)] for v in range(n)] for _ in range(n)]
    coeff = np.zeros((n * n, 2, limbs))
    coeff[:, 0, 0] = C[:, :, 0].reshape(-1)
    coeff[:, 1, 0] = C[:, :, 1].reshape(-1)
    x = rng.integers(-9, 10, size=(n, 2))
    X = np.zeros((1, n, 2, limbs))
    X[0, :, 0, 0] = x[:, 0]
    X[0, :, 1, 0] = x[:, 1]
    return system_from_terms(n, n, limbs, polys, coeff), X, C, x


def special_gaussian_system(n, m, k, D, limbs, seed):
    """Random sparse system with coefficients in Z[i] (|re|,|im| <= 3) and a point in {±1, ±i}^n.

    Every monomial value is a unit in Z[i] and every partial is a small Gaussian
    integer, so all intermediates are exact doubles (P5): the GPU output must
    equal the exact result bitwise.
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    polys = []
    cl = []
    for i in range(n):
        terms = []
        for t in range(m):
            kk = min(k, n)
            vars_ = sorted(rng.choice(n, kk, replace=False).tolist())
            exps = rng.integers(1, D + 1, kk).tolist()
            terms.append(list(zip(vars_, exps)))
            cl.append(rng.integers(-3, 4, size=2))
        polys.append(terms)
    coeff = np.zeros((len(cl), 2, limbs))
    coeff[:, :, 0] = np.asarray(cl)
    units = np.array([[1, 0], [-1, 0], [0, 1], [0, -1]])
    X = np.zeros((1, n, 2, limbs))
    X[0, :, :, 0] = units[rng.integers(0, 4, size=n)]
    return system_from_terms(n, n, limbs, polys, coeff), X


def special_univariate_system(degree, limbs, seed):
    """n = 1, f(x) = sum_{d=0}^{degree} c_d x^d (P4: reduces to Horner / mpmath.polyval).

    The constant term c_0 is a k = 0 term.  Returns (system, X, thetas_c, theta_x).
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    polys = [[[]] + [[(0, d)] for d in range(1, degree + 1)]]
    thetas_c = rng.uniform(0.0, 2.0 * math.pi, size=degree + 1)
    theta_x = rng.uniform(0.0, 2.0 * math.pi, size=(1, 1))
    coeff = unit_circle_limbs(thetas_c, limbs, 1)
    X = unit_circle_limbs(theta_x, limbs, 1)
    return system_from_terms(1, 1, limbs, polys, coeff), X


def homogeneous_system(n, m, k, d, limbs, seed, points=1):
    """Every term of f_i has total degree d_i = d + (i % 3) (P8 Euler identity:
    sum_v x_v J_{i,v} = d_i f_i).  Exponent vectors are compositions of d_i into k
    positive parts.  Returns (system, X, degrees)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    polys = []
    degs = []
    thetas_c = np.empty(n * m)
    for i in range(n):
        di = d + (i % 3)
        degs.append(di)
        kk = min(k, n, di)
        terms = []
        for t in range(m):
            vars_ = sorted(rng.choice(n, kk, replace=False).tolist())
            cuts = sorted(rng.choice(np.arange(1, di), kk - 1, replace=False).tolist()) if kk > 1 else []
            bounds = [0] + cuts + [di]
            exps = [bounds[j + 1] - bounds[j] for j in range(kk)]
            thetas_c[i * m + t] = rng.uniform(0.0, 2.0 * math.pi)
            terms.append(list(zip(vars_, exps)))
        polys.append(terms)
    thetas_x = rng.uniform(0.0, 2.0 * math.pi, size=(points, n))
    coeff = unit_circle_limbs(thetas_c, limbs, 1)
    X = unit_circle_limbs(thetas_x, limbs, 1)
    return system_from_terms(n, n, limbs, polys, coeff), X, degs


# ---------------------------------------------------------------------------
# Homotopy inputs (NEXT-3): target coefficients on the same support, and real t values
# ---------------------------------------------------------------------------

def homotopy_target(system, seed, workers=None) -> np.ndarray:
    """Target coefficients c_target [n_terms][2][L] on the system's support: unit-circle,
    angles from ``PCG64(seed)`` (the start coefficients are the system's own)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    thetas = rng.uniform(0.0, 2.0 * math.pi, size=system.n_terms)
    return unit_circle_limbs(thetas, system.limbs, workers)


def real_limbs(values, limbs: int) -> np.ndarray:
    """Real numbers (float, int or Fraction) → [len][limbs] float64 limbs (greedy split)."""
    prec = 64 * limbs + 64
    out = np.zeros((len(values), limbs))
    for j, v in enumerate(values):
        if hasattr(v, "numerator") and not isinstance(v, (int, float)):
            mp = from_rational(v.numerator, v.denominator, prec)
        elif isinstance(v, int):
            mp = from_int(v)
        else:
            mp = from_float(float(v))
        out[j] = split_limbs(mp, limbs, prec)
    return out


def random_t(P, limbs, seed) -> np.ndarray:
    """P seeded values of t in (0, 1) with full DD/QD limbs: t = u / 2^(53 L) for a uniform
    integer u, so every limb is significant (the tracker's t are sums of step sizes)."""
    from fractions import Fraction

    rng = np.random.Generator(np.random.PCG64(seed))
    bits = 53 * limbs
    vals = []
    for _ in range(P):
        u = 0
        for _w in range((bits + 31) // 32):
            u = (u << 32) | int(rng.integers(0, 1 << 32))
        u >>= (((bits + 31) // 32) * 32 - bits)
        vals.append(Fraction(u, 1 << bits))
    return real_limbs(vals, limbs)


# ---------------------------------------------------------------------------
# Common-support systems (NEXT-2; Table 1)
# ---------------------------------------------------------------------------

@dataclass
class CommonArrays:
    """A common-support system in the layout of phc_system_create_common: M monomials
    (CSR ``mono_ptr``/``var_idx``/``exponent``) shared by all n_eq polynomials, dense
    coefficients ``coeff`` [n_eq][M][2][L]."""

    n_eq: int
    n_var: int
    limbs: int
    mono_ptr: np.ndarray
    var_idx: np.ndarray
    exponent: np.ndarray
    coeff: np.ndarray

    @property
    def n_mono(self) -> int:
        return int(self.mono_ptr.shape[0] - 1)


def common_support_system(n, M, kmin, kmax, amax, limbs, seed, points=1, workers=None):
    """Table 1 shaped system (reading N2-1): n variables and equations, M shared
    monomials; monomial j has k_j ~ U{kmin..kmax} distinct sorted variables with exponents
    ~ U{1..amax}; unit-circle coefficients C[i][j] and points.  Returns (CommonArrays, X)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    mono_ptr, vi, ex = [0], [], []
    for _ in range(M):
        k = int(rng.integers(kmin, kmax + 1))
        vs = sorted(rng.choice(n, k, replace=False).tolist())
        es = rng.integers(1, amax + 1, k).tolist()
        vi += vs
        ex += es
        mono_ptr.append(len(vi))
    thetas_c = rng.uniform(0.0, 2.0 * math.pi, size=(n, M))
    thetas_x = rng.uniform(0.0, 2.0 * math.pi, size=(points, n))
    coeff = unit_circle_limbs(thetas_c, limbs, workers)
    X = unit_circle_limbs(thetas_x, limbs, workers)
    return CommonArrays(n, n, limbs, np.asarray(mono_ptr, np.int64), np.asarray(vi, np.int32),
                        np.asarray(ex, np.int32), np.ascontiguousarray(coeff)), X


# NEXT-2 configs: the Table 1 shape in complex QD (the precision of the paper's
# tracking runs) and DD, single point and batch
COMMON_CONFIGS = {
    "common": dict(n=40, M=200, kmin=10, kmax=30, amax=3, limbs=4, points=1),
    "common_dd": dict(n=40, M=200, kmin=10, kmax=30, amax=3, limbs=2, points=1),
    "common_batch": dict(n=40, M=200, kmin=10, kmax=30, amax=3, limbs=2, points=8192),
}


def common_config(name: str, seed: int = 1, points: int | None = None, workers=None):
    c = COMMON_CONFIGS[name]
    P = c["points"] if points is None else points
    return common_support_system(c["n"], c["M"], c["kmin"], c["kmax"], c["amax"], c["limbs"], seed, P, workers)


def expand_common(cs: CommonArrays) -> SystemArrays:
    """The same polynomials as an ordinary system (term (i, j) = C[i][j] x^{a_j}), for the
    oracle and for the per-term path."""
    monos = []
    for j in range(cs.n_mono):
        a, b = int(cs.mono_ptr[j]), int(cs.mono_ptr[j + 1])
        monos.append(list(zip(cs.var_idx[a:b].tolist(), cs.exponent[a:b].tolist())))
    polys = [[list(m) for m in monos] for _ in range(cs.n_eq)]
    return system_from_terms(cs.n_eq, cs.n_var, cs.limbs, polys, cs.coeff.reshape(-1, 2, cs.limbs))


# ---------------------------------------------------------------------------
# Tracker inputs (NEXT-4): a total-degree homotopy with known start solutions
# ---------------------------------------------------------------------------

def total_degree_homotopy(n, limbs, seed):
    """Quadratic target system with a total-degree start system on one shared support.

    Support of every polynomial: all monomials of total degree <= 2 in n variables.  Target
    coefficients: unit-circle (seeded).  Start coefficients: gamma_i for x_i^2, -gamma_i for
    the constant, 0 elsewhere (g_i = gamma_i (x_i^2 - 1), gamma_i a seeded unit-circle
    constant: the "gamma trick" that keeps the paths regular for generic gamma).  Start
    solutions: the 2^n points of {+1, -1}^n, exact.  Returns (system with start coefficients,
    coeff_target, X_start [2^n][n][2][L])."""
    rng = np.random.Generator(np.random.PCG64(seed))
    monos = [[]] + [[(v, 1)] for v in range(n)]
    for a in range(n):
        for b in range(a, n):
            monos.append([(a, 2)] if a == b else [(a, 1), (b, 1)])
    M = len(monos)
    th_target = rng.uniform(0.0, 2.0 * math.pi, size=n * M)
    th_gamma = rng.uniform(0.0, 2.0 * math.pi, size=n)
    target = unit_circle_limbs(th_target, limbs).reshape(n * M, 2, limbs)
    gamma = unit_circle_limbs(th_gamma, limbs)
    start = np.zeros((n * M, 2, limbs))
    for i in range(n):
        j_sq = monos.index([(i, 2)])
        start[i * M + j_sq] = gamma[i]
        start[i * M + 0] = -gamma[i]
    s = system_from_terms(n, n, limbs, [[list(m) for m in monos] for _ in range(n)], start)
    X = np.zeros((2 ** n, n, 2, limbs))
    for k in range(2 ** n):
        for v in range(n):
            X[k, v, 0, 0] = -1.0 if (k >> v) & 1 else 1.0
    return s, target, X


def as_common(system, coeff_target=None):
    """A system whose polynomials all list the same terms in the same order, as a
    common-support system (CommonArrays) plus, if given, its target coefficients as the dense
    [n_eq][M][2][L] matrix.  Raises ValueError otherwise.  Host bookkeeping only."""
    terms0 = [fac for _, fac in system.terms(0)]
    M = len(terms0)
    for i in range(1, system.n_eq):
        if [fac for _, fac in system.terms(i)] != terms0:
            raise ValueError("polynomials do not share one support")
    mono_ptr, vi, ex = [0], [], []
    for fac in terms0:
        for v, a in fac:
            vi.append(v)
            ex.append(a)
        mono_ptr.append(len(vi))
    L = system.limbs
    c = CommonArrays(system.n_eq, system.n_var, L, np.asarray(mono_ptr, np.int64), np.asarray(vi, np.int32),
                     np.asarray(ex, np.int32), np.ascontiguousarray(system.coeff.reshape(system.n_eq, M, 2, L)))
    if coeff_target is None:
        return c
    return c, np.ascontiguousarray(np.asarray(coeff_target).reshape(system.n_eq, M, 2, L))
