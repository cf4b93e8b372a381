// NEXT-4: the predictor and the per-path bookkeeping of the path tracker
// (Alg. 1; the quadratic predictor of §5), for a batch of
// paths tracked side by side on one device.  The corrector is the Newton step of
// kernels_newton.cuh on the homotopy (NEXT-3); the step-size control runs on the host
// (phc.cu, phc_track_paths).
//
// History per path p (the paper's x*, x*_prev, x*_prev1 at t > t_prev > t_prev1):
//   t_hist [P][3][L]   real t of the three most recent ACCEPTED points, slot 0 newest
//   x_hist [P][3][n][2][L]
//   n_hist [P]         number of valid slots (1..3)
// Compact per-iteration buffers index the active paths a = 0..A-1 through idx[a] = p.
#pragma once
#include "arith.cuh"

namespace phc {

// Predictor (§5): t_new = min(t + lambda, 1) and, per coordinate independently, the value at
// t_new of the interpolant through the last h = min(n_hist, order + 1) accepted points:
//   h = 1: x0;  h = 2: secant  x0 + (t_new - t0) d01;
//   h = 3: parabola  x0 + (t_new - t0) (d01 + (t_new - t1) d012)   (Newton divided differences,
//          d01 = (x0 - x1) / (t0 - t1), d12 = (x1 - x2) / (t1 - t2), d012 = (d01 - d12) / (t0 - t2)).
// One thread per (active path, coordinate); coordinate 0 also writes t_new and the clip flag.
template <int L>
__global__ void predict_kernel(int n, int64_t A, const int32_t* __restrict__ idx, const int32_t* __restrict__ n_hist,
                               const double* __restrict__ t_hist, const double* __restrict__ x_hist,
                               const double* __restrict__ lam, const double* __restrict__ t_in, int order,
                               double* __restrict__ tc, double* __restrict__ xc, int32_t* __restrict__ clipped) {
  using P = Prec<L>;
  using C = typename P::C;
  using R = typename P::real;
  constexpr int cd = 2 * L;
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= A * n) return;
  const int64_t a = gid / n;
  const int i = (int)(gid % n);
  const int64_t p = idx ? idx[a] : a;
  const R t0 = P::rload(t_hist + (p * 3 + 0) * L);
  R tn;
  bool clip = false;
  if (t_in) {  // given target t (phc_predict_batch)
    tn = P::rload(t_in + a * L);
  } else {     // the tracker's step: t + lambda, clipped to 1
    tn = P::radd(t0, P::rfrom(lam[p]));
    const R over = P::rsub(tn, P::rfrom(1.0));
    clip = over.x[0] >= 0.0;
    if (clip) tn = P::rfrom(1.0);
  }
  const int h = min(n_hist[p], order + 1);
  const int64_t xs = (int64_t)n * cd;  // stride between history slots
  const double* xh = x_hist + p * 3 * xs + (int64_t)i * cd;
  const C x0 = cload<L>(xh);
  C out = x0;
  if (h >= 2) {
    const R t1 = P::rload(t_hist + (p * 3 + 1) * L);
    const C x1 = cload<L>(xh + xs);
    const R r01 = P::rdiv(P::rfrom(1.0), P::rsub(t0, t1));
    const C d01 = P::mul_real(P::sub(x0, x1), r01);
    C inner = d01;
    if (h >= 3) {
      const R t2 = P::rload(t_hist + (p * 3 + 2) * L);
      const C x2 = cload<L>(xh + 2 * xs);
      const C d12 = P::mul_real(P::sub(x1, x2), P::rdiv(P::rfrom(1.0), P::rsub(t1, t2)));
      const C d012 = P::mul_real(P::sub(d01, d12), P::rdiv(P::rfrom(1.0), P::rsub(t0, t2)));
      inner = P::add(d01, P::mul_real(d012, P::rsub(tn, t1)));
    }
    out = P::add(x0, P::mul_real(inner, P::rsub(tn, t0)));
  }
  cstore<L>(xc + (a * n + i) * cd, out);
  if (i == 0 && tc) {
    P::rstore(tc + a * L, tn);
    clipped[a] = clip ? 1 : 0;
  }
}

// Accept the corrected points of the active paths with accept[a] != 0: shift the history
// (slot 1 -> 2, 0 -> 1, corrected -> 0).  One thread per (active path, coordinate);
// coordinate 0 also shifts t and counts the slot.  Rejected paths keep their history
// bitwise (the step back of Alg. 1).
template <int L>
__global__ void accept_kernel(int n, int64_t A, const int32_t* __restrict__ idx, const int32_t* __restrict__ accept,
                              const double* __restrict__ tc, const double* __restrict__ xc, int32_t* __restrict__ n_hist,
                              double* __restrict__ t_hist, double* __restrict__ x_hist) {
  constexpr int cd = 2 * L;
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= A * n) return;
  const int64_t a = gid / n;
  if (!accept[a]) return;
  const int i = (int)(gid % n);
  const int64_t p = idx[a];
  const int64_t xs = (int64_t)n * cd;
  double* xh = x_hist + p * 3 * xs + (int64_t)i * cd;
  for (int c = 0; c < cd; ++c) {
    xh[2 * xs + c] = xh[xs + c];
    xh[xs + c] = xh[c];
    xh[c] = xc[(a * n + i) * cd + c];
  }
  if (i == 0) {
    double* th = t_hist + p * 3 * L;
    for (int c = 0; c < L; ++c) {
      th[2 * L + c] = th[L + c];
      th[L + c] = th[c];
      th[c] = tc[a * L + c];
    }
    n_hist[p] = min(n_hist[p] + 1, 3);
  }
}

// Step-size control, step back and stop criterion of Alg. 1 (reading T1) for the
// active paths of one tracker step, on the device (the host only looks at the statuses once
// per window of steps, phc_track_paths).  One thread per active path a = 0..A-1:
//   corrected at the first Newton iteration k whose residual res[k][a] <= tol (a singular
//   step or a non-finite residual before that fails the correction); accepted steps expand
//   lambda (capped at step_max) and finish the path when the predictor clipped t to 1;
//   rejected steps contract lambda and fail the path below step_min; max_steps caps the steps.
// Paths that stopped earlier in the window (stat != 0) are left untouched (acc = 0).
struct TrackCtl {
  double step_min, step_max, expand, contract, tol;
  int max_newton, max_steps;
};
__global__ void control_kernel(int64_t A, const int32_t* __restrict__ idx, const TrackCtl c,
                               const double* __restrict__ res, const int32_t* __restrict__ nst,
                               const int32_t* __restrict__ clipped, int32_t* __restrict__ acc,
                               int32_t* __restrict__ stat, double* __restrict__ lam, int64_t* __restrict__ steps,
                               int64_t* __restrict__ succ, int64_t* __restrict__ iters,
                               double* __restrict__ min_step, double* __restrict__ sum_step) {
  const int64_t a = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= A) return;
  const int64_t p = idx[a];
  if (stat[p] != 0) {
    acc[a] = 0;
    return;
  }
  bool conv = false, bad = false;
  int64_t it = 0;
  for (int k = 0; k < c.max_newton && !conv && !bad; ++k) {
    ++it;
    const double r = res[(int64_t)k * A + a];
    if (nst[(int64_t)k * A + a] != 0 || !isfinite(r))
      bad = true;
    else if (r <= c.tol)
      conv = true;
  }
  iters[p] += it;
  const int64_t sp = ++steps[p];
  const bool ok = conv && !bad;
  acc[a] = ok ? 1 : 0;
  int32_t st = 0;
  double l = lam[p];
  if (ok) {
    succ[p] += 1;
    min_step[p] = fmin(min_step[p], l);
    sum_step[p] += l;
    if (clipped[a]) st = 1;  // reached t = 1 with a successful correction there
    l = fmin(l * c.expand, c.step_max);
  } else {
    l *= c.contract;
    if (l < c.step_min) st = 2;
  }
  if (st == 0 && sp >= c.max_steps) st = 2;
  lam[p] = l;
  stat[p] = st;
}

// Start: slot 0 = the start solution at t = 0, one valid slot.
template <int L>
__global__ void track_init_kernel(int n, int64_t P_, const double* __restrict__ x, int32_t* __restrict__ n_hist,
                                  double* __restrict__ t_hist, double* __restrict__ x_hist) {
  constexpr int cd = 2 * L;
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= P_ * n) return;
  const int64_t p = gid / n;
  const int i = (int)(gid % n);
  for (int c = 0; c < cd; ++c) x_hist[(p * 3 * n + i) * cd + c] = x[(p * n + i) * cd + c];
  if (i == 0) {
    for (int c = 0; c < 3 * L; ++c) t_hist[p * 3 * L + c] = 0.0;
    n_hist[p] = 1;
  }
}

// End: x[p] = newest accepted point (slot 0); t_end[p] = its t.
template <int L>
__global__ void track_finish_kernel(int n, int64_t P_, const double* __restrict__ t_hist,
                                    const double* __restrict__ x_hist, double* __restrict__ x,
                                    double* __restrict__ t_end) {
  constexpr int cd = 2 * L;
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= P_ * n) return;
  const int64_t p = gid / n;
  const int i = (int)(gid % n);
  for (int c = 0; c < cd; ++c) x[(p * n + i) * cd + c] = x_hist[(p * 3 * n + i) * cd + c];
  if (i == 0 && t_end)
    for (int c = 0; c < L; ++c) t_end[p * L + c] = t_hist[p * 3 * L + c];
}

// Gather / scatter of points between full and compact (active-path) buffers.
__global__ void gather_rows_kernel(int64_t A, int64_t row, const int32_t* __restrict__ idx,
                                   const double* __restrict__ full, double* __restrict__ compact) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= A * row) return;
  const int64_t a = gid / row, c = gid % row;
  compact[gid] = full[(int64_t)idx[a] * row + c];
}
__global__ void scatter_rows_kernel(int64_t A, int64_t row, const int32_t* __restrict__ idx,
                                    const double* __restrict__ compact, double* __restrict__ full) {
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= A * row) return;
  const int64_t a = gid / row, c = gid % row;
  full[(int64_t)idx[a] * row + c] = compact[gid];
}

}  // namespace phc
