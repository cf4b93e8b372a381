// NEXT-1: the rest of one Newton iteration of Alg. 2 (PAPER.md
// P:256-324) after the evaluation: residual ||F||, Gaussian elimination with
// partial pivoting on [J | -F] ("the largest number in the current column",
// P:342-343), back substitution and the update z := z + dz.
//
// Three kernels, one result (same pivot rule, same operations per entry, same order):
//  * newton_solve_kernel: one CTA per point, [J | -F] in shared memory (n (n+1) complex values
//    up to ~200 KB); the paper's per-column pivot barrier is a __syncthreads, its
//    row-per-thread assignment a (row, column) grid-stride over the CTA;
//  * newton_warp_kernel: n <= 32, one warp per point (lane = row), no block barriers;
//  * the multi-kernel elimination (newton_*_kernel below): matrices beyond shared memory, two
//    launches per column over all points, the trailing update spread over many SMs.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "arith.cuh"

namespace phc {

struct NewtonArgs {
  const double* X;  // [P][n][2][L]
  const double* F;  // [P][n][2][L]
  const double* J;  // [P][n][n][2][L]
  double* Xnew;     // [P][n][2][L] (may alias X)
  double* resid;    // [P] max_i |F_i| (binary64)
  int32_t* status;  // [P] 0 = ok, 1 = singular (zero pivot column)
  double* Mg;       // global workspace [P][n][n+1][2][L] when the matrix does not fit shared memory
  int n;
  int64_t n_points;
};

template <int L>
__global__ void __launch_bounds__(512) newton_solve_kernel(const NewtonArgs a) {
  using P = Prec<L>;
  using C = typename P::C;
  extern __shared__ __align__(16) double nsm[];
  __shared__ double red_v[32];
  __shared__ int red_i[32];
  __shared__ int s_piv, s_bad;
  __shared__ __align__(16) double s_inv[2 * L];   // reciprocal of the current pivot
  __shared__ __align__(16) double s_inv2[2 * L];  // ... of the next column's (look-ahead)
  const int64_t p = blockIdx.x;
  if (p >= a.n_points) return;
  const int n = a.n, cols = n + 1, cd = 2 * L;
  const int tid = threadIdx.x, T = blockDim.x, lane = tid & 31, wid = tid >> 5, nwarp = T >> 5;
  double* M = nsm;
  double* invd = M + (size_t)n * cols * cd;  // n pivot reciprocals after the matrix
  auto at = [&](int i, int j) { return M + ((size_t)i * cols + j) * cd; };
  auto ldm = [&](int i, int j) { return sload<L>(at(i, j)); };  // generic: shared or global
  auto stm = [&](int i, int j, const C& v) { sstore<L>(at(i, j), v); };
  const double* Fp = a.F + (size_t)p * n * cd;
  const double* Jp = a.J + (size_t)p * n * n * cd;
  // load [J | -F]; residual max_i |F_i|
  double rmax = 0.0;
  for (int e = tid; e < n * cols; e += T) {
    const int i = e / cols, j = e % cols;
    if (j < n) {
      stm(i, j, cload<L>(Jp + ((size_t)i * n + j) * cd));
    } else {
      const C f = cload<L>(Fp + (size_t)i * cd);
      rmax = fmax(rmax, sqrt(P::abs2_hi(f)));
      stm(i, j, P::neg(f));
    }
  }
  for (int o = 16; o; o >>= 1) rmax = fmax(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
  if (lane == 0) red_v[wid] = rmax;
  if (tid == 0) s_bad = 0;
  __syncthreads();
  if (tid == 0) {
    double r = 0.0;
    for (int w = 0; w < nwarp; ++w) r = fmax(r, red_v[w]);
    a.resid[p] = r;
  }
  __syncthreads();
  // Elimination with partial pivoting and a one-column look-ahead: while warps 1.. update
  // the trailing columns k+2.. of step k, warp 0 updates column k+1, finds its pivot and
  // forms the pivot reciprocal, so the serial reciprocal overlaps the update (three block
  // barriers per column instead of six).  Same operations per entry as before.
  // column 0: pivot (block-wide), swap, reciprocal
  {
    double best = -1.0;
    int bi = n;
    for (int i = tid; i < n; i += T) {
      const double v = P::abs2_hi(ldm(i, 0));
      if (v > best) { best = v; bi = i; }
    }
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
    }
    if (lane == 0) { red_v[wid] = best; red_i[wid] = bi; }
    __syncthreads();
    if (tid == 0) {
      double b = -1.0;
      int ix = n;
      for (int w = 0; w < nwarp; ++w)
        if (red_v[w] > b || (red_v[w] == b && red_i[w] < ix)) { b = red_v[w]; ix = red_i[w]; }
      s_piv = ix;
      if (!(b > 0.0)) s_bad = 1;
    }
    __syncthreads();
    if (!s_bad) {
      const int pv = s_piv;
      if (pv != 0)
        for (int j = tid; j < cols; j += T) {
          const C u = ldm(0, j), v = ldm(pv, j);
          stm(0, j, v);
          stm(pv, j, u);
        }
      __syncthreads();
      if (tid == 0) {
        const C inv = P::recip(ldm(0, 0));
        sstore<L>(s_inv, inv);
        sstore<L>(invd, inv);
      }
      __syncthreads();
    }
  }
  for (int k = 0; k < n && !s_bad; ++k) {
    const C inv = sload<L>(s_inv);
    // multipliers l_i = M[i][k] / M[k][k], stored in column k
    for (int i = k + 1 + tid; i < n; i += T) stm(i, k, P::mul(ldm(i, k), inv));
    __syncthreads();  // (1)
    if (k == n - 1) break;
    if (wid == 0) {
      // look-ahead: column k+1, its pivot among rows k+1.., the pivot reciprocal
      for (int i = k + 1 + lane; i < n; i += 32)
        stm(i, k + 1, P::sub(ldm(i, k + 1), P::mul(ldm(i, k), ldm(k, k + 1))));
      __syncwarp();
      double best = -1.0;
      int bi = n;
      for (int i = k + 1 + lane; i < n; i += 32) {
        const double v = P::abs2_hi(ldm(i, k + 1));
        if (v > best) { best = v; bi = i; }
      }
      for (int o = 16; o; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
      }
      if (lane == 0) {
        if (!(best > 0.0)) {
          s_bad = 1;
        } else {
          s_piv = bi;
          sstore<L>(s_inv2, P::recip(ldm(bi, k + 1)));
        }
      }
    } else {
      // trailing update M[i][j] -= l_i M[k][j], i > k, j > k + 1
      const int rows = n - k - 1, ucols = cols - k - 2;
      for (int e = tid - 32; e < rows * ucols; e += T - 32) {
        const int i = k + 1 + e / ucols, j = k + 2 + e % ucols;
        stm(i, j, P::sub(ldm(i, j), P::mul(ldm(i, k), ldm(k, j))));
      }
    }
    __syncthreads();  // (2)
    if (s_bad) break;
    const int pv = s_piv;
    if (pv != k + 1)
      for (int j = k + 1 + tid; j < cols; j += T) {
        const C u = ldm(k + 1, j), v = ldm(pv, j);
        stm(k + 1, j, v);
        stm(pv, j, u);
      }
    if (tid == 0) {
      const C inv2 = sload<L>(s_inv2);
      sstore<L>(s_inv, inv2);
      sstore<L>(invd + (size_t)(k + 1) * cd, inv2);
    }
    __syncthreads();  // (3)
  }
  __syncthreads();
  if (s_bad) {
    if (tid == 0) a.status[p] = 1;
    for (int e = tid; e < n; e += T)
      cstore<L>(a.Xnew + ((size_t)p * n + e) * cd, cload_rw<L>(a.X + ((size_t)p * n + e) * cd));
    return;
  }
  // back substitution: x_i = M[i][n] / M[i][i], then M[r][n] -= M[r][i] x_i for r < i
  for (int i = n - 1; i >= 0; --i) {
    if (tid == 0) {
      const C inv = sload<L>(invd + (size_t)i * cd);
      stm(i, n, P::mul(ldm(i, n), inv));
    }
    __syncthreads();
    const C xi = ldm(i, n);
    for (int r = tid; r < i; r += T) stm(r, n, P::sub(ldm(r, n), P::mul(ldm(r, i), xi)));
    __syncthreads();
  }
  // z := z + dz
  for (int e = tid; e < n; e += T) {
    const double* xp = a.X + ((size_t)p * n + e) * cd;
    cstore<L>(a.Xnew + ((size_t)p * n + e) * cd, P::add(cload_rw<L>(xp), ldm(e, n)));
  }
  if (tid == 0) a.status[p] = 0;
}

// ---------------------------------------------------------------------------------------
// Small systems (n <= 32): one WARP per point, [J | -F] in the warp's slice of shared memory;
// no block barriers -- the pivot is a warp argmax over lane = row, every lane computes the
// pivot reciprocal itself (same inputs, same bits), the row swap is one column per lane, lane
// i forms multiplier i, and the trailing update is spread over the lanes by (row, column)
// pairs.  Same pivot rule, operations and order per entry as newton_solve_kernel, so the
// two kernels give bitwise identical steps; this one avoids ~5 block barriers per column
// (the tracker's corrector at n = 8: 26 us -> a few us per call).
// ---------------------------------------------------------------------------------------
template <int L>
__global__ void __launch_bounds__(128) newton_warp_kernel(const NewtonArgs a) {
  using P = Prec<L>;
  using C = typename P::C;
  extern __shared__ __align__(16) double wsm[];
  const int n = a.n, cols = n + 1, cd = 2 * L;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int64_t p = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib;
  if (p >= a.n_points) return;  // warp-uniform
  double* M = wsm + (size_t)wib * n * cols * cd;
  auto at = [&](int i, int j) { return M + ((size_t)i * cols + j) * cd; };
  const double* Fp = a.F + (size_t)p * n * cd;
  const double* Jp = a.J + (size_t)p * n * n * cd;
  double rmax = 0.0;
  if (lane < n) {
    for (int j = 0; j < n; ++j) sstore<L>(at(lane, j), cload<L>(Jp + ((size_t)lane * n + j) * cd));
    const C f = cload<L>(Fp + (size_t)lane * cd);
    rmax = sqrt(P::abs2_hi(f));
    sstore<L>(at(lane, n), P::neg(f));
  }
  for (int o = 16; o; o >>= 1) rmax = fmax(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
  if (lane == 0) a.resid[p] = rmax;
  __syncwarp();
  C inv_diag = P::zero();  // lane i keeps 1 / U[i][i] for the back substitution
  for (int k = 0; k < n; ++k) {
    double best = -1.0;
    int bi = n;
    if (lane >= k && lane < n) {
      best = P::abs2_hi(sload<L>(at(lane, k)));
      bi = lane;
    }
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
    }
    if (!(best > 0.0)) {  // zero pivot column: singular, x unchanged
      for (int e = lane; e < n; e += 32)
        cstore<L>(a.Xnew + ((size_t)p * n + e) * cd, cload_rw<L>(a.X + ((size_t)p * n + e) * cd));
      if (lane == 0) a.status[p] = 1;
      return;
    }
    if (bi != k)
      for (int j = k + lane; j < cols; j += 32) {
        const C u = sload<L>(at(k, j)), v = sload<L>(at(bi, j));
        sstore<L>(at(k, j), v);
        sstore<L>(at(bi, j), u);
      }
    __syncwarp();
    const C inv = P::recip(sload<L>(at(k, k)));
    if (lane == k) inv_diag = inv;
    if (lane > k && lane < n) sstore<L>(at(lane, k), P::mul(sload<L>(at(lane, k)), inv));
    __syncwarp();
    // trailing update spread over the lanes by (row, column) pairs: ceil((n-k-1)(n-k) / 32)
    // entries per lane instead of a whole row of n-k entries
    const int w = n - k;  // columns k+1 .. n
    const int ne = (n - k - 1) * w;
    for (int e = lane; e < ne; e += 32) {
      const int i = k + 1 + e / w, j = k + 1 + e % w;
      sstore<L>(at(i, j), P::sub(sload<L>(at(i, j)), P::mul(sload<L>(at(i, k)), sload<L>(at(k, j)))));
    }
    __syncwarp();
  }
  // back substitution, column oriented as in newton_solve_kernel
  for (int i = n - 1; i >= 0; --i) {
    if (lane == i) sstore<L>(at(i, n), P::mul(sload<L>(at(i, n)), inv_diag));
    __syncwarp();
    const C xi = sload<L>(at(i, n));
    if (lane < i) sstore<L>(at(lane, n), P::sub(sload<L>(at(lane, n)), P::mul(sload<L>(at(lane, i)), xi)));
    __syncwarp();
  }
  if (lane < n) {
    const double* xp = a.X + ((size_t)p * n + lane) * cd;
    cstore<L>(a.Xnew + ((size_t)p * n + lane) * cd, P::add(cload_rw<L>(xp), sload<L>(at(lane, n))));
  }
  if (lane == 0) a.status[p] = 0;
}

// ---------------------------------------------------------------------------------------
// Multi-kernel elimination for systems whose augmented matrix does not fit shared memory
// (e.g. n = 256 QD: 4.2 MB per point): every step k is two launches over all points of the
// chunk, so the trailing update of one point spreads over many SMs instead of one CTA.
//   newton_load_kernel      [J | -F] -> Mg, residual, status := 0          (one CTA per point)
//   newton_pivot_kernel<k>  pivot search in column k, row swap, pivot reciprocal, multipliers
//                           l_i = M[i][k] / M[k][k] stored in column k    (one CTA per point)
//   newton_update_kernel<k> M[i][j] -= l_i M[k][j], i > k, j > k          (many CTAs per point)
//   newton_backsub_kernel   back substitution and z := z + dz              (one CTA per point)
// Same pivot rule, operations and order per entry as newton_solve_kernel, so the two paths
// give the same result bitwise for a given matrix.
// ---------------------------------------------------------------------------------------
template <int L>
__global__ void __launch_bounds__(256) newton_load_kernel(const NewtonArgs a) {
  using P = Prec<L>;
  using C = typename P::C;
  __shared__ double red_v[32];
  const int64_t p = blockIdx.x;
  if (p >= a.n_points) return;
  const int n = a.n, cols = n + 1, cd = 2 * L;
  const int tid = threadIdx.x, T = blockDim.x, lane = tid & 31, wid = tid >> 5, nwarp = T >> 5;
  double* M = a.Mg + (size_t)p * ((size_t)n * cols + n) * cd;
  const double* Fp = a.F + (size_t)p * n * cd;
  const double* Jp = a.J + (size_t)p * n * n * cd;
  double rmax = 0.0;
  for (int e = tid; e < n * cols; e += T) {
    const int i = e / cols, j = e % cols;
    if (j < n) {
      sstore<L>(M + (size_t)e * cd, cload<L>(Jp + ((size_t)i * n + j) * cd));
    } else {
      const C f = cload<L>(Fp + (size_t)i * cd);
      rmax = fmax(rmax, sqrt(P::abs2_hi(f)));
      sstore<L>(M + (size_t)e * cd, P::neg(f));
    }
  }
  for (int o = 16; o; o >>= 1) rmax = fmax(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
  if (lane == 0) red_v[wid] = rmax;
  __syncthreads();
  if (tid == 0) {
    double r = 0.0;
    for (int w = 0; w < nwarp; ++w) r = fmax(r, red_v[w]);
    a.resid[p] = r;
    a.status[p] = 0;
  }
}

template <int L>
__global__ void __launch_bounds__(256) newton_pivot_kernel(const NewtonArgs a, int k) {
  using P = Prec<L>;
  using C = typename P::C;
  __shared__ double red_v[32];
  __shared__ int red_i[32];
  __shared__ int s_piv, s_bad;
  __shared__ __align__(16) double s_inv[2 * L];
  const int64_t p = blockIdx.x;
  if (p >= a.n_points || a.status[p]) return;
  const int n = a.n, cols = n + 1, cd = 2 * L;
  const int tid = threadIdx.x, T = blockDim.x, lane = tid & 31, wid = tid >> 5, nwarp = T >> 5;
  double* M = a.Mg + (size_t)p * ((size_t)n * cols + n) * cd;
  double* invd = M + (size_t)n * cols * cd;
  auto at = [&](int i, int j) { return M + ((size_t)i * cols + j) * cd; };
  double best = -1.0;
  int bi = n;
  for (int i = k + tid; i < n; i += T) {
    const double v = P::abs2_hi(sload<L>(at(i, k)));
    if (v > best) { best = v; bi = i; }
  }
  for (int o = 16; o; o >>= 1) {
    const double ov = __shfl_xor_sync(0xffffffffu, best, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
  }
  if (lane == 0) { red_v[wid] = best; red_i[wid] = bi; }
  __syncthreads();
  if (tid == 0) {
    double b = -1.0;
    int ix = n;
    for (int w = 0; w < nwarp; ++w)
      if (red_v[w] > b || (red_v[w] == b && red_i[w] < ix)) { b = red_v[w]; ix = red_i[w]; }
    s_piv = ix;
    s_bad = !(b > 0.0);
    if (s_bad) a.status[p] = 1;
  }
  __syncthreads();
  if (s_bad) return;
  const int pv = s_piv;
  if (pv != k)
    for (int j = k + tid; j < cols; j += T) {
      const C u = sload<L>(at(k, j)), v = sload<L>(at(pv, j));
      sstore<L>(at(k, j), v);
      sstore<L>(at(pv, j), u);
    }
  __syncthreads();
  if (tid == 0) {
    const C inv = P::recip(sload<L>(at(k, k)));
    sstore<L>(s_inv, inv);
    sstore<L>(invd + (size_t)k * cd, inv);
  }
  __syncthreads();
  const C inv = sload<L>(s_inv);
  for (int i = k + 1 + tid; i < n; i += T) sstore<L>(at(i, k), P::mul(sload<L>(at(i, k)), inv));
}

template <int L>
__global__ void __launch_bounds__(256) newton_update_kernel(const NewtonArgs a, int k) {
  using P = Prec<L>;
  const int64_t p = blockIdx.y;
  if (p >= a.n_points || a.status[p]) return;
  const int n = a.n, cols = n + 1, cd = 2 * L;
  const int ucols = cols - k - 1;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= (int64_t)(n - k - 1) * ucols) return;
  const int i = k + 1 + (int)(e / ucols), j = k + 1 + (int)(e % ucols);
  double* M = a.Mg + (size_t)p * ((size_t)n * cols + n) * cd;
  auto at = [&](int r, int c) { return M + ((size_t)r * cols + c) * cd; };
  sstore<L>(at(i, j), P::sub(sload<L>(at(i, j)), P::mul(sload<L>(at(i, k)), sload<L>(at(k, j)))));
}

template <int L>
__global__ void __launch_bounds__(256) newton_backsub_kernel(const NewtonArgs a) {
  using P = Prec<L>;
  using C = typename P::C;
  const int64_t p = blockIdx.x;
  if (p >= a.n_points) return;
  const int n = a.n, cols = n + 1, cd = 2 * L;
  const int tid = threadIdx.x, T = blockDim.x;
  if (a.status[p]) {
    for (int e = tid; e < n; e += T)
      cstore<L>(a.Xnew + ((size_t)p * n + e) * cd, cload_rw<L>(a.X + ((size_t)p * n + e) * cd));
    return;
  }
  double* M = a.Mg + (size_t)p * ((size_t)n * cols + n) * cd;
  double* invd = M + (size_t)n * cols * cd;
  auto at = [&](int r, int c) { return M + ((size_t)r * cols + c) * cd; };
  for (int i = n - 1; i >= 0; --i) {
    if (tid == 0) sstore<L>(at(i, n), P::mul(sload<L>(at(i, n)), sload<L>(invd + (size_t)i * cd)));
    __syncthreads();
    const C xi = sload<L>(at(i, n));
    for (int r = tid; r < i; r += T) sstore<L>(at(r, n), P::sub(sload<L>(at(r, n)), P::mul(sload<L>(at(r, i)), xi)));
    __syncthreads();
  }
  for (int e = tid; e < n; e += T) {
    const double* xp = a.X + ((size_t)p * n + e) * cd;
    cstore<L>(a.Xnew + ((size_t)p * n + e) * cd, P::add(cload_rw<L>(xp), sload<L>(at(e, n))));
  }
}

}  // namespace phc
