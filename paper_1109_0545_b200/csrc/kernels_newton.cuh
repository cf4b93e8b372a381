// NEXT-1: the rest of one Newton iteration of Alg. 2 (PAPER.md
// P:256-324) after the evaluation: residual ||F||, Gaussian elimination with
// partial pivoting on [J | -F] ("the largest number in the current column",
// P:342-343), back substitution and the update z := z + dz.
//
// Four eliminations, one result (same pivot rule, same operations per entry, same order;
// tested bitwise):
//  * newton_solve_kernel: one CTA per point, [J | -F] in shared memory (n (n+1) complex values
//    up to ~200 KB, real and imaginary planes); the paper's per-column pivot barrier
//     is one __syncthreads per column after a look-ahead warp, its row-per-thread
//    assignment a (row, column) grid-stride over the CTA;
//  * newton_warp_kernel: n <= 32, one warp per point (lane = row), no block barriers;
//  * the multi-kernel elimination (newton_*_kernel below): matrices beyond shared memory, two
//    launches per column over all points, the trailing update spread over many SMs;
//  * newton_coop_kernel: matrices beyond shared memory and few points, one persistent
//    cooperative launch (grid-wide barriers instead of kernel boundaries, one per column).
// Plus the loop control of Alg. 2 to tolerance (newton_exit_kernel, phc_newton_solve_batch).
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "arith.cuh"

namespace phc {

// Residual maximum that propagates NaN (fmax drops it): once an operand is NaN the result is
// NaN, so a non-finite F always reaches resid[] and the !isfinite(r) exits in phc.h fire.
__device__ __forceinline__ double nan_max(double a, double b) { return (b != b || b > a) ? b : a; }

// Phase timeline of the eliminations (diagnostic build -DPHC_NEWTON_TRACE=1, tools/newton_phase.cu):
// %globaltimer stamps of point 0 / CTA 0, thread 0: [0] solve kernel, [1] cooperative kernel;
// stamps 0 start, 1 matrix loaded, 2 elimination done, 3 back substitution done.
#ifndef PHC_NEWTON_TRACE
#define PHC_NEWTON_TRACE 0
#endif
#if PHC_NEWTON_TRACE
__device__ unsigned long long g_newton_phase[2][4];
// per column of the solve kernel: [0] start, [1] look-ahead update done, [2] pivot, reciprocal
// and multipliers done, [3] last trailing-update warp done (atomicMax), [4] after the barrier
__device__ unsigned long long g_newton_cols[128][5];
PHC_DEV unsigned long long ntime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define NEWTON_C(k, s, cond) \
  if ((cond) && (k) < 128) g_newton_cols[k][s] = ntime();
#define NEWTON_CMAX(k, s, cond) \
  if ((cond) && (k) < 128) atomicMax(&g_newton_cols[k][s], ntime());
#define NEWTON_T(kind, s, cond)                                               \
  if (cond) {                                                                 \
    unsigned long long t_;                                                    \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                    \
    g_newton_phase[kind][s] = t_;                                             \
  }
#else
#define NEWTON_T(kind, s, cond)
#define NEWTON_C(k, s, cond)
#define NEWTON_CMAX(k, s, cond)
#endif


// The pivot reciprocal (the serial step of every elimination column) computed by a whole
// warp: lane 0 divides the real part by |a|^2, lane 1 the imaginary part -- P::recip's own
// operations, so the value is bitwise P::recip(a) -- and every lane receives the result.  The
// two long divisions then run side by side instead of interleaved in one thread.
// Call with the full warp converged.
// The eliminations' arithmetic, shared by every kernel below so that all of them form the
// same operations in the same order.  PHC_NEWTON_LAZY: products and differences are lazy
// values (arith.cuh: DD (hi, lo) unnormalised, QD level expansions), renormalised where a
// value is divided by (the pivot) or leaves the elimination (dz); pivots are compared by the
// leading part of the value (the sum of its limbs in binary64).
#ifndef PHC_NEWTON_LAZY
#define PHC_NEWTON_LAZY 0
#endif
template <int L>
PHC_DEV typename Prec<L>::C emul(const typename Prec<L>::C& a, const typename Prec<L>::C& b) {
  if constexpr (PHC_NEWTON_LAZY) return Prec<L>::mul_lazy(a, b);
  else return Prec<L>::mul(a, b);
}
template <int L>
PHC_DEV typename Prec<L>::C efms(const typename Prec<L>::C& c, const typename Prec<L>::C& a,
                                 const typename Prec<L>::C& b) {
  if constexpr (PHC_NEWTON_LAZY) return Prec<L>::add_lazy(c, Prec<L>::neg(Prec<L>::mul_lazy(a, b)));
  else return Prec<L>::sub(c, Prec<L>::mul(a, b));
}
template <int L>
PHC_DEV typename Prec<L>::C enorm(const typename Prec<L>::C& a) {
  if constexpr (PHC_NEWTON_LAZY) return Prec<L>::norm(a);
  else return a;
}
template <int L>
PHC_DEV double ehi2(const typename Prec<L>::C& a) {
  if constexpr (PHC_NEWTON_LAZY) {
    double re = a.re.x[L - 1], im = a.im.x[L - 1];
#pragma unroll
    for (int i = L - 2; i >= 0; --i) {
      re += a.re.x[i];
      im += a.im.x[i];
    }
    return re * re + im * im;
  } else {
    return Prec<L>::abs2_hi(a);
  }
}
template <int L>
PHC_DEV typename Prec<L>::C recip_warp(const typename Prec<L>::C& a_in, int lane) {
  using P = Prec<L>;
  typename P::C r;
  const typename P::C a = enorm<L>(a_in);
  const typename P::real d = P::abs2(a);
  const typename P::real q = P::rdiv((lane & 1) ? a.im : a.re, d);
#pragma unroll
  for (int i = 0; i < L; ++i) {
    r.re.x[i] = __shfl_sync(0xffffffffu, q.x[i], 0);
    r.im.x[i] = -__shfl_sync(0xffffffffu, q.x[i], 1);
  }
  return r;
}

// Back substitution, row-scaled, the same in every elimination: with
// d_r = 1 / U[r][r] (the stored pivot reciprocals), one parallel pass forms
//   c_r = b_r d_r  and  N[r][j] = U[r][j] d_r  (r < j < n),
// then the sweep c_r -= N[r][j] x_j for j = n-1, ..., r+1 in that order, x_j = c_j once row j
// has received all its terms.  Its dependent chain is one efms per row (the column-oriented
// form had a product, an efms and two block barriers per row).
//
// sweep_warp: one warp, lane l holding rows l, l + 32, ... (R per lane, n <= 32 R) in registers,
// x_j broadcast by shuffles: no block barriers.  ldN(r, j) reads N[r][j], ldC(r) the scaled c_r.
template <int L, int R, class LdN, class LdC>
PHC_DEV void sweep_warp(int n, int lane, LdN ldN, LdC ldC, typename Prec<L>::C (&c)[R]) {
  using C = typename Prec<L>::C;
#pragma unroll
  for (int q = 0; q < R; ++q)
    if (lane + 32 * q < n) c[q] = ldC(lane + 32 * q);
  for (int j = n - 1; j >= 1; --j) {
    const int oq = j >> 5, ol = j & 31;
    C src = c[0];
#pragma unroll
    for (int q = 1; q < R; ++q)
      if (oq == q) src = c[q];
    C xj;
#pragma unroll
    for (int i = 0; i < L; ++i) {
      xj.re.x[i] = __shfl_sync(0xffffffffu, src.re.x[i], ol);
      xj.im.x[i] = __shfl_sync(0xffffffffu, src.im.x[i], ol);
    }
#pragma unroll
    for (int q = 0; q < R; ++q) {
      const int r = lane + 32 * q;
      if (r < j) c[q] = efms<L>(c[q], ldN(r, j), xj);
    }
  }
}

// Component h (0: real, 1: imaginary) of a complex product or update on its own lane.  With
// -i z = (z.im, -z.re) (exact), im(c - a b) = re((-i c) - a (-i b)) and im(a b) = re(a (-i b)):
// the real part of the same operation on rotated operands.  Every product in it pairs two
// negated factors or none, and round-to-nearest is sign-symmetric, so the component is bitwise
// the full operation's; the unused imaginary half is dead code after inlining.  Two lanes per
// entry halve the instructions a lane issues on the elimination's serial chain.
template <int L>
PHC_DEV typename Prec<L>::C rot_if(const typename Prec<L>::C& z, bool h) {
  typename Prec<L>::C r;
#pragma unroll
  for (int i = 0; i < L; ++i) {
    r.re.x[i] = h ? z.im.x[i] : z.re.x[i];
    r.im.x[i] = h ? -z.re.x[i] : z.im.x[i];
  }
  return r;
}
template <int L>
PHC_DEV typename Prec<L>::C cpart(const typename Prec<L>::real& x) {
  typename Prec<L>::C r;
  r.re = x;
  r.im = x;  // not read: only the real part of results built from it is used
  return r;
}
// sweep_warp with two lanes per row (lane t: row t / 2, component t & 1; R2 slots per lane,
// 2n <= 32 R2), bitwise sweep_warp's result.  ldC(r, h) reads component h of the scaled c_r.
template <int L, int R2, class LdN, class LdC>
PHC_DEV void sweep_warp2(int n, int lane, LdN ldN, LdC ldC, typename Prec<L>::real (&c)[R2]) {
  using C = typename Prec<L>::C;
  using real = typename Prec<L>::real;
#pragma unroll
  for (int q = 0; q < R2; ++q) {
    const int t = lane + 32 * q;
    if (t < 2 * n) c[q] = ldC(t >> 1, t & 1);
  }
  for (int j = n - 1; j >= 1; --j) {
    const int oq = (2 * j) >> 5, ol = (2 * j) & 31;  // x_j.re on lane ol, x_j.im on ol + 1
    real src = c[0];
#pragma unroll
    for (int q = 1; q < R2; ++q)
      if (oq == q) src = c[q];
    C xj;
#pragma unroll
    for (int i = 0; i < L; ++i) {
      xj.re.x[i] = __shfl_sync(0xffffffffu, src.x[i], ol);
      xj.im.x[i] = __shfl_sync(0xffffffffu, src.x[i], ol + 1);
    }
#pragma unroll
    for (int q = 0; q < R2; ++q) {
      const int t = lane + 32 * q, r = t >> 1;
      if (r < j) c[q] = efms<L>(cpart<L>(c[q]), ldN(r, j), rot_if<L>(xj, t & 1)).re;
    }
  }
}

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

// Complex entries kept as a real and an imaginary plane (the shared-memory eliminations):
// entry offset o (in doubles within a plane), L doubles per part, 16-byte accesses.
template <int L>
PHC_DEV typename Prec<L>::C plane_ld(const double* re, const double* im, size_t o) {
  typename Prec<L>::C v;
#pragma unroll
  for (int q = 0; q < L; q += 2) {
    const double2 x = *reinterpret_cast<const double2*>(re + o + q);
    const double2 y = *reinterpret_cast<const double2*>(im + o + q);
    v.re.x[q] = x.x;
    v.re.x[q + 1] = x.y;
    v.im.x[q] = y.x;
    v.im.x[q + 1] = y.y;
  }
  return v;
}
template <int L>
PHC_DEV void plane_st(double* re, double* im, size_t o, const typename Prec<L>::C& v) {
#pragma unroll
  for (int q = 0; q < L; q += 2) {
    *reinterpret_cast<double2*>(re + o + q) = make_double2(v.re.x[q], v.re.x[q + 1]);
    *reinterpret_cast<double2*>(im + o + q) = make_double2(v.im.x[q], v.im.x[q + 1]);
  }
}

// Shared memory of newton_solve_kernel: [J | -F], the pivot reciprocals, two row permutations.
__host__ __device__ inline size_t solve_smem_bytes(int n, int L) {
  return ((size_t)n * (n + 1) + n) * 2 * L * sizeof(double) + (size_t)2 * n * sizeof(int);
}

// One CTA per point, [J | -F] in shared memory, one block barrier per column.  Rows are
// addressed through a permutation (row exchanges swap two entries, rows are not moved), kept
// twice: warps 1.. run the trailing update of step k through `cur` while warp 0 -- the
// look-ahead -- updates column k+1, finds its pivot, writes the exchanged permutation to
// `nxt`, forms the pivot reciprocal (recip_warp) and the multipliers of column k+1; then one
// __syncthreads and the buffers swap roles.  The look-ahead chain is the critical path of a
// column, so the update runs on the warps that do not share warp 0's scheduler (warp w issues
// on SMSP w % 4).  Same pivot choices and per-entry operations, in the same order, as the
// other eliminations (bitwise equal steps, tested).
template <int L>
__global__ void __launch_bounds__(512) newton_solve_kernel(const NewtonArgs a) {
  using P = Prec<L>;
  using C = typename P::C;
  extern __shared__ __align__(16) double nsm[];
  __shared__ double red_v[32];
  __shared__ int red_i[32];
  // s_bad[c & 1] = 1 when pivot column c is zero.  Double-buffered: warp 0 writes column
  // k + 1's slot during iteration k while the other warps may still be reading column k's
  // slot in the loop condition (one slot would let them leave the loop one barrier early)
  __shared__ int s_bad[2];
  const int64_t p = blockIdx.x;
  if (p >= a.n_points) return;
  const int n = a.n, cols = n + 1, cd = 2 * L;
  const int tid = threadIdx.x, T = blockDim.x, lane = tid & 31, wid = tid >> 5, nwarp = T >> 5;
  // [J | -F] as two planes, real parts then imaginary parts ([n][n+1][L] each): the lanes of
  // a warp read consecutive entries of a row, 16-byte DD parts at a 16-byte stride, so a
  // quarter-warp's LDS.128 is one conflict-free wavefront (the interleaved [re][im] layout
  // put two lanes on each bank: 46% of the wavefronts were conflicts)
  double* Mre = nsm;
  double* Mim = Mre + (size_t)n * cols * L;
  double* invd = Mim + (size_t)n * cols * L;  // n pivot reciprocals after the matrix
  int* pbuf = reinterpret_cast<int*>(invd + (size_t)n * cd);  // [2][n] row permutations
  auto ldE = [&](int r, int c) { return plane_ld<L>(Mre, Mim, ((size_t)r * cols + c) * L); };
  auto stE = [&](int r, int c, const C& v) { plane_st<L>(Mre, Mim, ((size_t)r * cols + c) * L, v); };
  auto st_part = [&](int r, int c, int h, const typename P::real& v) {
    double* q = (h ? Mim : Mre) + ((size_t)r * cols + c) * L;
#pragma unroll
    for (int i = 0; i < L; i += 2) *reinterpret_cast<double2*>(q + i) = make_double2(v.x[i], v.x[i + 1]);
  };
  auto ld_part = [&](int r, int c, int h) {
    const double* q = (h ? Mim : Mre) + ((size_t)r * cols + c) * L;
    typename P::real v;
#pragma unroll
    for (int i = 0; i < L; i += 2) {
      const double2 x = *reinterpret_cast<const double2*>(q + i);
      v.x[i] = x.x;
      v.x[i + 1] = x.y;
    }
    return v;
  };
  NEWTON_T(0, 0, p == 0 && tid == 0)
  const double* Fp = a.F + (size_t)p * n * cd;
  const double* Jp = a.J + (size_t)p * n * n * cd;
  // load [J | -F]; residual max_i |F_i|; identity permutation
  double rmax = 0.0;
  for (int e = tid; e < n * cols; e += T) {
    const int i = e / cols, j = e % cols;
    if (j < n) {
      stE(i, j, cload<L>(Jp + ((size_t)i * n + j) * cd));
    } else {
      const C f = cload<L>(Fp + (size_t)i * cd);
      rmax = nan_max(rmax, sqrt(P::abs2_hi(f)));
      stE(i, j, P::neg(f));
    }
  }
  for (int i = tid; i < n; i += T) pbuf[i] = i;
  for (int o = 16; o; o >>= 1) rmax = nan_max(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
  if (lane == 0) red_v[wid] = rmax;
  if (tid == 0) s_bad[0] = s_bad[1] = 0;
  __syncthreads();
  if (tid == 0) {
    double r = 0.0;
    for (int w = 0; w < nwarp; ++w) r = nan_max(r, red_v[w]);
    a.resid[p] = r;
  }
  // warp 0: pivot of column c among logical rows c.. of `src`, exchanged permutation to `dst`,
  // reciprocal, multipliers of column c (rows > c).  False when the column is zero.
  auto pivot_column = [&](const int* src, int* dst, int c) -> bool {
    double best = -1.0;
    int bi = n;
    for (int i = c + lane; i < n; i += 32) {
      const double v = ehi2<L>(ldE(src[i], c));
      if (v > best) { best = v; bi = i; }
    }
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
    }
    if (!(best > 0.0)) return false;
    for (int i = lane; i < n; i += 32) dst[i] = (i == c) ? src[bi] : (i == bi ? src[c] : src[i]);
    __syncwarp();
    const C inv = recip_warp<L>(ldE(dst[c], c), lane);
    if (lane == 0) sstore<L>(invd + (size_t)c * cd, inv);
    for (int i = c + 1 + lane; i < n; i += 32) stE(dst[i], c, emul<L>(ldE(dst[i], c), inv));
    return true;
  };
  NEWTON_T(0, 1, p == 0 && tid == 0)
  int cur = 0;  // pbuf + cur * n: the permutation after the exchanges of columns < k + 1
  if (wid == 0 && !pivot_column(pbuf, pbuf + n, 0) && lane == 0) s_bad[0] = 1;
  __syncthreads();
  cur = 1;
  for (int k = 0; k < n - 1 && !s_bad[k & 1]; ++k) {
    const int* pc = pbuf + cur * n;
    int* pn = pbuf + (cur ^ 1) * n;
    NEWTON_C(k, 0, p == 0 && tid == 0)
    if (wid == 0) {
      // look-ahead: column k+1 of the rows below k, then its pivot, exchange, multipliers
      if constexpr (L == 4) {
        // QD: one component per lane (rot_if; measured 1.14 -> 1.00 us per column for c3;
        // DD lost 0.07 us per column this way and keeps one entry per lane)
        const C pkh = rot_if<L>(ldE(pc[k], k + 1), lane & 1);
        for (int t0 = 0; t0 < 2 * (n - k - 1); t0 += 32) {
          const int t = t0 + lane, i = k + 1 + (t >> 1), h = t & 1;
          typename P::real v;
          if (i < n) v = efms<L>(cpart<L>(ld_part(pc[i], k + 1, h)), ldE(pc[i], k), pkh).re;
          __syncwarp();  // the pair's loads of the entry precede its stores
          if (i < n) st_part(pc[i], k + 1, h, v);
        }
      } else {
        const C pk = ldE(pc[k], k + 1);
        for (int i = k + 1 + lane; i < n; i += 32)
          stE(pc[i], k + 1, efms<L>(ldE(pc[i], k + 1), ldE(pc[i], k), pk));
      }
      __syncwarp();
      NEWTON_C(k, 1, p == 0 && lane == 0)
      if (!pivot_column(pc, pn, k + 1) && lane == 0) s_bad[(k + 1) & 1] = 1;
      NEWTON_C(k, 2, p == 0 && lane == 0)
    } else if ((wid & 3) != 0 || nwarp <= 4) {
      // trailing update M[i][j] -= l_i M[k][j], i > k, j > k + 1, off warp 0's SMSP
      const int worker = (nwarp > 4) ? (wid >> 2) * 3 + (wid & 3) - 1 : wid - 1;
      const int nworker = (nwarp > 4) ? (nwarp >> 2) * 3 : nwarp - 1;
      const int rows = n - k - 1, ucols = cols - k - 2;
      const int pr = pc[k];
      for (int e = worker * 32 + lane; e < rows * ucols; e += nworker * 32) {
        const int i = k + 1 + e / ucols, j = k + 2 + e % ucols;
        const int r = pc[i];
        stE(r, j, efms<L>(ldE(r, j), ldE(r, k), ldE(pr, j)));
      }
      NEWTON_CMAX(k, 3, p == 0 && lane == 0)
    }
    __syncthreads();
    NEWTON_C(k, 4, p == 0 && tid == 0)
    cur ^= 1;
  }
  if (s_bad[0] | s_bad[1]) {
    if (tid == 0) a.status[p] = 1;
    for (int e = tid; e < n; e += T)
      cstore<L>(a.Xnew + ((size_t)p * n + e) * cd, cload_rw<L>(a.X + ((size_t)p * n + e) * cd));
    return;
  }
  NEWTON_T(0, 2, p == 0 && tid == 0)
  // back substitution (row-scaled, sweep_warp above): c_r = b_r d_r, N[r][j] = U[r][j] d_r
  // in place, then warp 0 sweeps with the rows in registers
  const int* pf = pbuf + cur * n;
  for (int e = tid; e < n * cols; e += T) {
    const int r = e / cols, j = e % cols;
    if (j > r) stE(pf[r], j, emul<L>(ldE(pf[r], j), sload<L>(invd + (size_t)r * cd)));
  }
  __syncthreads();
  // QD: half-rows per lane (n <= 55 fits 200 KB of shared memory; c3 sweep 51 -> 45 us);
  // DD: whole rows (n <= 78)
  if constexpr (L == 2) {
    constexpr int R = 3;
    PHC_CHECK(n <= 32 * R);
    if (wid == 0) {
      C c[R];
      sweep_warp<L, R>(n, lane, [&](int r, int j) { return ldE(pf[r], j); }, [&](int r) { return ldE(pf[r], n); }, c);
      NEWTON_T(0, 3, p == 0 && tid == 0)
#pragma unroll
      for (int q = 0; q < R; ++q) {
        const int e = lane + 32 * q;
        if (e < n) {
          const double* xp = a.X + ((size_t)p * n + e) * cd;
          cstore<L>(a.Xnew + ((size_t)p * n + e) * cd, P::add(cload_rw<L>(xp), enorm<L>(c[q])));
        }
      }
    }
  } else if (wid == 0) {
    constexpr int R2 = 4;
    PHC_CHECK(2 * n <= 32 * R2);
    typename P::real c[R2];
    sweep_warp2<L, R2>(n, lane, [&](int r, int j) { return ldE(pf[r], j); },
                       [&](int r, int h) { return ld_part(pf[r], n, h); }, c);
    NEWTON_T(0, 3, p == 0 && tid == 0)
    // z := z + dz, one component per lane
#pragma unroll
    for (int q = 0; q < R2; ++q) {
      const int t = lane + 32 * q, e = t >> 1, h = t & 1;
      if (e < n) {
        double* xo = a.Xnew + ((size_t)p * n + e) * cd + h * L;
        const double* xp = a.X + ((size_t)p * n + e) * cd + h * L;
        typename P::real xv;
#pragma unroll
        for (int i = 0; i < L; ++i) xv.x[i] = xp[i];
        const typename P::real v = P::add(cpart<L>(xv), enorm<L>(cpart<L>(c[q]))).re;
#pragma unroll
        for (int i = 0; i < L; ++i) xo[i] = v.x[i];
      }
    }
  }
  if (tid == 0) a.status[p] = 0;
}

// Alg. 2's loop control (phc_newton_solve_batch) after Newton iteration k (0-based) of all
// points: a point still running records the iteration, its residual and the updated point,
// and stops when the residual it tested passed (!(res > tol)), was not finite, or its
// Jacobian was singular, or when k was the last iteration.  One thread per (point, coordinate);
// coordinate 0 also writes the scalars.  The running flags are double-buffered by iteration
// parity (act_cur read by every thread of a point, act_next written by coordinate 0), so no
// thread of a point can see the flag its own iteration clears.
template <int L>
__global__ void newton_exit_kernel(int n, int64_t P_, int k, int max_it, double tol, const double* __restrict__ res,
                                   const int32_t* __restrict__ st, const double* __restrict__ xw,
                                   const int32_t* __restrict__ act_cur, int32_t* __restrict__ act_next,
                                   double* __restrict__ x_out, double* __restrict__ residual,
                                   int32_t* __restrict__ iterations, int32_t* __restrict__ status) {
  constexpr int cd = 2 * L;
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= P_ * n) return;
  const int64_t p = gid / n;
  const int i = (int)(gid % n);
  if (!act_cur[p]) {
    if (i == 0) act_next[p] = 0;
    return;
  }
  for (int c = 0; c < cd; ++c) x_out[(p * n + i) * cd + c] = xw[(p * n + i) * cd + c];
  if (i != 0) return;
  const double r = res[p];
  iterations[p] = k + 1;
  residual[p] = r;
  int32_t out = -1;  // -1: keep iterating
  if (st[p] != 0) out = 2;
  else if (!isfinite(r)) out = 1;
  else if (!(r > tol)) out = (r >= tol) ? 1 : 0;
  else if (k + 1 >= max_it) out = 1;
  if (out >= 0) status[p] = out;
  act_next[p] = out < 0 ? 1 : 0;
}
static __global__ void newton_solve_init_kernel(int64_t P_, int32_t* __restrict__ active, double* __restrict__ residual,
                                                int32_t* __restrict__ iterations, int32_t* __restrict__ status,
                                                double tol, int max_it) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P_) return;
  // parity-0 running flags: Alg. 2 enters its loop only while ||h|| = 1 > tol
  active[p] = (max_it > 0 && 1.0 > tol) ? 1 : 0;
  residual[p] = 1.0;                   // the paper's initial ||h|| := 1
  iterations[p] = 0;
  status[p] = (1.0 >= tol) ? 1 : 0;    // the value for max_it = 0 (fail := ||h|| >= tol)
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
  // the warp's [J | -F] as real and imaginary planes (as in newton_solve_kernel)
  double* Mre = wsm + (size_t)wib * n * cols * cd;
  double* Mim = Mre + (size_t)n * cols * L;
  auto ldE = [&](int r, int c) { return plane_ld<L>(Mre, Mim, ((size_t)r * cols + c) * L); };
  auto stE = [&](int r, int c, const C& v) { plane_st<L>(Mre, Mim, ((size_t)r * cols + c) * L, v); };
  const double* Fp = a.F + (size_t)p * n * cd;
  const double* Jp = a.J + (size_t)p * n * n * cd;
  // coalesced: consecutive lanes read consecutive entries of J
  for (int e = lane; e < n * n; e += 32) stE(e / n, e % n, cload<L>(Jp + (size_t)e * cd));
  double rmax = 0.0;
  if (lane < n) {
    const C f = cload<L>(Fp + (size_t)lane * cd);
    rmax = sqrt(P::abs2_hi(f));
    stE(lane, n, P::neg(f));
  }
  for (int o = 16; o; o >>= 1) rmax = nan_max(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
  if (lane == 0) a.resid[p] = rmax;
  __syncwarp();
  for (int k = 0; k < n; ++k) {
    double best = -1.0;
    int bi = n;
    if (lane >= k && lane < n) {
      best = ehi2<L>(ldE(lane, k));
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
        const C u = ldE(k, j), v = ldE(bi, j);
        stE(k, j, v);
        stE(bi, j, u);
      }
    __syncwarp();
    const C inv = recip_warp<L>(ldE(k, k), lane);
    if (lane > k && lane < n) stE(lane, k, emul<L>(ldE(lane, k), inv));
    __syncwarp();
    if (lane == 0) stE(k, k, inv);  // U[k][k] is not read again: its slot keeps d_k = 1 / U[k][k]
    // trailing update spread over the lanes by (row, column) pairs: ceil((n-k-1)(n-k) / 32)
    // entries per lane instead of a whole row of n-k entries
    const int w = n - k;  // columns k+1 .. n
    const int ne = (n - k - 1) * w;
    for (int e = lane; e < ne; e += 32) {
      const int i = k + 1 + e / w, j = k + 1 + e % w;
      stE(i, j, efms<L>(ldE(i, j), ldE(i, k), ldE(k, j)));
    }
    __syncwarp();
  }
  // back substitution, row-scaled as in newton_solve_kernel (d_r on the diagonal)
  for (int e = lane; e < n * cols; e += 32) {
    const int r = e / cols, j = e % cols;
    if (j > r) stE(r, j, emul<L>(ldE(r, j), ldE(r, r)));
  }
  __syncwarp();
  C c[1];
  sweep_warp<L, 1>(n, lane, [&](int r, int j) { return ldE(r, j); }, [&](int r) { return ldE(r, n); }, c);
  if (lane < n) {
    const double* xp = a.X + ((size_t)p * n + lane) * cd;
    cstore<L>(a.Xnew + ((size_t)p * n + lane) * cd, P::add(cload_rw<L>(xp), enorm<L>(c[0])));
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
      rmax = nan_max(rmax, sqrt(P::abs2_hi(f)));
      sstore<L>(M + (size_t)e * cd, P::neg(f));
    }
  }
  for (int o = 16; o; o >>= 1) rmax = nan_max(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
  if (lane == 0) red_v[wid] = rmax;
  __syncthreads();
  if (tid == 0) {
    double r = 0.0;
    for (int w = 0; w < nwarp; ++w) r = nan_max(r, red_v[w]);
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
    const double v = ehi2<L>(sload<L>(at(i, k)));
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
  if (wid == 0) {
    const C inv = recip_warp<L>(sload<L>(at(k, k)), lane);
    if (lane == 0) {
      sstore<L>(s_inv, inv);
      sstore<L>(invd + (size_t)k * cd, inv);
    }
  }
  __syncthreads();
  const C inv = sload<L>(s_inv);
  for (int i = k + 1 + tid; i < n; i += T) sstore<L>(at(i, k), emul<L>(sload<L>(at(i, k)), inv));
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
  sstore<L>(at(i, j), efms<L>(sload<L>(at(i, j)), sload<L>(at(i, k)), sload<L>(at(k, j))));
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
  // row-scaled back substitution (sweep_warp's operations and order): scale, then one block
  // barrier per row with c in column n
  for (int e = tid; e < n * cols; e += T) {
    const int r = e / cols, j = e % cols;
    if (j > r) sstore<L>(at(r, j), emul<L>(sload<L>(at(r, j)), sload<L>(invd + (size_t)r * cd)));
  }
  __syncthreads();
  for (int j = n - 1; j >= 1; --j) {
    const C xj = sload<L>(at(j, n));
    for (int r = tid; r < j; r += T) sstore<L>(at(r, n), efms<L>(sload<L>(at(r, n)), sload<L>(at(r, j)), xj));
    __syncthreads();
  }
  for (int e = tid; e < n; e += T) {
    const double* xp = a.X + ((size_t)p * n + e) * cd;
    cstore<L>(a.Xnew + ((size_t)p * n + e) * cd, P::add(cload_rw<L>(xp), enorm<L>(sload<L>(at(e, n)))));
  }
}

// ---------------------------------------------------------------------------------------
// Few points with matrices beyond shared memory (large QD single point: n = 256, 4.2 MB):
// one persistent cooperative launch of one CTA per SM per point, in place of the 2n launches
// of the multi-kernel path (whose ~10 us per launch were the cost: 4.9 ms for n = 256).
// Per column k, one grid-wide barrier:
//   CTA 0 (look-ahead): column k+1 of rows i > k updated, its pivot (largest leading-limb
//     modulus, ties to the lowest row), the row exchange (in the permutation perm_g: rows
//     are not moved), the pivot reciprocal (recip_warp) and the multipliers of column k+1;
//   CTAs 1..G-1: the trailing update of step k, rows i > k, columns j >= k+2.
// CTA 0's chain is the critical path, so its operands stay on chip: the updated column in
// shared memory (pivot search and reciprocal read it there), each thread's multipliers in
// registers for the next column's update (thread t owns logical rows c+1+t, c+1+t+T, ...
// of column c in both steps).  Rows are addressed through the permutation (the other CTAs
// take a snapshot after the barrier); the CTA kernel's row swaps move only columns that are
// read later, so the per-entry operations, their order and the pivot choices are those of
// newton_solve_kernel: bitwise the same step (tested).  Back substitution and update on CTA 0.
// ---------------------------------------------------------------------------------------
// complex load through L2 (ld.global.cg): the cooperative kernel's CTAs read entries other
// CTAs wrote before the last grid barrier, never a stale L1 line
template <int L>
PHC_DEV typename Prec<L>::C ldl2(const double* p) {
  typename Prec<L>::C v;
#pragma unroll
  for (int q = 0; q < L; q += 2) {
    const double2 r = __ldcg(reinterpret_cast<const double2*>(p + q));
    const double2 m = __ldcg(reinterpret_cast<const double2*>(p + L + q));
    v.re.x[q] = r.x;
    v.re.x[q + 1] = r.y;
    v.im.x[q] = m.x;
    v.im.x[q + 1] = m.y;
  }
  return v;
}
#ifndef PHC_COOP_TRACE
#define PHC_COOP_TRACE 0
#endif
#if PHC_COOP_TRACE
__device__ unsigned long long g_coop_trace[4096][6];
PHC_DEV unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define COOP_T(k, s) \
  if (tid == 0 && b == 0 && (k) < 4096) g_coop_trace[k][s] = gtime();
#else
#define COOP_T(k, s)
#endif
// c - a b and a b, as every elimination forms them
template <int L>
PHC_DEV typename Prec<L>::C cmul_c(const typename Prec<L>::C& a, const typename Prec<L>::C& b) {
  return emul<L>(a, b);
}
template <int L>
PHC_DEV typename Prec<L>::C cfms_c(const typename Prec<L>::C& c, const typename Prec<L>::C& a,
                                   const typename Prec<L>::C& b) {
  return efms<L>(c, a, b);
}
constexpr int kCoopThreads = 256;
constexpr int kCoopRows = 4;  // chain rows per thread of CTA 0: n <= 1 + 4 * 256
// shared memory of the cooperative kernel: colv, lmul [n][2L] + perm [n]
__host__ __device__ inline size_t coop_smem_bytes(int n, int L) {
  return (size_t)2 * n * 2 * L * sizeof(double) + (size_t)n * sizeof(int);
}
template <int L>
__global__ void __launch_bounds__(kCoopThreads) newton_coop_kernel(const NewtonArgs a,
                                                                   int32_t* __restrict__ perm_g,  // [2][n]
                                                                   double* __restrict__ red_g,
                                                                   int32_t* __restrict__ flag_g) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  using P = Prec<L>;
  using C = typename P::C;
  extern __shared__ __align__(16) double csm[];
  const int n = a.n, cols = n + 1, cd = 2 * L;
  // CTA 0's on-chip columns, indexed by PHYSICAL row: colv = the look-ahead column c (pivot
  // search, reciprocal, multipliers), lmul = the multipliers of column c
  double* colv = csm;
  double* lmul = colv + (size_t)n * cd;
  int* perm = reinterpret_cast<int*>(lmul + (size_t)n * cd);  // [n] row permutation
  __shared__ double red_v[32];
  __shared__ int red_i[32];
  __shared__ int s_bad;
  __shared__ int s_front;  // back substitution: lowest logical row whose x is published
  __shared__ __align__(16) double s_inv[2 * L];
  const int tid = threadIdx.x, T = blockDim.x, lane = tid & 31, wid = tid >> 5, nwarp = T >> 5;
  const int G = gridDim.x, b = blockIdx.x;
  auto cval = [&](const double* base, int ph) { return sload<L>(base + (size_t)ph * cd); };
  // CTA 0, warp 0: final argmax over the warps' candidates (ties to the lowest logical row),
  // exchange of logical rows c and the winner, pivot reciprocal.  Uniform across warp 0.
  auto pivot_and_recip = [&](double* invd, int c) {
    double best = lane < nwarp ? red_v[lane] : -1.0;
    int bi = lane < nwarp ? red_i[lane] : n;
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
    }
    if (!(best > 0.0)) {
      if (lane == 0) {
        s_bad = 1;
        flag_g[c & 1] = 1;  // column c's slot: see the read in the k loop
      }
      return;
    }
    PHC_CHECK(bi >= c && bi < n);
    const int ph = perm[bi];  // physical pivot row (all lanes read before lane 0 swaps)
    __syncwarp();
    const C inv = recip_warp<L>(cval(colv, ph), lane);
    if (lane == 0) {
      perm[bi] = perm[c];
      perm[c] = ph;
      sstore<L>(s_inv, inv);
      sstore<L>(invd + (size_t)c * cd, inv);
    }
  };
  // CTA 0: multipliers l_i = colv / pivot of the logical rows i > c (after the exchange)
  auto multipliers = [&](double* M, int c) {
    const C inv = sload<L>(s_inv);
    for (int i = c + 1 + tid; i < n; i += T) {
      const int ph = perm[i];
      const C l = cmul_c<L>(cval(colv, ph), inv);
      sstore<L>(lmul + (size_t)ph * cd, l);
      sstore<L>(M + ((size_t)ph * cols + c) * cd, l);
    }
    // the permutation after exchange c goes to buffer c & 1: the other CTAs read buffer
    // (c - 1) & 1 while this one is written (no torn snapshot)
    for (int i = tid; i < n; i += T) perm_g[(size_t)(c & 1) * n + i] = perm[i];
  };
  // per-thread candidate -> warp argmax -> red_v / red_i
  auto warp_candidates = [&](double best, int bi) {
    for (int o = 16; o; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
    }
    if (lane == 0) { red_v[wid] = best; red_i[wid] = bi; }
  };
  for (int64_t p = 0; p < a.n_points; ++p) {
    double* M = a.Mg + (size_t)p * ((size_t)n * cols + n) * cd;
    NEWTON_T(1, 0, p == 0 && b == 0 && tid == 0)
    double* invd = M + (size_t)n * cols * cd;
    auto at = [&](int r, int c) { return M + ((size_t)r * cols + c) * cd; };
    const double* Fp = a.F + (size_t)p * n * cd;
    const double* Jp = a.J + (size_t)p * n * n * cd;
    // [J | -F] and the residual, spread over the grid
    double rmax = 0.0;
    for (int64_t e = (int64_t)b * T + tid; e < (int64_t)n * cols; e += (int64_t)G * T) {
      const int i = (int)(e / cols), j = (int)(e % cols);
      if (j < n) {
        sstore<L>(at(i, j), cload<L>(Jp + ((size_t)i * n + j) * cd));
      } else {
        const C f = cload<L>(Fp + (size_t)i * cd);
        rmax = nan_max(rmax, sqrt(P::abs2_hi(f)));
        sstore<L>(at(i, j), P::neg(f));
      }
    }
    for (int o = 16; o; o >>= 1) rmax = nan_max(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
    if (lane == 0) red_v[wid] = rmax;
    __syncthreads();
    if (tid == 0) {
      double r = 0.0;
      for (int w = 0; w < nwarp; ++w) r = nan_max(r, red_v[w]);
      red_g[b] = r;
      s_bad = 0;
    }
    if (b == 0 && tid == 0) flag_g[0] = flag_g[1] = 0;
    grid.sync();
    if (b == 0) {
      // column 0: pivot, exchange, reciprocal, multipliers; column 1 kept for step 0
      if (tid == 0) {
        double r = 0.0;
        for (int q = 0; q < G; ++q) r = nan_max(r, __ldcg(red_g + q));
        a.resid[p] = r;
      }
      double best = -1.0;
      int bi = n;
      for (int i = tid; i < n; i += T) {
        perm[i] = i;
        const C v = ldl2<L>(at(i, 0));
        sstore<L>(colv + (size_t)i * cd, v);
        const double m = ehi2<L>(v);
        if (m > best) { best = m; bi = i; }
      }
      warp_candidates(best, bi);
      __syncthreads();
      if (wid == 0) pivot_and_recip(invd, 0);
      __syncthreads();
      if (!s_bad) multipliers(M, 0);
    }
    grid.sync();
    NEWTON_T(1, 1, p == 0 && b == 0 && tid == 0)
    for (int k = 0; k < n - 1; ++k) {
      if (b == 0) {
        if (s_bad) break;
        COOP_T(k, 0)
        // look-ahead column k+1: v = M[i][k+1] - l_i u_k (u_k = column k+1 of pivot row k)
        const C uk = ldl2<L>(at(perm[k], k + 1));
        double best = -1.0;
        int bi = n;
#pragma unroll
        for (int q = 0; q < kCoopRows; ++q) {
          const int i = k + 1 + tid + q * T;
          if (i < n) {
            const int ph = perm[i];
            const C v = cfms_c<L>(ldl2<L>(at(ph, k + 1)), cval(lmul, ph), uk);
            sstore<L>(colv + (size_t)ph * cd, v);
            const double m = ehi2<L>(v);
            if (m > best) { best = m; bi = i; }
          }
        }
        warp_candidates(best, bi);
        __syncthreads();
        COOP_T(k, 1)
        if (wid == 0) pivot_and_recip(invd, k + 1);
        __syncthreads();
        COOP_T(k, 2)
        if (!s_bad) multipliers(M, k + 1);
        COOP_T(k, 3)
      } else {
        // column k's pivot status, written by CTA 0 before the last grid barrier.  Column k+1's
        // status goes to the other slot during this iteration, so an early write cannot make
        // this CTA leave the loop one grid barrier before CTA 0 (barrier counts would diverge)
        if (tid == 0) s_bad = __ldcg(flag_g + (k & 1));
        __syncthreads();
        if (s_bad) break;  // grid-uniform
        for (int i = tid; i < n; i += T) {
          perm[i] = __ldcg(perm_g + (size_t)(k & 1) * n + i);
          PHC_CHECK(perm[i] >= 0 && perm[i] < n);
        }
        __syncthreads();
        // trailing update of step k: rows i > k, columns j >= k + 2 (CTA 0 takes k+1)
        const int rows = n - k - 1, ucols = cols - k - 2;
        const int64_t ne = ucols > 0 ? (int64_t)rows * ucols : 0;
        const double* prow = at(perm[k], 0);
        for (int64_t e = (int64_t)(b - 1) * T + tid; e < ne; e += (int64_t)(G - 1) * T) {
          const int i = k + 1 + (int)(e / ucols), j = k + 2 + (int)(e % ucols);
          double* rw = at(perm[i], 0);
          sstore<L>(rw + (size_t)j * cd, cfms_c<L>(ldl2<L>(rw + (size_t)j * cd), ldl2<L>(rw + (size_t)k * cd),
                                                   ldl2<L>(prow + (size_t)j * cd)));
        }
      }
      COOP_T(k, 4)
      grid.sync();
      COOP_T(k, 5)
    }
    NEWTON_T(1, 2, p == 0 && b == 0 && tid == 0)
    // singular or not, grid-uniform: every column's flag was set before a grid barrier
    __syncthreads();
    if (tid == 0) s_bad = __ldcg(flag_g) | __ldcg(flag_g + 1);
    __syncthreads();
    if (s_bad) {
      if (b == 0) {
        if (tid == 0) a.status[p] = 1;
        for (int e = tid; e < n; e += T)
          cstore<L>(a.Xnew + ((size_t)p * n + e) * cd, cload_rw<L>(a.X + ((size_t)p * n + e) * cd));
      }
    } else {
      // row-scaled back substitution (sweep_warp's operations and order): the scaling pass
      // spread over the grid, then CTA 0 sweeps with c in shared memory, one barrier per row
      if (b != 0)
        for (int i = tid; i < n; i += T) perm[i] = __ldcg(perm_g + (size_t)((n - 1) & 1) * n + i);
      __syncthreads();
      for (int64_t e = (int64_t)b * T + tid; e < (int64_t)n * cols; e += (int64_t)G * T) {
        const int r = (int)(e / cols), j = (int)(e % cols);
        if (j > r) {
          double* q = at(perm[r], j);
          sstore<L>(q, cmul_c<L>(ldl2<L>(q), ldl2<L>(invd + (size_t)r * cd)));
        }
      }
      grid.sync();
      if (b == 0) {
        double* cv = colv;  // c by logical row
        if (n <= T) {
          // One row per thread, no block barrier per row: warp w holds rows [32w, 32w+32) in
          // registers, applies x_j of the rows above it as they are published (phase 1, j
          // descending), then sweeps its own rows with shuffles and publishes each x_j when it
          // is final (phase 2).  Only the critical row waits: the chain is one efms per row
          // plus one publication per warp.  Per row the same operations in the same order.
          volatile int* vfront = &s_front;  // x_j published <=> front <= j (decreasing)
          if (tid == 0) *vfront = n;
          const int r = tid, lo = wid * 32, hi = min(lo + 32, n) - 1;
          const int ph = r < n ? perm[r] : 0;
          C c = r < n ? ldl2<L>(at(ph, n)) : P::zero();
          __syncthreads();
          if (lo < n) {
            // N[r][j] is fetched one step ahead through both phases (L2 latency off the chain)
            C nx = (r < n - 1) ? ldl2<L>(at(ph, n - 1)) : P::zero();
            for (int j = n - 1; j > hi; --j) {  // phase 1: rows of the warps above
              if (lane == 0)
                while (*vfront > j) {
                }
              __syncwarp();
              __threadfence_block();
              const C xj = sload<L>(cv + (size_t)j * cd);
              const C nj = nx;
              if (r < j - 1) nx = ldl2<L>(at(ph, j - 1));
              if (r < n) c = cfms_c<L>(c, nj, xj);
            }
            for (int j = hi; j >= lo && j >= 1; --j) {  // phase 2: this warp's rows
              const C nj = nx;
              if (r < j - 1) nx = ldl2<L>(at(ph, j - 1));
              C xj;
#pragma unroll
              for (int i = 0; i < L; ++i) {
                xj.re.x[i] = __shfl_sync(0xffffffffu, c.re.x[i], j - lo);
                xj.im.x[i] = __shfl_sync(0xffffffffu, c.im.x[i], j - lo);
              }
              if (lane == j - lo) {
                sstore<L>(cv + (size_t)j * cd, c);
                __threadfence_block();
                *vfront = j;
              }
              if (r < j) c = cfms_c<L>(c, nj, xj);
            }
            if (lane == 0) {  // row lo is final
              sstore<L>(cv + (size_t)lo * cd, c);
              __threadfence_block();
              *vfront = lo;
            }
          }
          __syncthreads();
        } else {
          for (int r = tid; r < n; r += T) sstore<L>(cv + (size_t)r * cd, ldl2<L>(at(perm[r], n)));
          // N[tid][j] of the next step is fetched one step ahead (its L2 latency off the chain)
          const int ph0 = tid < n ? perm[tid] : 0;
          C nx = tid < n - 1 ? ldl2<L>(at(ph0, n - 1)) : P::zero();
          __syncthreads();
          for (int j = n - 1; j >= 1; --j) {
            const C xj = sload<L>(cv + (size_t)j * cd);
            const C nj = nx;
            if (tid < j - 1) nx = ldl2<L>(at(ph0, j - 1));
            if (tid < j) sstore<L>(cv + (size_t)tid * cd, cfms_c<L>(sload<L>(cv + (size_t)tid * cd), nj, xj));
            for (int r = tid + T; r < j; r += T)
              sstore<L>(cv + (size_t)r * cd, cfms_c<L>(sload<L>(cv + (size_t)r * cd), ldl2<L>(at(perm[r], j)), xj));
            __syncthreads();
          }
        }
        NEWTON_T(1, 3, p == 0 && tid == 0)
        for (int e = tid; e < n; e += T) {
          const double* xp = a.X + ((size_t)p * n + e) * cd;
          cstore<L>(a.Xnew + ((size_t)p * n + e) * cd, P::add(cload_rw<L>(xp), enorm<L>(sload<L>(cv + (size_t)e * cd))));
        }
        if (tid == 0) a.status[p] = 0;
      }
    }
    grid.sync();  // perm_g, red_g and flag_g are reused by the next point
  }
}

}  // namespace phc
