// Latency path for calls with few points (DESIGN.md §4
// "latency path"): the same evaluation as the fused block kernel, reorganised so that one
// point's work spreads over many warps with short dependency chains.
//
//  * One warp per TERM (not per block of 32 terms): lane l holds factor l of the term,
//    u_l = x^{a_l} and d_l = a_l x^{a_l - 1} from the power table (idle lanes u = 1, d = 0).
//  * The products of all factors but one (the paper's omega_m = psi_{m-1} phi_{k-m},
//    P:549-561) come from an inclusive prefix scan psi (with the coefficient folded into lane
//    0, reading C3) and an inclusive suffix scan phi over the lanes: 5 shuffle steps each,
//    then g_l = psi_{l-1} phi_{l+1} d_l.  Dependency path ~8 products instead of ~k; about
//    2x the products of the sequential chains (reading N2-3) -- the right trade only when the
//    GPU would otherwise be mostly idle.
//  * CTA (point p, polynomial i, split s) takes a fixed contiguous range of the terms of
//    f_i; warp w of the CTA takes terms w, w + W, ... of the range and adds its g_l into its
//    own shared-memory row (a term's variables are distinct: no conflicts within the warp);
//    the CTA sums the W rows in warp order.  With S > 1 splits the S partial rows go to a
//    global scratch and the last CTA of the polynomial to arrive (atomic counter) sums them
//    in split order.  The order is fixed
//    per system (W, S do not depend on the call), so results are bitwise reproducible.
//  * The power table of the point is built in shared memory by each CTA (one thread per
//    entry, binary powering).
#pragma once
#include "arith.cuh"

namespace phc {

struct ScanArgs {
  const int64_t* poly_ptr;
  const int64_t* term_ptr;
  const uint32_t* fac;  // var | exp << 16
  const double* coeff;
  const double* coeff2;  // homotopy target (NEXT-3) or nullptr
  const double* T;       // t per point when coeff2
  const double* X;
  double* F;
  double* J;
  double* part;  // S > 1: [P][n_eq][S][n_var + 1][2L] partial rows (col n_var = F)
  int* count;    // S > 1: [P][n_eq] arrival counters (zero between calls)
  int n_eq, n_var, E, S;
  int64_t n_points;
};

template <int L>
PHC_DEV typename Prec<L>::C cpow_scan(const typename Prec<L>::C& x, int e) {
  using P = Prec<L>;
  if (e == 0) return P::one();
  int top = 31 - __clz(e);
  typename P::C r = x;
  for (int b = top - 1; b >= 0; --b) {
    r = P::mul(r, r);
    if ((e >> b) & 1) r = P::mul(r, x);
  }
  return r;
}

// One out-of-line copy of the QD complex product: the per-term code calls it ~13 times, and
// inlining every call made the kernel 11k instructions, whose instruction-cache misses were the
// top stall (ncu: no_instruction 4.1 of 9 cycles per issue).  DD products stay inline.
template <int L>
__device__ __noinline__ typename Prec<L>::C cmul_ool(const typename Prec<L>::C a, const typename Prec<L>::C b) {
  return Prec<L>::mul(a, b);
}
// two independent products in one call (the psi and phi scans advance together: ILP)
template <int L>
struct CPair {
  typename Prec<L>::C a, b;
};
template <int L>
__device__ __noinline__ CPair<L> cmul2_ool(const typename Prec<L>::C a1, const typename Prec<L>::C b1,
                                           const typename Prec<L>::C a2, const typename Prec<L>::C b2) {
  CPair<L> r;
  r.a = Prec<L>::mul(a1, b1);
  r.b = Prec<L>::mul(a2, b2);
  return r;
}
// the same with lazy products (QD: the level sums, not renormalised; arith.cuh) for chains
// whose values only feed further products -- the segmented kernel renormalises what it stores
template <int L>
__device__ __noinline__ CPair<L> cmul2l_ool(const typename Prec<L>::C a1, const typename Prec<L>::C b1,
                                            const typename Prec<L>::C a2, const typename Prec<L>::C b2) {
  CPair<L> r;
  r.a = Prec<L>::mul_lazy(a1, b1);
  r.b = Prec<L>::mul_lazy(a2, b2);
  return r;
}
template <int L>
PHC_DEV typename Prec<L>::C smul(const typename Prec<L>::C& a, const typename Prec<L>::C& b) {
  if constexpr (L == 4) return cmul_ool<L>(a, b);
  else return Prec<L>::mul(a, b);
}

// partial rows written by other CTAs: read through L2 (ld.global.cg), never a stale L1 line
template <int L>
PHC_DEV typename Prec<L>::C cload_cg(const double* p) {
  typename Prec<L>::C v;
  double d[2 * L];
#pragma unroll
  for (int q = 0; q < 2 * L; q += 2) {
    double2 t = __ldcg(reinterpret_cast<const double2*>(p + q));
    d[q] = t.x;
    d[q + 1] = t.y;
  }
#pragma unroll
  for (int q = 0; q < L; ++q) { v.re.x[q] = d[q]; v.im.x[q] = d[L + q]; }
  return v;
}

template <int L>
PHC_DEV typename Prec<L>::C shfl_c(const typename Prec<L>::C& v, int delta, bool up) {
  typename Prec<L>::C r;
#pragma unroll
  for (int i = 0; i < L; ++i) {
    r.re.x[i] = up ? __shfl_up_sync(0xffffffffu, v.re.x[i], delta) : __shfl_down_sync(0xffffffffu, v.re.x[i], delta);
    r.im.x[i] = up ? __shfl_up_sync(0xffffffffu, v.im.x[i], delta) : __shfl_down_sync(0xffffffffu, v.im.x[i], delta);
  }
  return r;
}

template <int L>
__global__ void __launch_bounds__(256) poly_scan_kernel(const ScanArgs a) {
  using P = Prec<L>;
  using C = typename P::C;
  constexpr int cd = 2 * L;
  extern __shared__ __align__(16) double sm[];
  const int W = blockDim.x >> 5;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t cta = blockIdx.x;
  const int s = (int)(cta % a.S);
  const int i = (int)((cta / a.S) % a.n_eq);
  const int64_t p = cta / ((int64_t)a.S * a.n_eq);
  if (p >= a.n_points) return;
  const int twoE = 2 * a.E;
  double* pt = sm;                                         // [(n_var)][2E][cd]
  double* rows = sm + (size_t)a.n_var * twoE * cd;         // [W][n_var][cd]
  double* fpart = rows + (size_t)W * a.n_var * cd;         // [W][cd]
  // power table of point p: U[v][e-1] = x_v^e, Dd[v][e-1] = e x_v^(e-1)
  for (int idx = threadIdx.x; idx < a.n_var * a.E; idx += blockDim.x) {
    const int v = idx / a.E, e = idx % a.E + 1;
    const C x = cload<L>(a.X + (p * a.n_var + v) * cd);
    const C pm = cpow_scan<L>(x, e - 1);
    row_st<L>(pt, (size_t)v * twoE + e - 1, e == 1 ? x : P::mul(pm, x));
    row_st<L>(pt, (size_t)v * twoE + a.E + e - 1, e == 1 ? pm : P::mul_int(pm, (double)e));
  }
  for (int e = threadIdx.x; e < W * a.n_var * cd / 2; e += blockDim.x)
    reinterpret_cast<double2*>(rows)[e] = make_double2(0.0, 0.0);
  typename P::real tt = P::one().re, omt = P::one().re;
  if (a.coeff2) {
    tt = P::rload(a.T + p * L);
    omt = P::one_minus(tt);
  }
  __syncthreads();
  const int64_t t0 = a.poly_ptr[i], nt = a.poly_ptr[i + 1] - t0;
  const int64_t r0 = t0 + nt * s / a.S, r1 = t0 + nt * (s + 1) / a.S;  // this split's terms
  PHC_CHECK(nt >= 0 && r0 <= r1);
  C fsum = P::zero();
  for (int64_t t = r0 + warp; t < r1; t += W) {
    const int64_t f0 = a.term_ptr[t];
    const int k = (int)(a.term_ptr[t + 1] - f0);
    C c = cload<L>(a.coeff + t * cd);
    if (a.coeff2) c = P::add(P::mul_real(c, omt), P::mul_real(cload<L>(a.coeff2 + t * cd), tt));
    C u = P::one(), d = P::zero();
    int v = -1;
    if (lane < k) {
      const uint32_t w = a.fac[f0 + lane];
      v = (int)(w & 0xffffu);
      const int e = (int)((w >> 16) & 0xffu);
      PHC_CHECK(v < a.n_var && e >= 1 && e <= a.E);
      u = row_ld<L>(pt, (size_t)v * twoE + e - 1);
      d = row_ld<L>(pt, (size_t)v * twoE + a.E + e - 1);
    }
    // every lane multiplies (by 1 where the scan has no partner): no divergence around the
    // out-of-line product
    C pre = smul<L>(lane == 0 ? c : P::one(), u);  // psi with the coefficient folded in
    C suf = u;                                     // phi
#pragma unroll 1
    for (int off = 1; off < 32; off <<= 1) {
      const C x1 = shfl_c<L>(pre, off, true), x2 = shfl_c<L>(suf, off, false);
      if constexpr (L == 4) {
        const CPair<L> r = cmul2_ool<L>(lane >= off ? x1 : P::one(), pre, suf, lane + off < 32 ? x2 : P::one());
        pre = r.a;
        suf = r.b;
      } else {
        pre = P::mul(lane >= off ? x1 : P::one(), pre);
        suf = P::mul(suf, lane + off < 32 ? x2 : P::one());
      }
    }
    C before = shfl_c<L>(pre, 1, true), after = shfl_c<L>(suf, 1, false);
    if (lane == 0) before = c;
    if (lane == 31) after = P::one();
    const C g = smul<L>(smul<L>(before, d), after);
    if (lane < k) {  // entry index relative to `rows` (the swizzle depends on it)
      const size_t idx = (size_t)warp * a.n_var + v;
      row_st<L>(rows, idx, P::add(row_ld<L>(rows, idx), g));
    }
    const C y = shfl_c<L>(pre, 31, false);  // only lane 0 reads lane 31's full product
    if (k == 0) {                           // constant term: value c
      fsum = P::add(fsum, c);
    } else {
      fsum = P::add(fsum, y);
    }
    __syncwarp();
  }
  if (lane == 0) sstore<L>(fpart + (size_t)warp * cd, fsum);
  __syncthreads();
  // CTA totals in warp order; S == 1 writes F and J, S > 1 writes the partial row
  const bool direct = a.S == 1;
  for (int col = threadIdx.x; col <= a.n_var; col += blockDim.x) {
    C acc;
    if (col < a.n_var) {
      acc = row_ld<L>(rows, (size_t)col);
      for (int w = 1; w < W; ++w) acc = P::add(acc, row_ld<L>(rows, (size_t)w * a.n_var + col));
    } else {
      acc = sload<L>(fpart);
      for (int w = 1; w < W; ++w) acc = P::add(acc, sload<L>(fpart + (size_t)w * cd));
    }
    if (direct) {
      if (col < a.n_var)
        cstore<L>(a.J + ((p * a.n_eq + i) * (int64_t)a.n_var + col) * cd, acc);
      else
        cstore<L>(a.F + (p * a.n_eq + i) * cd, acc);
    } else {
      cstore<L>(a.part + (((p * a.n_eq + i) * a.S + s) * (int64_t)(a.n_var + 1) + col) * cd, acc);
    }
  }
  if (direct) return;
  // the last CTA of (p, i) to arrive sums the S partial rows in split order
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(a.count + p * a.n_eq + i, 1) == a.S - 1;
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const double* src = a.part + ((p * a.n_eq + i) * a.S) * (int64_t)(a.n_var + 1) * cd;
  for (int col = threadIdx.x; col <= a.n_var; col += blockDim.x) {
    C acc = cload_cg<L>(src + (size_t)col * cd);
    for (int q = 1; q < a.S; ++q) acc = P::add(acc, cload_cg<L>(src + ((size_t)q * (a.n_var + 1) + col) * cd));
    if (col < a.n_var)
      cstore<L>(a.J + ((p * a.n_eq + i) * (int64_t)a.n_var + col) * cd, acc);
    else
      cstore<L>(a.F + (p * a.n_eq + i) * cd, acc);
  }
  if (threadIdx.x == 0) a.count[p * a.n_eq + i] = 0;  // ready for the next call
}

// ---------------------------------------------------------------------------
// Segmented latency path (DESIGN.md §4 "segmented latency path"): the same evaluation as
// poly_scan_kernel with G lanes per term instead of 32, so a warp carries TPW = 32 / G terms
// and a lane up to two factors (k <= 2G).  Lane g of a term's segment holds factors 2g and
// 2g+1 (u_j = x^{a_j}, d_j = a_j x^{a_j - 1}; a missing factor is u = 1, d = 0):
//   T  = u_0 u_1,  Q_0 = d_0 u_1                                  (2 products)
//   M  = c * (product of T over the lanes before),  after = product of T over the lanes after
//        (inclusive scans of the shifted T: ceil(log2 G) steps of 2 products)
//   g_0 = M (Q_0 after),  g_1 = M (u_0 (d_1 after)),  y = M T   (6 products; y on the
//   segment's last lane is the term's value)
// The prefix/suffix products are the paper's psi/phi (§6) over the segment's
// lanes, the lane's own factors combined as in a two-factor Speelpenning product, the
// coefficient folded into the prefix (reading C3): 8 + 2 ceil(log2 G) products per lane in
// 4 + ceil(log2 G) dependent steps of two independent products each (c3: 16 products per lane
// in 8 steps, against 13 products on all 32 lanes per term for poly_scan_kernel).  The
// power table comes from block_power_table_kernel (global, one thread per entry, the primary
// of a programmatic dependent launch).  Accumulation: per (warp, term slot) shared-memory rows
// (the variables of one term are distinct; different slots own different rows), summed in a
// fixed order, then the S split partial rows as in poly_scan_kernel: bitwise reproducible for
// a given system.  Products and sums are lazy QD values (arith.cuh qd_dot2_parts /
// qd_add_levels, reading R4), renormalised when F and J are stored.
constexpr int kSegMaxWarps = 8;
// PHC_SEG_TRACE (diagnostic builds only): per-CTA %globaltimer stamps of the kernel's phases
// (start, table ready, products done, rows summed, end; then the SM id), read back with
// phc_debug_seg_trace
#ifndef PHC_SEG_TRACE
#define PHC_SEG_TRACE 0
#endif
#if PHC_SEG_TRACE
__device__ unsigned long long g_seg_trace[4096][8];
#define PHC_SEG_STAMP(k)                                                   \
  if (threadIdx.x == 0 && blockIdx.x < 4096) {                             \
    unsigned long long t_;                                                 \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_));                 \
    g_seg_trace[blockIdx.x][k] = t_;                                       \
  }
#else
#define PHC_SEG_STAMP(k)
#endif

template <int L>
PHC_DEV typename Prec<L>::C shfl_idx(const typename Prec<L>::C& v, int src) {
  typename Prec<L>::C r;
#pragma unroll
  for (int i = 0; i < L; ++i) {
    r.re.x[i] = __shfl_sync(0xffffffffu, v.re.x[i], src);
    r.im.x[i] = __shfl_sync(0xffffffffu, v.im.x[i], src);
  }
  return r;
}
// one out-of-line lazy complex addition (QD: level-wise, arith.cuh qd_add_levels; the kernel
// adds in several places, one copy of the code), and two independent ones in one call; sums are
// renormalised when they are stored
template <int L>
__device__ __noinline__ typename Prec<L>::C cadd_ool(const typename Prec<L>::C a, const typename Prec<L>::C b) {
  return Prec<L>::add_lazy(a, b);
}
template <int L>
__device__ __noinline__ CPair<L> cadd2_ool(const typename Prec<L>::C a1, const typename Prec<L>::C b1,
                                           const typename Prec<L>::C a2, const typename Prec<L>::C b2) {
  CPair<L> r;
  r.a = Prec<L>::add_lazy(a1, b1);
  r.b = Prec<L>::add_lazy(a2, b2);
  return r;
}
template <int L, int G>
__global__ void __launch_bounds__(kSegMaxWarps * 32) poly_seg_kernel(const ScanArgs a, const double* __restrict__ PT) {
  using P = Prec<L>;
  using C = typename P::C;
  constexpr int cd = 2 * L;
  constexpr int TPW = 32 / G;
  static_assert(G >= 2 && G <= 32, "segment shape");
  extern __shared__ __align__(16) double sm[];
  const int W = blockDim.x >> 5;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int slot = lane / G, g = lane - slot * G;
  const int64_t cta = blockIdx.x;
  const int s = (int)(cta % a.S);
  const int i = (int)((cta / a.S) % a.n_eq);
  const int64_t p = cta / ((int64_t)a.S * a.n_eq);
  if (p >= a.n_points) return;
  PHC_SEG_STAMP(0)
#if PHC_SEG_TRACE
  if (threadIdx.x == 0 && blockIdx.x < 4096) {
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    g_seg_trace[blockIdx.x][7] = smid;
  }
#endif
  const int nv = a.n_var;
  double* rows = sm;                                 // [W][TPW][n_var][cd]
  double* fpart = rows + (size_t)W * TPW * nv * cd;  // [W][TPW][cd]: the slots' term-value sums
  for (int e = threadIdx.x; e < W * TPW * (nv + 1) * cd / 2; e += blockDim.x)
    reinterpret_cast<double2*>(rows)[e] = make_double2(0.0, 0.0);
  typename P::real tt = P::one().re, omt = P::one().re;
  if (a.coeff2) {
    tt = P::rload(a.T + p * L);
    omt = P::one_minus(tt);
  }
  const int64_t t0 = a.poly_ptr[i], nt = a.poly_ptr[i + 1] - t0;
  const int64_t r0 = t0 + nt * s / a.S, r1 = t0 + nt * (s + 1) / a.S;  // this split's terms
  PHC_CHECK(nt >= 0 && r0 <= r1);
  __syncthreads();
  bool waited = false;
  const int twoE = 2 * a.E;
  const double* pt = PT + p * (int64_t)(nv + 1) * twoE * cd;
  const int dummy = nv * twoE;  // U = 1, D = 0
  bool first = true;  // the slot rows are still zero: store instead of add
  for (int64_t tb = r0 + (int64_t)warp * TPW; tb < r1; tb += (int64_t)W * TPW) {
    const int64_t t = tb + slot;
    const bool live = slot < TPW && t < r1;
    int k = 0;
    int64_t f0 = 0;
    C c = P::one();
    if (live) {
      f0 = a.term_ptr[t];
      k = (int)(a.term_ptr[t + 1] - f0);
      c = cload<L>(a.coeff + t * cd);
      if (a.coeff2) c = P::add(P::mul_real(c, omt), P::mul_real(cload<L>(a.coeff2 + t * cd), tt));
    }
    PHC_CHECK(k <= 2 * G);
    const int nf = live ? max(0, min(2, k - 2 * g)) : 0;
    int eu[2], var[2];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      eu[q] = dummy;
      var[q] = -1;
      if (q < nf) {
        const uint32_t w = a.fac[f0 + 2 * g + q];
        const int v = (int)(w & 0xffffu), e = (int)((w >> 16) & 0xffu);
        PHC_CHECK(v < nv && e >= 1 && e <= a.E);
        eu[q] = v * twoE + e - 1;
        var[q] = v;
      }
    }
    if (!waited) {
      // the power table of the primary kernel is complete and visible from here on (the term's
      // words and coefficient above are loaded while it runs)
      asm volatile("griddepcontrol.wait;" ::: "memory");
      waited = true;
      PHC_SEG_STAMP(1)
    }
    const C u0 = cload<L>(pt + (size_t)eu[0] * cd), u1 = cload<L>(pt + (size_t)eu[1] * cd);
    const C d0 = cload<L>(pt + (size_t)(eu[0] + a.E) * cd), d1 = cload<L>(pt + (size_t)(eu[1] + a.E) * cd);
    // every product goes through the one out-of-line (lazy) pair product: its code (~12 KB)
    // stays in the 32 KB L1.5 instruction cache, where a three-product function (~22 KB) next
    // to it missed on every call (ncu: no_instruction 463 of its 820 stall samples)
    CPair<L> r = cmul2l_ool<L>(u0, u1, d0, u1);
    const C T = r.a, Q0 = r.b;  // T = u0 u1, Q0 = d0 u1
    // inclusive scans of the shifted values: the prefix of (c, T_0, .., T_{G-2}) over the
    // segment is M = c * (product of the factors before the lane), the suffix of
    // (T_1, .., T_{G-1}, 1) the product of those after it -- no products for c or the shift
    C pre = shfl_c<L>(T, 1, true), suf = shfl_c<L>(T, 1, false);
    if (g == 0) pre = c;
    if (g == G - 1) suf = P::one();
#pragma unroll 1
    for (int off = 1; off < G; off <<= 1) {
      const C x1 = shfl_c<L>(pre, off, true), x2 = shfl_c<L>(suf, off, false);
      r = cmul2l_ool<L>(g >= off ? x1 : P::one(), pre, suf, g + off < G ? x2 : P::one());
      pre = r.a;
      suf = r.b;
    }
    const C M = pre;
    r = cmul2l_ool<L>(Q0, suf, d1, suf);  // R0 = Q0 after, X1 = d1 after
    r = cmul2l_ool<L>(M, r.a, u0, r.b);   // g0 = M R0, R1 = u0 X1
    const C g0 = r.a;
    r = cmul2l_ool<L>(M, r.b, M, T);      // g1 = M R1, y = M T (the term's value on the last lane)
    const C g1 = r.a, y = r.b;
    PHC_SEG_STAMP(2)
    // accumulate the gradients into the slot's rows (entry index relative to `rows`: the
    // swizzle depends on it)
    const int sl = warp * TPW + (slot < TPW ? slot : 0);
    const size_t rbase = (size_t)sl * nv;
    double* fs = fpart + (size_t)sl * cd;
    const bool last = live && g == G - 1;  // holds the term's value y
    if (first) {
      if (nf > 0) row_st<L>(rows, rbase + var[0], g0);
      if (nf > 1) row_st<L>(rows, rbase + var[1], g1);
      if (last) sstore<L>(fs, y);
    } else {
      const C z = P::zero();
      const CPair<L> ra = cadd2_ool<L>(nf > 0 ? row_ld<L>(rows, rbase + var[0]) : z, g0,
                                       nf > 1 ? row_ld<L>(rows, rbase + var[1]) : z, g1);
      const C fy = cadd_ool<L>(last ? sload<L>(fs) : z, y);
      if (nf > 0) row_st<L>(rows, rbase + var[0], ra.a);
      if (nf > 1) row_st<L>(rows, rbase + var[1], ra.b);
      if (last) sstore<L>(fs, fy);
    }
    first = false;
    __syncwarp();
  }
  __syncthreads();
  PHC_SEG_STAMP(3)
  // CTA totals in (warp, slot) order; S == 1 writes F and J, S > 1 writes the partial row
  const bool direct = a.S == 1;
  for (int col = threadIdx.x; col <= nv; col += blockDim.x) {
    // the (warp, slot) copies in order
    C acc = col < nv ? row_ld<L>(rows, (size_t)col) : sload<L>(fpart);
    for (int q = 1; q < W * TPW; ++q)
      acc = cadd_ool<L>(acc, col < nv ? row_ld<L>(rows, (size_t)q * nv + col) : sload<L>(fpart + (size_t)q * cd));
    if (direct) {
      if (col < nv)
        cstore<L>(a.J + ((p * a.n_eq + i) * (int64_t)nv + col) * cd, P::norm(acc));
      else
        cstore<L>(a.F + (p * a.n_eq + i) * cd, P::norm(acc));
    } else {
      cstore<L>(a.part + (((p * a.n_eq + i) * a.S + s) * (int64_t)(nv + 1) + col) * cd, acc);
    }
  }
  if (direct) {
    PHC_SEG_STAMP(4)
    return;
  }
  // the last CTA of (p, i) to arrive sums the S partial rows in split order
  __shared__ int s_last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) s_last = atomicAdd(a.count + p * a.n_eq + i, 1) == a.S - 1;
  __syncthreads();
  PHC_SEG_STAMP(4)
  if (!s_last) return;
  __threadfence();
  const double* src = a.part + ((p * a.n_eq + i) * a.S) * (int64_t)(nv + 1) * cd;
  for (int col = threadIdx.x; col <= nv; col += blockDim.x) {
    C acc = cload_cg<L>(src + (size_t)col * cd);
    for (int q = 1; q < a.S; ++q) acc = cadd_ool<L>(acc, cload_cg<L>(src + ((size_t)q * (nv + 1) + col) * cd));
    if (col < nv)
      cstore<L>(a.J + ((p * a.n_eq + i) * (int64_t)nv + col) * cd, P::norm(acc));
    else
      cstore<L>(a.F + (p * a.n_eq + i) * cd, P::norm(acc));
  }
  if (threadIdx.x == 0) a.count[p * a.n_eq + i] = 0;  // ready for the next call
  __syncthreads();
  PHC_SEG_STAMP(5)
}

}  // namespace phc
