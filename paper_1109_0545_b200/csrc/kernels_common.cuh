// NEXT-2: common-support systems, the paper's two-stage evaluation
// (Alg. 2 "V := Monomial_Evaluation" then "Y := Coefficient_Product", PAPER.md P:269-284,
// P:329-333; the Table 1 system "40 variables with a common support of 200 monomials",
// P:355-358).
//
// Every polynomial f_i = sum_j C[i][j] x^{a_j} uses the same M monomials.  Stage V evaluates
// each monomial once per point, with all its partials (the generic term kernel with unit
// coefficients: value x^{a_j} and g_{j,m} = a_m x^{a_j - e_m}, kernels_generic.cuh).  Stage Y
// is then a complex DD/QD product of the shared coefficient matrix with the monomial data:
//     F[i]    = sum_j C[i][j] V_j
//     J[i][v] = sum_{j : v in vars(j)} C[i][j] g_{j, slot of v}
// i.e. [F | J] = C [V | D] with D the sparse M x n matrix of partials.
#pragma once
#include "arith.cuh"

namespace phc {

// Coefficient product (stage Y), one thread per (point, column c, tile of TI rows).
// Column c = 0 is F (list: every monomial j, value Y[p][j]); column c = v + 1 is J[:, v]
// (list: the factor slots q of variable v, in increasing monomial order, value G[p][q]).
// Consecutive threads take consecutive row tiles of the same column: the C^T loads of a
// warp are contiguous and the monomial value is a broadcast.  Sums run in list order
// (deterministic), lazily, renormalised once at the end.
//   cl_ptr [n_var + 2], cl_j [entries] (monomial), cl_q [entries] (factor index, -1 for F)
//   cT     [M][n_eq][2][L]  (C transposed)
template <int L, int TI>
__global__ void coef_product_kernel(const int64_t* __restrict__ cl_ptr, const int32_t* __restrict__ cl_j,
                                    const int64_t* __restrict__ cl_q, const double* __restrict__ cT,
                                    const double* __restrict__ cT2, const double* __restrict__ T,
                                    const double* __restrict__ Y, const double* __restrict__ G, int n_eq, int n_var,
                                    int64_t M, int64_t n_factors, int64_t n_points, double* __restrict__ F,
                                    double* __restrict__ J) {
  using P = Prec<L>;
  using C = typename P::C;
  constexpr int cd = 2 * L;
  const int tiles = (n_eq + TI - 1) / TI;
  const int64_t per_point = (int64_t)(n_var + 1) * tiles;
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= n_points * per_point) return;
  const int64_t p = gid / per_point;
  const int r = (int)(gid % per_point);
  const int c = r / tiles;
  const int i0 = (r % tiles) * TI;
  C acc[TI];
#pragma unroll
  for (int u = 0; u < TI; ++u) acc[u] = P::zero();
  typename P::real tt = P::one().re, omt = P::one().re;
  if (cT2) {
    tt = P::rload(T + p * L);
    omt = P::one_minus(tt);
  }
  const double* Yp = Y + p * M * cd;
  const double* Gp = G + p * n_factors * cd;
  for (int64_t e = cl_ptr[c]; e < cl_ptr[c + 1]; ++e) {
    const int j = cl_j[e];
    PHC_CHECK(j >= 0 && j < M && (c == 0 || (cl_q[e] >= 0 && cl_q[e] < n_factors)));
    const C val = (c == 0) ? cload<L>(Yp + (int64_t)j * cd) : cload<L>(Gp + cl_q[e] * cd);
    const double* crow = cT + ((int64_t)j * n_eq + i0) * cd;
#pragma unroll
    for (int u = 0; u < TI; ++u)
      if (i0 + u < n_eq) {
        C c = cload<L>(crow + u * cd);
        if (cT2)  // homotopy (NEXT-3): c(t) = (1 - t) c_s + t c_f
          c = P::add(P::mul_real(c, omt), P::mul_real(cload<L>(cT2 + ((int64_t)j * n_eq + i0 + u) * cd), tt));
        acc[u] = P::accum(acc[u], P::mul_lazy(c, val));
      }
  }
#pragma unroll
  for (int u = 0; u < TI; ++u) {
    if (i0 + u >= n_eq) break;
    const C v = P::norm(acc[u]);
    if (c == 0)
      cstore<L>(F + (p * n_eq + i0 + u) * cd, v);
    else
      cstore<L>(J + ((p * n_eq + i0 + u) * (int64_t)n_var + (c - 1)) * cd, v);
  }
}

// Latency variant of the monomial stage (calls with few points, monomials with k <= 32):
// one warp per (point, monomial), lane l holding factor l (u_l = x^{a_l}, d_l = a_l x^{a_l-1}
// from the power table; idle lanes u = 1, d = 0).  The products of all factors but one
// (the paper's omega_m = psi_{m-1} phi_{k-m}) come from an inclusive prefix scan
// (psi) and an inclusive suffix scan (phi) over the warp, 5 shuffle steps each, then
// g_l = psi_{l-1} phi_{l+1} d_l: a dependency path of ~7 products instead of ~2k, for ~2x the
// products of the sequential chains (reading N2-3).  Writes Y[p][j] = x^{a_j} and
// G[p][q] = g for the monomial's factor slots q, like term_kernel with unit coefficients.
template <int L>
__global__ void monomial_scan_kernel(const int64_t* __restrict__ term_ptr, const uint32_t* __restrict__ fac,
                                     const double* __restrict__ PT, int n_var, int E, int64_t M, int64_t n_factors,
                                     int64_t n_points, double* __restrict__ Y, double* __restrict__ G) {
  using P = Prec<L>;
  using C = typename P::C;
  constexpr int cd = 2 * L;
  const int lane = threadIdx.x & 31;
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (wid >= n_points * M) return;  // warp-uniform
  const int64_t p = wid / M, j = wid % M;
  const int64_t f0 = term_ptr[j];
  const int k = (int)(term_ptr[j + 1] - f0);
  const double* pt = PT + p * (int64_t)(n_var + 1) * (2 * E) * cd;
  C u = P::one(), d = P::zero();
  if (lane < k) {
    const uint32_t w = fac[f0 + lane];
    const int64_t e = (int64_t)(w & 0xffffu) * 2 * E + ((w >> 16) & 0xffu) - 1;
    u = cload<L>(pt + e * cd);
    d = cload<L>(pt + (e + E) * cd);
  }
  auto shfl = [](const C& v, int delta, bool up) {
    C r;
#pragma unroll
    for (int i = 0; i < L; ++i) {
      r.re.x[i] = up ? __shfl_up_sync(0xffffffffu, v.re.x[i], delta) : __shfl_down_sync(0xffffffffu, v.re.x[i], delta);
      r.im.x[i] = up ? __shfl_up_sync(0xffffffffu, v.im.x[i], delta) : __shfl_down_sync(0xffffffffu, v.im.x[i], delta);
    }
    return r;
  };
  C pre = u, suf = u;  // inclusive prefix / suffix products
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const C a = shfl(pre, off, true), b = shfl(suf, off, false);
    if (lane >= off) pre = P::mul(a, pre);
    if (lane + off < 32) suf = P::mul(suf, b);
  }
  C before = shfl(pre, 1, true), after = shfl(suf, 1, false);
  if (lane == 0) before = P::one();
  if (lane == 31) after = P::one();
  if (lane < k) cstore<L>(G + (p * n_factors + f0 + lane) * cd, P::mul(P::mul(before, d), after));
  if (lane == 31) cstore<L>(Y + (p * M + j) * cd, pre);
}

// Batch variant of the coefficient product over transposed monomial data (Y^T [M][P],
// G^T [n_factors][P], from term_kernel<..., PTFAST>): threads run over points, so a warp
// walks one column list with one row tile -- its coefficient loads are warp-uniform
// broadcasts and its value loads one contiguous line per list entry.  Per output the same
// operations in the same order as coef_product_kernel (bitwise the same results).
template <int L, int TI>
__global__ void coef_product_pt_kernel(const int64_t* __restrict__ cl_ptr, const int32_t* __restrict__ cl_j,
                                       const int64_t* __restrict__ cl_q, const double* __restrict__ cT,
                                       const double* __restrict__ cT2, const double* __restrict__ T,
                                       const double* __restrict__ Yt, const double* __restrict__ Gt, int n_eq,
                                       int n_var, int64_t n_points, double* __restrict__ F, double* __restrict__ J) {
  using P = Prec<L>;
  using C = typename P::C;
  constexpr int cd = 2 * L;
  const int tiles = (n_eq + TI - 1) / TI;
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int c = blockIdx.y / tiles;
  const int i0 = (blockIdx.y % tiles) * TI;
  if (p >= n_points) return;
  C acc[TI];
#pragma unroll
  for (int u = 0; u < TI; ++u) acc[u] = P::zero();
  typename P::real tt = P::one().re, omt = P::one().re;
  if (cT2) {
    tt = P::rload(T + p * L);
    omt = P::one_minus(tt);
  }
  for (int64_t e = cl_ptr[c]; e < cl_ptr[c + 1]; ++e) {
    const int j = cl_j[e];
    const int64_t row = (c == 0) ? (int64_t)j : cl_q[e];
    const C val = cload<L>((c == 0 ? Yt : Gt) + (row * n_points + p) * cd);
    const double* crow = cT + ((int64_t)j * n_eq + i0) * cd;
#pragma unroll
    for (int u = 0; u < TI; ++u)
      if (i0 + u < n_eq) {
        C cf = cload<L>(crow + u * cd);
        if (cT2) cf = P::add(P::mul_real(cf, omt), P::mul_real(cload<L>(cT2 + ((int64_t)j * n_eq + i0 + u) * cd), tt));
        acc[u] = P::accum(acc[u], P::mul_lazy(cf, val));
      }
  }
#pragma unroll
  for (int u = 0; u < TI; ++u) {
    if (i0 + u >= n_eq) break;
    const C v = P::norm(acc[u]);
    if (c == 0)
      cstore<L>(F + (p * n_eq + i0 + u) * cd, v);
    else
      cstore<L>(J + ((p * n_eq + i0 + u) * (int64_t)n_var + (c - 1)) * cd, v);
  }
}

// Latency variant of the coefficient product for calls with few points: one warp per
// (point, column c, row i); the 32 lanes stride over the column's list (lane l takes entries
// l, l + 32, ...) and the partial sums meet in a fixed shuffle tree.  ~32x the parallelism of
// coef_product_kernel at the cost of the tree (worthwhile only when the grid would otherwise be
// a fraction of a wave).  Different summation order: the two variants agree within the
// tolerance, each is deterministic (reading N2-2).
template <int L>
__global__ void coef_product_split_kernel(const int64_t* __restrict__ cl_ptr, const int32_t* __restrict__ cl_j,
                                          const int64_t* __restrict__ cl_q, const double* __restrict__ cT,
                                          const double* __restrict__ cT2, const double* __restrict__ T,
                                          const double* __restrict__ Y, const double* __restrict__ G, int n_eq,
                                          int n_var, int64_t M, int64_t n_factors, int64_t n_points,
                                          double* __restrict__ F, double* __restrict__ J) {
  using P = Prec<L>;
  using C = typename P::C;
  constexpr int cd = 2 * L;
  const int lane = threadIdx.x & 31;
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t per_point = (int64_t)(n_var + 1) * n_eq;
  if (wid >= n_points * per_point) return;  // warp-uniform
  const int64_t p = wid / per_point;
  const int r = (int)(wid % per_point);
  const int c = r / n_eq, i = r % n_eq;
  const double* Yp = Y + p * M * cd;
  const double* Gp = G + p * n_factors * cd;
  C acc = P::zero();
  typename P::real tt = P::one().re, omt = P::one().re;
  if (cT2) {
    tt = P::rload(T + p * L);
    omt = P::one_minus(tt);
  }
  for (int64_t e = cl_ptr[c] + lane; e < cl_ptr[c + 1]; e += 32) {
    const int j = cl_j[e];
    const C val = (c == 0) ? cload<L>(Yp + (int64_t)j * cd) : cload<L>(Gp + cl_q[e] * cd);
    C cf = cload<L>(cT + ((int64_t)j * n_eq + i) * cd);
    if (cT2) cf = P::add(P::mul_real(cf, omt), P::mul_real(cload<L>(cT2 + ((int64_t)j * n_eq + i) * cd), tt));
    acc = P::accum(acc, P::mul_lazy(cf, val));
  }
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) {
    C o;
#pragma unroll
    for (int k = 0; k < L; ++k) {
      o.re.x[k] = __shfl_down_sync(0xffffffffu, acc.re.x[k], d);
      o.im.x[k] = __shfl_down_sync(0xffffffffu, acc.im.x[k], d);
    }
    acc = P::add_lazy(acc, o);
  }
  if (lane == 0) {
    const C v = P::norm(acc);
    if (c == 0)
      cstore<L>(F + (p * n_eq + i) * cd, v);
    else
      cstore<L>(J + ((p * n_eq + i) * (int64_t)n_var + (c - 1)) * cd, v);
  }
}

}  // namespace phc
