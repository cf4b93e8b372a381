// Generic (any system shape) kernels of the evaluation path: power table, per-term
// Speelpenning products + coefficient product, deterministic CSR reductions.
// SURVEY.md §8(a) rows a2-a8; DESIGN.md "kernels".
//
// These handle every valid system (variable k per term, constant terms, duplicate
// terms, k up to PHC_MAX_K).  The specialised warp-per-block kernels in
// kernels_block.cuh cover the benchmark shapes faster; both compute the same
// per-term arithmetic in the same order, so their results are bitwise identical.
#pragma once
#include "arith.cuh"

namespace phc {

// Power table (row a2).  For each point p and variable v (plus a dummy variable
// v = n_var used for padding):
//   U[a-1]   = x_v^a          a = 1..E   (repeated multiplication, reading C4)
//   Dd[a-1]  = a * x_v^(a-1)  a = 1..E   (the exponent factor of reading C3, folded here)
// Layout: PT[p][v][2E][2L] (U entries then Dd entries), one complex per entry.
// The dummy variable has U = 1, Dd = 0.
template <int L>
__global__ void power_table_kernel(const double* __restrict__ X, int n_var, int E, int64_t n_points,
                                   double* __restrict__ PT) {
  using P = Prec<L>;
  using C = typename P::C;
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t per_point = n_var + 1;
  if (gid >= n_points * per_point) return;
  const int64_t p = gid / per_point;
  const int v = (int)(gid % per_point);
  double* row = PT + ((p * per_point + v) * (2 * E)) * (2 * L);
  if (v == n_var) {
    for (int a = 0; a < E; ++a) {
      cstore<L>(row + a * 2 * L, P::one());
      cstore<L>(row + (E + a) * 2 * L, P::zero());
    }
    return;
  }
  const C x = cload<L>(X + (p * n_var + v) * 2 * L);
  C pw = P::one();  // x^(a-1)
  for (int a = 1; a <= E; ++a) {
    cstore<L>(row + (E + a - 1) * 2 * L, a == 1 ? pw : P::mul_int(pw, (double)a));
    pw = (a == 1) ? x : P::mul(pw, x);
    cstore<L>(row + (a - 1) * 2 * L, pw);
  }
}

// Per-term kernel (rows a3-a6), one thread per (point, term).  With coeff2 != nullptr the
// coefficient is the homotopy blend at the point's t (NEXT-3).
// For a term c * prod_{j=1..k} u_j with u_j = x_{i_j}^{a_j}, d_j = a_j x_{i_j}^{a_j - 1}:
//   suffix  s_q = u_{k-q+1} ... u_k              (q = 1..k-1; the paper's phi)
//   prefix  r_m = c u_1 ... u_m                  (m = 0..k;   the paper's psi with the
//                                                  coefficient folded in)
//   value   y   = r_k                             (the term c x^a)
//   partial g_m = r_{m-1} * d_m * s_{k-m}        (c * a_m x^{a - e_m}: the shifted monomial
//                                                  c * common-factor * omega_m)
// i.e. 4k-3 complex products per term.
// Packed factor word: bits 0-15 variable, bits 16-23 exponent.
// PTFAST (the common-support batch path): threads run over points (the term tables are
// warp-uniform loads) and Y, G are stored transposed, [t][p] and [f][p], so the coefficient
// product reads 32 points' values of one monomial as one contiguous 1 KB (DD) line.
template <int L, int MAXK, bool PTFAST = false>
__global__ void term_kernel(const int64_t* __restrict__ term_ptr, const uint32_t* __restrict__ fac,
                            const double* __restrict__ coeff, const double* __restrict__ coeff2,
                            const double* __restrict__ T, const double* __restrict__ PT, int n_var, int E,
                            int64_t n_terms, int64_t n_factors, int64_t n_points, double* __restrict__ Y,
                            double* __restrict__ G) {
  using P = Prec<L>;
  using C = typename P::C;
  const int64_t t = PTFAST ? (int64_t)blockIdx.y : (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t p = PTFAST ? (int64_t)blockIdx.x * blockDim.x + threadIdx.x : (int64_t)blockIdx.y;
  if (t >= n_terms || p >= n_points) return;
  const double* pt = PT + p * (int64_t)(n_var + 1) * (2 * E) * (2 * L);
  const int64_t f0 = term_ptr[t];
  const int k = (int)(term_ptr[t + 1] - f0);
  C r = cload<L>(coeff + t * 2 * L);
  if (coeff2) {  // NEXT-3 homotopy: c(t) = (1 - t) c_start + t c_target (reading H1)
    const typename P::real tt = P::rload(T + p * L);
    r = P::add(P::mul_real(r, P::one_minus(tt)), P::mul_real(cload<L>(coeff2 + t * 2 * L), tt));
  }
  PHC_CHECK(k >= 0 && k <= MAXK);
  auto U = [&](uint32_t w) { return cload<L>(pt + ((int64_t)(w & 0xffffu) * 2 * E + ((w >> 16) & 0xffu) - 1) * 2 * L); };
  auto Dd = [&](uint32_t w) { return cload<L>(pt + ((int64_t)(w & 0xffffu) * 2 * E + E + ((w >> 16) & 0xffu) - 1) * 2 * L); };
  C s[MAXK];
  if (k >= 2) {
    s[1] = U(fac[f0 + k - 1]);
    for (int q = 2; q <= k - 1; ++q) s[q] = P::mul(s[q - 1], U(fac[f0 + k - q]));
  }
  for (int m = 1; m <= k; ++m) {
    const uint32_t w = fac[f0 + m - 1];
    C gm = P::mul(r, Dd(w));
    if (m < k) gm = P::mul(gm, s[k - m]);
    const int64_t gi = PTFAST ? (f0 + m - 1) * n_points + p : p * n_factors + f0 + m - 1;
    cstore<L>(G + gi * 2 * L, gm);
    r = P::mul(r, U(w));
  }
  cstore<L>(Y + (PTFAST ? t * n_points + p : p * n_terms + t) * 2 * L, r);
}

// Reductions (row a7) and write of Y (row a8): one thread per (point, entry).
// Entries e < n_eq*n_var are J[i][v] = sum over the CSR list of factor slots (i, v),
// in increasing factor order (term order, then slot); entries e >= n_eq*n_var are
// F[i] = sum_{t in T_i} y_t in term order.  Empty lists give exact zeros.
template <int L>
__global__ void reduce_kernel(const int64_t* __restrict__ jptr, const int64_t* __restrict__ jidx,
                              const int64_t* __restrict__ poly_ptr, const double* __restrict__ Y,
                              const double* __restrict__ G, int n_eq, int n_var, int64_t n_terms, int64_t n_factors,
                              int64_t n_points, double* __restrict__ F, double* __restrict__ J) {
  using P = Prec<L>;
  using C = typename P::C;
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t p = blockIdx.y;
  const int64_t nj = (int64_t)n_eq * n_var;
  if (e >= nj + n_eq || p >= n_points) return;
  C acc = P::zero();
  if (e < nj) {
    const double* g = G + p * n_factors * 2 * L;
    for (int64_t q = jptr[e]; q < jptr[e + 1]; ++q) acc = P::add(acc, cload<L>(g + jidx[q] * 2 * L));
    cstore<L>(J + (p * nj + e) * 2 * L, acc);
  } else {
    const int i = (int)(e - nj);
    const double* y = Y + p * n_terms * 2 * L;
    for (int64_t t = poly_ptr[i]; t < poly_ptr[i + 1]; ++t) acc = P::add(acc, cload<L>(y + t * 2 * L));
    cstore<L>(F + (p * n_eq + i) * 2 * L, acc);
  }
}

}  // namespace phc
