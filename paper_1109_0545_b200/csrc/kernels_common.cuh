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
  const double* Yp = Y + p * M * cd;
  const double* Gp = G + p * n_factors * cd;
  for (int64_t e = cl_ptr[c]; e < cl_ptr[c + 1]; ++e) {
    const int j = cl_j[e];
    const C val = (c == 0) ? cload<L>(Yp + (int64_t)j * cd) : cload<L>(Gp + cl_q[e] * cd);
    const double* crow = cT + ((int64_t)j * n_eq + i0) * cd;
#pragma unroll
    for (int u = 0; u < TI; ++u)
      if (i0 + u < n_eq) acc[u] = P::add_lazy(acc[u], P::mul_lazy(cload<L>(crow + u * cd), val));
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

}  // namespace phc
