/* A plain C consumer of the C ABI (include/phc.h): no Python, no torch.  Builds the system
 *   f_0 = x0^2 x1 + (3 - 2i),   f_1 = x0 x1 x2 - x2^4
 * in complex double-double, evaluates F and J at x = (2, 3, 5) on device 0, and checks the
 * exact values (SPEC S:158, S:218 style hand computations):
 *   F = (12 + 3 - 2i, 30 - 625) = (15 - 2i, -595)
 *   J = [[2 x0 x1, x0^2, 0], [x1 x2, x0 x2, x0 x1 - 4 x2^3]] = [[12, 4, 0], [15, 10, -494]]
 * Then Alg. 2 to tolerance (phc_newton_solve_batch) on x^2 - 4 = 0 from x = 1: the root 2.
 * Build: gcc -O2 c_abi_demo.c -I../include -L../paper_1109_0545_b200 -lphc
 *        -I/usr/local/cuda/include -L/usr/local/cuda/lib64 -lcudart  */
#include <cuda_runtime.h>
#include <stdio.h>
#include <string.h>

#include "phc.h"

int main(void) {
  const int L = 2, n_eq = 2, n_var = 3;
  const int64_t poly_ptr[3] = {0, 2, 4};            /* terms 0-1 in f_0, 2-3 in f_1 */
  const int64_t term_ptr[5] = {0, 2, 2, 5, 6};      /* x0^2 x1 | const | x0 x1 x2 | x2^4 */
  const int32_t var_idx[6] = {0, 1, 0, 1, 2, 2};
  const int32_t exponent[6] = {2, 1, 1, 1, 1, 4};
  double coeff[4][2][2];
  memset(coeff, 0, sizeof coeff);
  coeff[0][0][0] = 1.0;                              /* 1 */
  coeff[1][0][0] = 3.0;  coeff[1][1][0] = -2.0;      /* 3 - 2i */
  coeff[2][0][0] = 1.0;                              /* 1 */
  coeff[3][0][0] = -1.0;                             /* -1 */
  phc_system* s = NULL;
  int rc = phc_system_create(&s, n_eq, n_var, L, 4, poly_ptr, term_ptr, var_idx, exponent, &coeff[0][0][0], 0);
  if (rc) { printf("create failed: %d %s\n", rc, phc_last_error()); return 1; }
  double x[3][2][2];
  memset(x, 0, sizeof x);
  x[0][0][0] = 2.0; x[1][0][0] = 3.0; x[2][0][0] = 5.0;
  double *dx, *df, *dj;
  cudaMalloc((void**)&dx, sizeof x);
  cudaMalloc((void**)&df, n_eq * 2 * L * sizeof(double));
  cudaMalloc((void**)&dj, n_eq * n_var * 2 * L * sizeof(double));
  cudaMemcpy(dx, x, sizeof x, cudaMemcpyHostToDevice);
  rc = phc_eval_jacobian(s, dx, df, dj, NULL);
  if (rc) { printf("eval failed: %d %s\n", rc, phc_last_error()); return 1; }
  double f[2][2][2], j[2][3][2][2];
  cudaMemcpy(f, df, sizeof f, cudaMemcpyDeviceToHost);
  cudaMemcpy(j, dj, sizeof j, cudaMemcpyDeviceToHost);
  const double fre[2] = {15, -595}, fim[2] = {-2, 0};
  const double jre[2][3] = {{12, 4, 0}, {15, 10, -494}};
  int bad = 0;
  for (int i = 0; i < 2; ++i) {
    bad |= f[i][0][0] != fre[i] || f[i][1][0] != fim[i] || f[i][0][1] != 0 || f[i][1][1] != 0;
    for (int v = 0; v < 3; ++v) bad |= j[i][v][0][0] != jre[i][v] || j[i][v][1][0] != 0;
  }
  printf("%s F = (%g%+gi, %g%+gi), J[1] = (%g, %g, %g); %s\n", phc_version(), f[0][0][0], f[0][1][0], f[1][0][0],
         f[1][1][0], j[1][0][0][0], j[1][1][0][0], j[1][2][0][0], bad ? "MISMATCH" : "exact");
  phc_system_destroy(s);
  cudaFree(dx);
  cudaFree(df);
  cudaFree(dj);
  /* Newton's method to tolerance on g = x^2 - 4 */
  const int64_t gp[2] = {0, 2}, gt[3] = {0, 1, 1};
  const int32_t gv[1] = {0}, ge[1] = {2};
  double gc[2][2][2];
  memset(gc, 0, sizeof gc);
  gc[0][0][0] = 1.0;
  gc[1][0][0] = -4.0;
  phc_system* g = NULL;
  rc = phc_system_create(&g, 1, 1, L, 2, gp, gt, gv, ge, &gc[0][0][0], 0);
  if (rc) { printf("create failed: %d %s\n", rc, phc_last_error()); return 1; }
  double z0[1][2][2] = {{{1.0, 0.0}, {0.0, 0.0}}}, z[1][2][2];
  double *dz, *dres;
  int32_t *dits, *dst;
  cudaMalloc((void**)&dz, sizeof z0);
  cudaMalloc((void**)&dres, sizeof(double));
  cudaMalloc((void**)&dits, sizeof(int32_t));
  cudaMalloc((void**)&dst, sizeof(int32_t));
  cudaMemcpy(dz, z0, sizeof z0, cudaMemcpyHostToDevice);
  rc = phc_newton_solve_batch(g, 1, dz, NULL, 1e-28, 20, dz, dres, dits, dst, NULL);
  if (rc) { printf("newton failed: %d %s\n", rc, phc_last_error()); return 1; }
  int32_t its = 0, stn = -1;
  cudaMemcpy(z, dz, sizeof z, cudaMemcpyDeviceToHost);
  cudaMemcpy(&its, dits, sizeof its, cudaMemcpyDeviceToHost);
  cudaMemcpy(&stn, dst, sizeof stn, cudaMemcpyDeviceToHost);
  const int nbad = stn != 0 || z[0][0][0] != 2.0 || z[0][1][0] != 0.0;
  printf("Newton on x^2 - 4 from 1: %d iterations, x = %.17g, status %d; %s\n", its, z[0][0][0], stn,
         nbad ? "MISMATCH" : "exact");
  phc_system_destroy(g);
  cudaFree(dz);
  cudaFree(dres);
  cudaFree(dits);
  cudaFree(dst);
  return bad | nbad;
}
