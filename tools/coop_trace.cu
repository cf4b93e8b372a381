// Per-column timeline of the cooperative elimination (PHC_COOP_TRACE build): CTA 0's
// look-ahead phases and the grid barrier, from %globaltimer, for one large QD point.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -rdc=false -DPHC_COOP_TRACE=1 -I paper_1109_0545_b200/csrc tools/coop_trace.cu -o tools/coop_trace.bin
#include <cstdio>
#include <vector>
#include "kernels_newton.cuh"
using namespace phc;

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : 256;
  const int L = 4, cd = 2 * L;
  std::vector<double> J((size_t)n * n * cd, 0.0), F((size_t)n * cd, 0.0), X((size_t)n * cd, 0.0);
  srand(1);
  for (size_t i = 0; i < J.size(); i += L) J[i] = rand() / (double)RAND_MAX - 0.5;
  for (size_t i = 0; i < F.size(); i += L) F[i] = rand() / (double)RAND_MAX - 0.5;
  double *dJ, *dF, *dX, *dXn, *dM, *dres, *dred;
  int *dst, *dperm;
  cudaMalloc(&dJ, J.size() * 8); cudaMalloc(&dF, F.size() * 8); cudaMalloc(&dX, X.size() * 8); cudaMalloc(&dXn, X.size() * 8);
  cudaMalloc(&dM, ((size_t)n * (n + 1) + n) * cd * 8); cudaMalloc(&dres, 8); cudaMalloc(&dst, 4);
  cudaMalloc(&dred, 4096 * 8); cudaMalloc(&dperm, (2 * n + 2) * 4);
  cudaMemcpy(dJ, J.data(), J.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dF, F.data(), F.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dX, X.data(), X.size() * 8, cudaMemcpyHostToDevice);
  NewtonArgs a{dX, dF, dJ, dXn, dres, dst, dM, n, 1};
  int* flag = dperm + 2 * n;
  void* args[] = {&a, &dperm, &dred, &flag};
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute((const void*)newton_coop_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  for (int rep = 0; rep < 3; ++rep)
    cudaLaunchCooperativeKernel((const void*)newton_coop_kernel<4>, dim3(nsm), dim3(256), args, coop_smem_bytes(n, 4), 0);
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  static unsigned long long tr[4096][6];
  cudaMemcpyFromSymbol(tr, g_coop_trace, sizeof(tr));
  double acc[5] = {0, 0, 0, 0, 0};
  for (int k = 0; k < n - 1; ++k) {
    for (int q = 0; q < 5; ++q) acc[q] += (double)(tr[k][q + 1] - tr[k][q]);
    if (k < n - 2) acc[4] += 0;  // barrier -> next column start counted in q = 4 (sync) below
  }
  double gap = 0;
  for (int k = 0; k + 1 < n - 1; ++k) gap += (double)(tr[k + 1][0] - tr[k][5]);
  printf("n=%d per column (us): look-ahead col %.2f  pivot+recip %.2f  multipliers %.2f  wait %.2f  grid.sync %.2f  snapshot %.2f  total %.1f us\n",
         n, acc[0] / 1e3 / (n - 1), acc[1] / 1e3 / (n - 1), acc[2] / 1e3 / (n - 1), acc[3] / 1e3 / (n - 1),
         acc[4] / 1e3 / (n - 1), gap / 1e3 / (n - 2), (double)(tr[n - 2][5] - tr[0][0]) / 1e3);
  return 0;
}
