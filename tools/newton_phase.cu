// Phase timeline of the Newton eliminations (PHC_NEWTON_TRACE build): matrix load,
// elimination, back substitution, for the shared-memory kernel (c3 shape: n = 40 QD, one point,
// 512 threads; c2 shape: n = 20 DD) and the cooperative kernel (n = 256 QD, one point).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -DPHC_NEWTON_TRACE=1 -I paper_1109_0545_b200/csrc tools/newton_phase.cu -o tools/newton_phase.bin
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "kernels_newton.cuh"
using namespace phc;

struct Bufs {
  double *J, *F, *X, *Xn, *M, *res, *red;
  int *st, *perm;
};

static Bufs make(int n, int L) {
  const int cd = 2 * L;
  std::vector<double> J((size_t)n * n * cd, 0.0), F((size_t)n * cd, 0.0), X((size_t)n * cd, 0.0);
  srand(1);
  for (size_t i = 0; i < J.size(); i += L) J[i] = rand() / (double)RAND_MAX - 0.5;
  for (size_t i = 0; i < F.size(); i += L) F[i] = rand() / (double)RAND_MAX - 0.5;
  Bufs b;
  cudaMalloc(&b.J, J.size() * 8); cudaMalloc(&b.F, F.size() * 8); cudaMalloc(&b.X, X.size() * 8);
  cudaMalloc(&b.Xn, X.size() * 8); cudaMalloc(&b.M, ((size_t)n * (n + 1) + n) * cd * 8);
  cudaMalloc(&b.res, 8); cudaMalloc(&b.st, 4); cudaMalloc(&b.red, 4096 * 8); cudaMalloc(&b.perm, (2 * n + 2) * 4);
  cudaMemcpy(b.J, J.data(), J.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(b.F, F.data(), F.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(b.X, X.data(), X.size() * 8, cudaMemcpyHostToDevice);
  return b;
}

static void report(const char* name, int kind, float ms_event) {
  unsigned long long tr[2][4];
  cudaMemcpyFromSymbol(tr, g_newton_phase, sizeof(tr));
  printf("{\"case\": \"%s\", \"load_us\": %.2f, \"elim_us\": %.2f, \"backsub_us\": %.2f, \"kernel_event_us\": %.2f}\n", name,
         (tr[kind][1] - tr[kind][0]) / 1e3, (tr[kind][2] - tr[kind][1]) / 1e3, (tr[kind][3] - tr[kind][2]) / 1e3,
         ms_event * 1e3);
}

template <int L>
static void solve_case(const char* name, int n, int threads) {
  Bufs b = make(n, L);
  NewtonArgs a{b.X, b.F, b.J, b.Xn, b.res, b.st, b.M, n, 1};
  const size_t sm = solve_smem_bytes(n, L);
  cudaFuncSetAttribute((const void*)newton_solve_kernel<L>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms = 0;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    newton_solve_kernel<L><<<1, threads, sm>>>(a);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) printf("%s: %s\n", name, cudaGetErrorString(e));
  report(name, 0, ms);
  // per-column split (the last launch): look-ahead update, pivot + reciprocal + multipliers,
  // the trailing update's finish relative to the column start, the barrier's release
  static unsigned long long tc[128][5];
  static const unsigned long long zero[128][5] = {};
  cudaMemcpyFromSymbol(tc, g_newton_cols, sizeof(tc));
  double upd = 0, piv = 0, trail = 0, col = 0;
  int nc = 0;
  for (int k = 0; k < n - 1 && k < 128; ++k, ++nc) {
    upd += (tc[k][1] - tc[k][0]) / 1e3;
    piv += (tc[k][2] - tc[k][1]) / 1e3;
    trail += (tc[k][3] > tc[k][0] ? tc[k][3] - tc[k][0] : 0) / 1e3;
    col += (tc[k][4] - tc[k][0]) / 1e3;
  }
  printf("  per column (us, mean of %d): look-ahead update %.2f, pivot+recip+multipliers %.2f, trailing update done at %.2f, column %.2f\n",
         nc, upd / nc, piv / nc, trail / nc, col / nc);
  for (int k = 0; k < n - 1 && k < 128; k += (n > 16 ? n / 8 : 1))
    printf("  k=%d: upd %.2f piv %.2f trail %.2f col %.2f\n", k, (tc[k][1] - tc[k][0]) / 1e3, (tc[k][2] - tc[k][1]) / 1e3,
           (tc[k][3] > tc[k][0] ? tc[k][3] - tc[k][0] : 0) / 1e3, (tc[k][4] - tc[k][0]) / 1e3);
  cudaMemcpyToSymbol(g_newton_cols, zero, sizeof(zero));
}

static void coop_case(const char* name, int n) {
  const int L = 4;
  Bufs b = make(n, L);
  NewtonArgs a{b.X, b.F, b.J, b.Xn, b.res, b.st, b.M, n, 1};
  int* flag = b.perm + 2 * n;
  void* args[] = {&a, &b.perm, &b.red, &flag};
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute((const void*)newton_coop_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms = 0;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    cudaLaunchCooperativeKernel((const void*)newton_coop_kernel<4>, dim3(nsm), dim3(kCoopThreads), args,
                                coop_smem_bytes(n, 4), 0);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
  }
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) printf("%s: %s\n", name, cudaGetErrorString(e));
  report(name, 1, ms);
}

int main() {
  solve_case<4>("c3 shape: solve kernel n=40 QD, 512 threads", 40, 512);
  solve_case<2>("c2 shape: solve kernel n=20 DD, 512 threads", 20, 512);
  solve_case<2>("batch shape: solve kernel n=32 DD, 128 threads", 32, 128);
  coop_case("large shape: cooperative kernel n=256 QD", 256);
  return 0;
}
