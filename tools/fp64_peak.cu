// FP64 pipe peak microbenchmark (SURVEY.md §2.4 N8, §8(d) "FP64 peak (the denominator)").
// Many independent DFMA / DADD chains per thread; flops = 2*#DFMA (+1 per DADD).
// Also measures dependent-chain latency of DFMA and DADD with one warp.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA error %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int CH>
__global__ void dfma_chains(double* out, int iters, double a, double b) {
  double r[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) r[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) r[c] = __fma_rn(r[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += r[c];
  if (s == 12345.678) out[0] = s;
}

template <int CH>
__global__ void dadd_chains(double* out, int iters, double b) {
  double r[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) r[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) r[c] = __dadd_rn(r[c], b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += r[c];
  if (s == 12345.678) out[0] = s;
}

__global__ void lat_dfma(double* out, long long* cyc, int iters, double a, double b) {
  double r = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) r = __fma_rn(r, a, b);
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[0] = r; }
}
__global__ void lat_dadd(double* out, long long* cyc, int iters, double b) {
  double r = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) r = __dadd_rn(r, b);
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[0] = r; }
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int clk_khz = 0; cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  printf("{\"device\": \"%s\", \"sm\": %d, \"cc\": \"%d.%d\", \"clock_khz\": %d, \"smem_per_sm\": %zu, \"smem_optin\": %zu, \"regs_per_sm\": %d, \"l2\": %d, \"mem_gb\": %.1f}\n",
         p.name, p.multiProcessorCount, p.major, p.minor, clk_khz, p.sharedMemPerMultiprocessor,
         p.sharedMemPerBlockOptin, p.regsPerMultiprocessor, p.l2CacheSize, p.totalGlobalMem / 1e9);
  double* d; long long* c; CK(cudaMalloc(&d, 8)); CK(cudaMalloc(&c, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 4096;
  const int CH = 8;
  for (int bpsm = 2; bpsm <= 8; bpsm *= 2) {
    int blocks = p.multiProcessorCount * bpsm, threads = 256;
    for (int w = 0; w < 3; ++w) dfma_chains<CH><<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
    CK(cudaDeviceSynchronize());
    float best = 1e30f;
    for (int rep = 0; rep < 10; ++rep) {
      cudaEventRecord(e0);
      dfma_chains<CH><<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    double flops = 2.0 * (double)blocks * threads * iters * CH;
    printf("{\"kind\": \"dfma\", \"blocks_per_sm\": %d, \"ms\": %.4f, \"tflops\": %.3f}\n", bpsm, best, flops / best / 1e9);
    best = 1e30f;
    for (int rep = 0; rep < 10; ++rep) {
      cudaEventRecord(e0);
      dadd_chains<CH><<<blocks, threads>>>(d, iters, 1e-7);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    flops = 1.0 * (double)blocks * threads * iters * CH;
    printf("{\"kind\": \"dadd\", \"blocks_per_sm\": %d, \"ms\": %.4f, \"tops\": %.3f}\n", bpsm, best, flops / best / 1e9);
  }
  // sustained: long run of DFMA (~2 s) to see the clock under load
  {
    int blocks = p.multiProcessorCount * 8, threads = 256;
    cudaEventRecord(e0);
    for (int r = 0; r < 40; ++r) dfma_chains<CH><<<blocks, threads>>>(d, iters * 4, 0.999999, 1e-7);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 40.0 * 2.0 * (double)blocks * threads * iters * 4 * CH;
    printf("{\"kind\": \"dfma_sustained\", \"ms\": %.3f, \"tflops\": %.3f}\n", ms, flops / ms / 1e9);
  }
  long long h;
  lat_dfma<<<1, 32>>>(d, c, 1 << 16, 0.999999, 1e-7); CK(cudaDeviceSynchronize());
  lat_dfma<<<1, 32>>>(d, c, 1 << 16, 0.999999, 1e-7); CK(cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost));
  printf("{\"kind\": \"dfma_latency_cycles\", \"value\": %.2f}\n", (double)h / (1 << 16));
  lat_dadd<<<1, 32>>>(d, c, 1 << 16, 1e-7); CK(cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost));
  printf("{\"kind\": \"dadd_latency_cycles\", \"value\": %.2f}\n", (double)h / (1 << 16));
  return 0;
}
