// Does an FP64 warp instruction with only 16 active lanes cost less FP64-pipe time than one
// with 32?  Each warp runs `iters` iterations of 8 independent DFMA chains with the lanes
// [0, active) active; time per launch with CUDA events, all SMs, 2 or 4 warps per scheduler.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chains(double* out, int iters, int active) {
  const int lane = threadIdx.x & 31;
  if (lane >= active) return;
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = 1.0 + 1e-9 * (threadIdx.x + i);
  const double b = 0.999999999, c = 1e-12;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, (size_t)sms * 4 * 1024 * sizeof(double));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 20000;
  for (int warps : {4, 8, 16}) {
    for (int active : {32, 16, 8, 1}) {
      chains<<<sms, warps * 32>>>(out, 100, active);
      cudaEventRecord(e0);
      chains<<<sms, warps * 32>>>(out, iters, active);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      const double warp_insts = (double)sms * warps * iters * 8;
      printf("{\"warps_per_sm\": %d, \"active_lanes\": %d, \"ms\": %.3f, \"warp_dfma_per_clk_per_sm\": %.3f}\n", warps,
             active, ms, warp_insts / sms / (ms * 1e-3 * 1.965e9));
    }
  }
  return 0;
}
