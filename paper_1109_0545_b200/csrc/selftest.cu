// Measurement and test hooks of the library: the FP64 peak microbenchmark (the roofline
// denominator) and the arithmetic-core self-test (phc_arith_test).
#include "runtime.h"
#include "kernels_selftest.cuh"

using namespace phc_rt;

extern "C" {

int phc_arith_test(int32_t op, int32_t limbs, int64_t n, const double* a, const double* b, double* out, void* stream) {
  g_err.clear();
  if (limbs != 2 && limbs != 4) return fail(PHC_EUNSUPPORTED, "limbs must be 2 or 4");
  if (op < 0 || op > 10) return fail(PHC_EINVAL, "unknown op %d", op);
  if (n < 0) return fail(PHC_EINVAL, "n < 0");
  if (n == 0) return PHC_OK;
  if (!a || !b || !out) return fail(PHC_EINVAL, "NULL pointer");
  cudaStream_t st = (cudaStream_t)stream;
  if (op == phc::kCplxRecipWarp) {
    const unsigned wgrid = (unsigned)((n + 3) / 4);
    if (limbs == 2)
      phc::recip_warp_test_kernel<2><<<wgrid, 128, 0, st>>>(n, a, out);
    else
      phc::recip_warp_test_kernel<4><<<wgrid, 128, 0, st>>>(n, a, out);
    CUDA_TRY(cudaGetLastError());
    return PHC_OK;
  }
  const unsigned grid = (unsigned)((n + 127) / 128);
  if (limbs == 2)
    phc::arith_test_kernel<2><<<grid, 128, 0, st>>>(op, n, a, b, out);
  else
    phc::arith_test_kernel<4><<<grid, 128, 0, st>>>(op, n, a, b, out);
  CUDA_TRY(cudaGetLastError());
  return PHC_OK;
}

}  // extern "C"


// ---------------------------------------------------------------------------
// FP64 peak microbenchmark
// ---------------------------------------------------------------------------
namespace {
__global__ void dfma_chains_kernel(double* out, int iters, double a, double b) {
  double r[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) r[c] = threadIdx.x * 1e-9 + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 8; ++c) r[c] = __fma_rn(r[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s += r[c];
  if (s == 12345.678) out[0] = s;
}
}  // namespace

extern "C" int phc_fp64_peak(int32_t device, double ms_target, double* tflops) {
  g_err.clear();
  if (!tflops) return fail(PHC_EINVAL, "NULL out");
  DeviceGuard g(device);
  cudaDeviceProp p;
  CUDA_TRY(cudaGetDeviceProperties(&p, device));
  double* d;
  CUDA_TRY(cudaMalloc(&d, 8));
  const int blocks = p.multiProcessorCount * 8, threads = 256, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) dfma_chains_kernel<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
  cudaEventRecord(e0);
  dfma_chains_kernel<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms1;
  cudaEventElapsedTime(&ms1, e0, e1);
  int reps = std::max(1, (int)(ms_target / std::max(ms1, 1e-3f)));
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) dfma_chains_kernel<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t err = cudaGetLastError();
  cudaFree(d);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (err != cudaSuccess) return fail(PHC_ECUDA, "peak kernel: %s", cudaGetErrorString(err));
  *tflops = 2.0 * blocks * (double)threads * iters * 8 * reps / (ms * 1e-3) / 1e12;
  return PHC_OK;
}
