// Single-thread dependent-chain latency of the DD/QD complex operations (clock cycles per op):
// the serial parts of the eliminations (pivot reciprocal, multiplier, update entry) are
// bound by these, not by FP64 throughput.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1109_0545_b200/csrc tools/op_latency.cu -o /tmp/op_latency
#include <cstdio>
#include "arith.cuh"
using namespace phc;

template <int L, int OP>
__global__ void lat(double* out, long long* cyc, int reps) {
  using P = Prec<L>;
  typename P::C x = P::one(), y = P::one();
  x.re.x[0] = 0.9; x.im.x[0] = 0.3; x.re.x[1] = 1e-17;
  y.re.x[0] = 0.8; y.im.x[0] = -0.6; y.im.x[1] = 3e-18;
  long long t0 = clock64();
  for (int i = 0; i < reps; ++i) {
    if constexpr (OP == 0) x = P::recip(x);
    if constexpr (OP == 1) x = P::mul(x, y);
    if constexpr (OP == 2) x = P::add(x, y);
    if constexpr (OP == 3) x = P::sub(x, P::mul(x, y));
    if constexpr (OP == 4) x.re = P::rdiv(y.re, x.re);
    if constexpr (OP == 5) x.re.x[0] = __ddiv_rn(y.re.x[0], x.re.x[0]);
    if constexpr (OP == 6) x.re.x[0] = __drcp_rn(x.re.x[0]);
    if constexpr (OP == 7) x.re = P::abs2(x);
    if constexpr (OP == 8) x.re.x[0] = __dmul_rn(x.re.x[0], y.re.x[0]);
    if constexpr (OP == 9) {
      if constexpr (L == 2) x.re = dd_div_rc(y.re, x.re);
      else x.re = qd_div_rc(y.re, x.re);
    }
    if constexpr (OP == 10) x.re.x[0] = __ddiv_rn(y.re.x[0], x.re.x[0] + 1e-300 * i);
  }
  long long t1 = clock64();
  out[0] = x.re.x[0] + x.im.x[0];
  cyc[0] = (t1 - t0) / reps;
}

int main() {
  double* o;
  long long* c;
  cudaMalloc(&o, 8);
  cudaMalloc(&c, 8);
  const char* names[] = {"recip", "mul", "add", "x - x*y", "rdiv", "ddiv", "drcp", "abs2", "dmul", "rdiv_rc", "ddiv2"};
  long long h;
#define RUN(L, OP)                                  \
  lat<L, OP><<<1, 1>>>(o, c, 64);                   \
  lat<L, OP><<<1, 1>>>(o, c, 256);                  \
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);     \
  printf("L=%d %-8s %lld cycles\n", L, names[OP], h);
  RUN(2, 0) RUN(2, 1) RUN(2, 2) RUN(2, 3) RUN(2, 4) RUN(2, 7) RUN(4, 0) RUN(4, 1) RUN(4, 2) RUN(4, 3) RUN(4, 4) RUN(4, 7)
  RUN(2, 5) RUN(2, 6) RUN(2, 8) RUN(2, 9) RUN(4, 9) RUN(2, 10)
  return 0;
}
