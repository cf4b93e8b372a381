// Self-test hook of the arithmetic core (pin P12): applies one DD/QD
// operation elementwise to device arrays so that tests/test_gpu_arith.py can check the
// error-free transformations for exactness and the DD/QD operations for accuracy against
// exact rationals.  Not on the evaluation path.
#pragma once
#include "arith.cuh"
#include "kernels_newton.cuh"

namespace phc {

enum ArithOp {
  kTwoSum = 0,    // a, b, out: [n] doubles -> out [n][2] = (s, e)
  kTwoProd = 1,   // same layout, (p, e)
  kRealAdd = 2,   // a, b, out: [n][L] real limbs
  kRealMul = 3,
  kRealDiv = 4,
  kCplxMul = 5,   // a, b, out: [n][2][L] complex
  kCplxAdd = 6,
  kCplxMulLazyNorm = 7,  // the hot path's lazy product followed by its renormalisation
  kCplxRecip = 8,        // out = 1 / a
  kRealMulD = 9,         // out = a * b[.][0] (QD x double / DD x double)
  kCplxRecipWarp = 10,   // out = 1 / a by recip_warp (kernels_newton.cuh), one warp per element
};

template <int L>
__global__ void arith_test_kernel(int op, int64_t n, const double* __restrict__ a, const double* __restrict__ b,
                                  double* __restrict__ out) {
  using P = Prec<L>;
  using C = typename P::C;
  using R = typename P::real;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  auto rl = [&](const double* p) { return P::rload(p + i * L); };
  auto rs = [&](const R& v) { P::rstore(out + i * L, v); };
  auto cl = [&](const double* p) {
    C v;
    for (int q = 0; q < L; ++q) { v.re.x[q] = p[(i * 2) * L + q]; v.im.x[q] = p[(i * 2 + 1) * L + q]; }
    return v;
  };
  auto cs = [&](const C& v) {
    for (int q = 0; q < L; ++q) { out[(i * 2) * L + q] = v.re.x[q]; out[(i * 2 + 1) * L + q] = v.im.x[q]; }
  };
  switch (op) {
    case kTwoSum: {
      double s, e;
      two_sum(a[i], b[i], s, e);
      out[2 * i] = s;
      out[2 * i + 1] = e;
      break;
    }
    case kTwoProd: {
      double p, e;
      two_prod(a[i], b[i], p, e);
      out[2 * i] = p;
      out[2 * i + 1] = e;
      break;
    }
    case kRealAdd: rs(P::radd(rl(a), rl(b))); break;
    case kRealMul: rs(P::rmul(rl(a), rl(b))); break;
    case kRealDiv: rs(P::rdiv(rl(a), rl(b))); break;
    case kCplxMul: cs(P::mul(cl(a), cl(b))); break;
    case kCplxAdd: cs(P::add(cl(a), cl(b))); break;
    case kCplxMulLazyNorm: cs(P::norm(P::mul_lazy(cl(a), cl(b)))); break;
    case kCplxRecip: cs(P::recip(cl(a))); break;
    case kRealMulD: {
      if constexpr (L == 2) rs(dd_mul_d(rl(a), b[i * L]));
      else rs(qd_mul_d(rl(a), b[i * L]));
      break;
    }
    default: break;
  }
}

// op 10: one warp per element, the eliminations' two-lane reciprocal
template <int L>
__global__ void recip_warp_test_kernel(int64_t n, const double* __restrict__ a, double* __restrict__ out) {
  using P = Prec<L>;
  const int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= n) return;  // warp-uniform
  typename P::C v;
  for (int q = 0; q < L; ++q) { v.re.x[q] = a[(i * 2) * L + q]; v.im.x[q] = a[(i * 2 + 1) * L + q]; }
  const typename P::C r = recip_warp<L>(v, lane);
  if (lane == 0)
    for (int q = 0; q < L; ++q) { out[(i * 2) * L + q] = r.re.x[q]; out[(i * 2 + 1) * L + q] = r.im.x[q]; }
}

}  // namespace phc
