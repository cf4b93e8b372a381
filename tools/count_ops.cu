// Count the FP64 SASS instructions of each arithmetic-core operation: one kernel per op,
// compiled for sm_100a; tools/count_ops.py disassembles and counts DADD/DMUL/DFMA.
#include "../paper_1109_0545_b200/csrc/arith.cuh"
using namespace phc;
#define OPK(NAME, L, EXPR)                                                          \
  __global__ void NAME(const double* in, double* out) {                             \
    using P = Prec<L>;                                                              \
    auto a = cload<L>(in);                                                          \
    auto b = cload<L>(in + 2 * L);                                                  \
    auto r = EXPR;                                                                  \
    cstore<L>(out, r);                                                              \
  }
OPK(k_dd_cmul, 2, P::mul(a, b))
OPK(k_dd_cmul_lazy, 2, P::mul_lazy(a, b))
OPK(k_dd_cadd, 2, P::add(a, b))
OPK(k_dd_cadd_lazy, 2, P::add_lazy(a, b))
OPK(k_dd_norm, 2, P::norm(a))
OPK(k_dd_cmulint, 2, P::mul_int(a, 3.0))
OPK(k_qd_cmul, 4, P::mul(a, b))
OPK(k_qd_cadd, 4, P::add(a, b))
OPK(k_qd_cmulint, 4, P::mul_int(a, 3.0))
