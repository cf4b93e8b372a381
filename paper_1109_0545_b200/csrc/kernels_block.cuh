// Fused warp-per-monomial-block kernel: power table, Speelpenning products, coefficient
// product and both reductions in one launch (BASELINE.json
// north_star "one-warp-per-monomial-block Speelpenning products ... warp-shuffle DD/QD
// reduction per polynomial and per Jacobian entry").
//
// Layout (host plan, plan_blocks below):
//  * The terms of polynomial i are cut into blocks of <= 32 terms, one term per lane.
//  * Every lane runs K factor slots (K = compiled bound >= max k; shorter terms are padded
//    with a dummy variable whose power-table row is U = 1, Dd = 0).  The order of a term's
//    factors over the slots is chosen by a bipartite edge colouring (lanes x variables) so
//    that at any slot at most R lanes of a block touch the same variable, and each such
//    lane owns a distinct replica r < R of the Jacobian row accumulator.  The Speelpenning
//    scheme needs no particular factor order (P:549-561 only uses "the product of all
//    factors but one"), so the colouring changes rounding order only.
//  * fac[block][slot][lane] = var | exp << 16 | rep << 24   (coalesced 128 B per slot)
//  * coef[block][lane][2][L]                                (256-bit vector loads)
//
// Per lane (= per term c * prod u_j, u_j = x_{v_j}^{a_j}, d_j = a_j x_{v_j}^{a_j-1}):
//   prefixes r_0 = c, r_m = r_{m-1} u_m and suffixes s_1 = u_K, s_q = s_{q-1} u_{K-q+1}
//   (the paper's psi with c folded in, and phi) run simultaneously, two dependency chains
//   (do_block); g_m = r_{m-1} d_m s_{K-m}; value y = r_K.  g_m is added into
//   row[rep][var] in shared memory (conflict-free by the colouring), slot after slot; y is
//   reduced over the warp with a shuffle tree.
// That is 4K-3 complex products per term, against the paper's 6k-5.
//
// Work split (fixed per system, so every point is evaluated bitwise identically):
//  * mode A (short polynomials or light terms, plan_blocks): a CTA takes one point and a
//    group of polynomials (the whole point for batches); warp w owns polynomials w, w+NW,
//    ...; it accumulates all their blocks in its private rows and writes F[i] and J[i][:]
//    itself (the grouping does not change any polynomial's arithmetic).
//  * mode B (>= 4 blocks per polynomial, or >= 2 with K >= 12): a CTA takes one (point,
//    polynomial); warp w owns blocks w, w+NW, ...; the CTA sums the warps' rows in warp order.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <map>
#include <mutex>
#include <vector>

#include "arith.cuh"

namespace phc {

constexpr int kWarp = 32;
// Layout 2: factor words pre-decoded on the host: the power-table entry e of (var, exp) (the
// dummy variable's U(1) entry for padding) and the accumulator row (the spare row n_var for
// padding), as e | row << 16 (1) or as the byte offset e * 128 | row << 24 (2: the offset is
// added to per-lane chunk-plane pointers; layout 2 implies (n_var + 1) 2E <= 800, n_var < 100):
// no index arithmetic or dummy test per factor on the device
#ifndef PHC_L2_PREDECODE
#define PHC_L2_PREDECODE 2
#endif
#ifndef PHC_DD_DEFER_RMW
#define PHC_DD_DEFER_RMW 1
#endif
// Warps per CTA (NW); the other layouts run 8 warps in one CTA per SM.
// Layout 2 runs 4-warp CTAs, two per SM (252 registers x 128 threads x 2 fits the register
// file, 2 x ~99 KB shared memory), each CTA covering a whole point's polynomials
// (PHC_PPC_MULT): one CTA's power-table prologue and row-total epilogue overlap the other's
// term work -- batch DD 4.57 -> 4.71 M evals/s against one 8-warp CTA per SM.
#ifndef PHC_DD_L2_WARPS
#define PHC_DD_L2_WARPS 4
#endif
#ifndef PHC_OTHER_WARPS
#define PHC_OTHER_WARPS 8
#endif
__host__ __device__ constexpr int block_warps(int L, int layout) {
  return (L == 2 && layout == 2) ? PHC_DD_L2_WARPS : PHC_OTHER_WARPS;
}
constexpr uint32_t kDummyVar = 0xFFFFu;
#ifndef PHC_JUNK_ROW
#define PHC_JUNK_ROW 1
#endif

struct BlockTables {
  uint32_t* fac = nullptr;
  double* coeff = nullptr;
  double* coeff2 = nullptr;  // homotopy target coefficients (NEXT-3), packed like coeff
  int32_t* blk = nullptr;  // poly_blk_ptr [n_eq + 1]
  double* PT = nullptr;    // global power table scratch (layout 0)
  int64_t pt_cap = 0;
};

struct HostBlockPlan {
  bool usable = false;
  int K = 0;           // slots per lane (compiled bound)
  int R = 1;           // replicas per row
  int E = 1;           // max exponent
  int mode = 0;        // 0 = A, 1 = B
  int nw = 8;          // warps per CTA (mode B: min(8, blocks per polynomial)); fixed per system
  int polys_per_cta = 1;
  int layout = 1;      // see LAYOUT above
  int64_t n_blocks = 0;
  size_t smem_bytes = 0;
  std::vector<uint32_t> fac;
  std::vector<double> coeff;
  std::vector<int32_t> blk;
  std::vector<int64_t> slot_term;  // [n_blocks * 32]: term of (block, lane), -1 for padding
  int64_t cm_per_point = 0;
  int64_t ca_per_point = 0;
  int64_t exec_flops_per_point = 0;
  int launches = 1;
};

// Executed FP64 flops (DADD = DMUL = 1, DFMA = 2) of the arithmetic core's operations,
// counted from arith.cuh (and checked against ncu's sm__sass_thread_inst_executed_op_d*):
// complex mul, lazy complex mul, complex add, lazy complex add, renormalisation,
// complex times small integer.
// complex times small integer, renormalisation of a lazy product inside an accumulator update.
struct OpFlops { int cm, cm_lazy, ca, ca_lazy, norm, ci, acc_norm; };
inline OpFlops op_flops(int L) {
  if (L == 2) return {50, 44, 22, 16, 12, 16, 0};
  if (PHC_QD_LAZY && PHC_QD_LAZY_ACC) return {468, 408, 183, 82, 60, 130, 0};
  if (PHC_QD_LAZY) return {468, 408, 183, 183, 60, 130, 60};
  return {468, 468, 183, 183, 0, 130, 0};
}

struct BlockArgs {
  const uint32_t* fac;
  const double* coef;
  const double* coef2;  // NEXT-3: target coefficients (packed like coef) or nullptr
  const double* T;      // NEXT-3: t per point [n_points][L] (real limbs) when coef2 != nullptr
  const int32_t* blk;
  const double* X;
  const double* PTg;
  double* F;
  double* J;
  int64_t n_points;
  int n_eq, n_var, E, R, mode, polys_per_cta;
};

// ---------------------------------------------------------------------------
// device helpers: shared-memory complex access and warp shuffles
// ---------------------------------------------------------------------------
template <int L>
PHC_DEV typename Prec<L>::C shfl_down(const typename Prec<L>::C& v, int d) {
  typename Prec<L>::C r;
#pragma unroll
  for (int i = 0; i < L; ++i) {
    r.re.x[i] = __shfl_down_sync(0xffffffffu, v.re.x[i], d);
    r.im.x[i] = __shfl_down_sync(0xffffffffu, v.im.x[i], d);
  }
  return r;
}
// lane 0 receives the sum over the warp in a fixed tree order (lazy adds, one final
// renormalisation)
template <int L>
PHC_DEV typename Prec<L>::C warp_sum(typename Prec<L>::C v) {
#pragma unroll
  for (int d = 16; d >= 1; d >>= 1) v = Prec<L>::add_lazy(v, shfl_down<L>(v, d));
  return Prec<L>::norm(v);
}


// x^e for 0 <= e < 256 by binary powering (square-and-multiply from the top bit): at most
// 2 log2(e) products on the dependency path instead of e - 1.
template <int L>
PHC_DEV typename Prec<L>::C cpow(const typename Prec<L>::C& x, int e) {
  using P = Prec<L>;
  if (e == 0) return P::one();
  int top = 31 - __clz(e);
  typename P::C r = x;
  for (int b = top - 1; b >= 0; --b) {
    r = P::mul(r, r);
    if ((e >> b) & 1) r = P::mul(r, x);
  }
  return r;
}

// Global power table for configurations whose table does not fit in shared memory (row
// a2, reading C4): one thread per entry (point, variable, a), U[a-1] = x^a and
// Dd[a-1] = a x^(a-1), both from one binary powering x^(a-1); the dummy row is U = 1,
// Dd = 0.  Dependency path <= 4 products (E <= 8) instead of 2E - 1 for a sequential row.
// Launched as the primary of a programmatic dependent launch: the block kernel starts
// while this one runs and waits (griddepcontrol.wait) before it reads the table.
template <int L>
__global__ void block_power_table_kernel(const double* __restrict__ X, int n_var, int E, int64_t n_points,
                                         double* __restrict__ PT) {
  using P = Prec<L>;
  asm volatile("griddepcontrol.launch_dependents;");
  const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t per = (int64_t)(n_var + 1) * E;
  if (gid >= n_points * per) return;
  const int64_t p = gid / per;
  const int r = (int)(gid % per);
  const int v = r / E, a = r % E + 1;
  double* row = PT + (p * (n_var + 1) + v) * (2 * E) * (2 * L);
  if (v == n_var) {
    cstore<L>(row + (a - 1) * 2 * L, P::one());
    cstore<L>(row + (E + a - 1) * 2 * L, P::zero());
    return;
  }
  const typename P::C x = cload<L>(X + (p * n_var + v) * 2 * L);
  const typename P::C pm = cpow<L>(x, a - 1);
  cstore<L>(row + (a - 1) * 2 * L, a == 1 ? x : P::mul(pm, x));
  cstore<L>(row + (E + a - 1) * 2 * L, a == 1 ? pm : P::mul_int(pm, (double)a));
}

// Shared-memory layouts of the power table (PT) and of the Jacobian row accumulators.
//  LAYOUT 0: PT in global memory ([v][2E][2L], per point), rows in shared memory as R
//            replicas [r][v][2L] per warp.
//  LAYOUT 1: PT in shared memory ([v][2E][2L]), rows as in layout 0.
//  LAYOUT 2: "class-interleaved" (small n): lane class c = lane & 7 owns a private copy of
//            the PT and of the rows; chunk j (a double2) of entry e of class c lives at
//            double2 index (j * NE + e) * 8 + c.  The 8 lanes of a quarter-warp (which one
//            LDS.128/STS.128 wavefront serves) are the 8 classes, so every access is
//            bank-conflict free whatever variables the lanes touch.  Rows need no replicas:
//            the edge colouring keeps the 4 lanes of a class on distinct variables per slot.
constexpr int kClasses = 8;

template <int L>
PHC_DEV void cls_store(double2* base, int NE, int e, int c, const typename Prec<L>::C& v) {
  double d[2 * L];
#pragma unroll
  for (int i = 0; i < L; ++i) { d[i] = v.re.x[i]; d[L + i] = v.im.x[i]; }
#pragma unroll
  for (int j = 0; j < L; ++j) base[((size_t)j * NE + e) * kClasses + c] = make_double2(d[2 * j], d[2 * j + 1]);
}
template <int L>
PHC_DEV typename Prec<L>::C cls_load(const double2* base, int NE, int e, int c) {
  double d[2 * L];
#pragma unroll
  for (int j = 0; j < L; ++j) {
    const double2 q = base[((size_t)j * NE + e) * kClasses + c];
    d[2 * j] = q.x;
    d[2 * j + 1] = q.y;
  }
  typename Prec<L>::C v;
#pragma unroll
  for (int i = 0; i < L; ++i) { v.re.x[i] = d[i]; v.im.x[i] = d[L + i]; }
  return v;
}

// One block of 32 terms on one warp: Speelpenning products + accumulation into the
// warp's rows in shared memory; returns the warp-reduced term sum on lane 0.
//
// Per lane, factors j = 1..K (slot order), u_j = x^{a_j}, d_j = a_j x^{a_j - 1}:
//   prefixes P_0 = c, P_j = P_{j-1} u_j          (the paper's psi_j with c folded in)
//   suffixes S_0 = 1, S_q = S_{q-1} u_{K-q+1}    (the paper's phi_q)
//   g_m = P_{m-1} S_{K-m} d_m                     (c * d/dx of the term for factor m)
//   y   = P_K                                      (the term's value)
// Both chains run at once (the paper's psi and phi recurrences): in phase 1
// (t = 1..H, H = K/2) P_1..P_H and S_1..S_H are formed and P_0..P_{H-1}, S_1..S_{H-1}
// kept; in phase 2 (t = 1..H) the running P_{H+t-1} and S_{H+t-1} each meet a kept
// partner, giving g_{H+t} = P_{H+t-1} S_{H-t} d_{H+t} and g_{H-t+1} = P_{H-t} S_{H+t-1}
// d_{H-t+1}, before both chains advance.  4K-3 complex products, critical path K
// products (two independent chains) instead of 2K-2 for a backward-then-forward sweep.
//
// Homotopy (NEXT-3): when hom, the coefficient is the blend
// c(t) = (1 - t) c_start + t c_target (reading H1), formed here before it is folded into P_0.

template <int L, int K, int LAYOUT, bool HOM>
PHC_DEV typename Prec<L>::C do_block(const BlockArgs& a, int64_t b, const double* pt, double* rows, int lane,
                                     const typename Prec<L>::real& omt, const typename Prec<L>::real& tt) {
  using P = Prec<L>;
  using C = typename P::C;
  constexpr int H = K / 2;
  static_assert(K % 2 == 0, "K must be even");
  const int twoE = 2 * a.E;
  const int cls = lane & (kClasses - 1);
  const int NE = (a.n_var + 1) * twoE;
  const uint32_t* fw = a.fac + (size_t)b * K * kWarp + lane;
  // entry index of U(var, exp) in the power table; Dd is E entries further
  // PHC_L2_PREDECODE == 2: word = (entry * 128) | row << 24, the entry's byte offset within a
  // chunk plane of the class-interleaved table (8 classes x 16 bytes per entry)
  constexpr bool L2B = (LAYOUT == 2 && PHC_L2_PREDECODE == 2);
  const int dd_off = L2B ? a.E * 128 : a.E;  // U -> Dd entry (index or byte offset)
  const char* ptc0 = L2B ? reinterpret_cast<const char*>(pt) + cls * 16 : nullptr;
  const char* ptc1 = L2B ? ptc0 + (size_t)NE * 128 : nullptr;
  auto entry = [&](uint32_t word) {
    if constexpr (L2B) {
      PHC_CHECK((word & 0x1ffffu) < (uint32_t)((a.n_var + 1) * twoE * 128));
      return (int)(word & 0x1ffffu);
    } else if constexpr (LAYOUT == 2 && PHC_L2_PREDECODE) {
      PHC_CHECK((word & 0xffffu) < (uint32_t)((a.n_var + 1) * twoE));
      return (int)(word & 0xffffu);
    }
    uint32_t v = word & 0xffffu;
    v = (v == kDummyVar) ? (uint32_t)a.n_var : v;
    const uint32_t ex = (word >> 16) & 0xffu;
    PHC_CHECK(v <= (uint32_t)a.n_var && ex >= 1 && ex <= (uint32_t)a.E);
    return (int)(v * twoE + ex - 1);
  };
  auto ld = [&](int e) -> C {
    if constexpr (L2B) {
      const double2 q0 = *reinterpret_cast<const double2*>(ptc0 + e);
      const double2 q1 = *reinterpret_cast<const double2*>(ptc1 + e);
      C v;
      v.re.x[0] = q0.x; v.re.x[1] = q0.y; v.im.x[0] = q1.x; v.im.x[1] = q1.y;
      return v;
    } else if constexpr (LAYOUT == 2) return cls_load<L>(reinterpret_cast<const double2*>(pt), NE, e, cls);
    else if constexpr (LAYOUT == 1) return row_ld<L>(pt, (size_t)e);
    else return cload<L>(pt + (size_t)e * 2 * L);
  };
  auto word_at = [&](int j) { return __ldg(fw + (j - 1) * kWarp); };  // factor j, 1-based
  // accumulate contribution g of factor word into the warp's row (all lanes in step).  Layout
  // 2 (PHC_JUNK_ROW): the padding slots (dummy variable, g = 0) add into a spare row n_var
  // instead of branching around the update -- no divergent branch per slot, batch DD +5%.
  // (The QD layouts keep the branch: the spare row cost them registers, c3 x1,024 -5%.)
  constexpr bool junk = PHC_JUNK_ROW && LAYOUT == 2;
  const int RS = a.n_var + (junk ? 1 : 0);  // row stride (per class / per replica)
  auto rmw = [&](uint32_t word, const C& g) {
    const uint32_t v = word & 0xffffu;
    if constexpr (junk && L2B) {
      const int ro = (int)(word >> 24) * 128;  // byte offset of the row entry within a chunk plane
      PHC_CHECK((word >> 24) <= (uint32_t)a.n_var);
      char* r0 = reinterpret_cast<char*>(rows) + cls * 16 + ro;
      char* r1 = r0 + (size_t)RS * 128;
      const double2 q0 = *reinterpret_cast<const double2*>(r0);
      const double2 q1 = *reinterpret_cast<const double2*>(r1);
      C acc;
      acc.re.x[0] = q0.x; acc.re.x[1] = q0.y; acc.im.x[0] = q1.x; acc.im.x[1] = q1.y;
      acc = P::accum(acc, g);
      *reinterpret_cast<double2*>(r0) = make_double2(acc.re.x[0], acc.re.x[1]);
      *reinterpret_cast<double2*>(r1) = make_double2(acc.im.x[0], acc.im.x[1]);
    } else if constexpr (junk) {
      const int vr = PHC_L2_PREDECODE ? (int)(word >> 16) : ((v == kDummyVar) ? a.n_var : (int)v);
      PHC_CHECK(vr <= a.n_var);
      double2* rw = reinterpret_cast<double2*>(rows);
      cls_store<L>(rw, RS, vr, cls, P::accum(cls_load<L>(rw, RS, vr, cls), g));
    } else if (v != kDummyVar) {
      PHC_CHECK(v < (uint32_t)a.n_var && (LAYOUT == 2 || (word >> 24) < (uint32_t)a.R));
      if constexpr (LAYOUT == 2) {
        double2* rw = reinterpret_cast<double2*>(rows);
        cls_store<L>(rw, RS, (int)v, cls, P::accum(cls_load<L>(rw, RS, (int)v, cls), g));
      } else {
        const size_t idx = (size_t)(word >> 24) * a.n_var + v;
        row_st<L>(rows, idx, P::accum(row_ld<L>(rows, idx), g));
      }
    }
    __syncwarp();
  };
  C Pk[H];  // P_0 .. P_{H-1}
  C Sk[H];  // S_1 .. S_{H-1} at Sk[1..H-1]
  C p = cload<L>(a.coef + ((size_t)b * kWarp + lane) * 2 * L);  // running P
  if constexpr (HOM)
    p = P::add(P::mul_real(p, omt), P::mul_real(cload<L>(a.coef2 + ((size_t)b * kWarp + lane) * 2 * L), tt));
  C q;                                                           // running S
  // phase 1
  auto phase1 = [&](int t, uint32_t w1, uint32_t w2) {  // w1 = word_at(t), w2 = word_at(K - t + 1)
    Pk[t - 1] = p;
    p = P::mul_lazy(p, ld(entry(w1)));
    const C u = ld(entry(w2));
    if (t == 1) {
      q = u;
    } else {
      Sk[t - 1] = q;
      q = P::mul_lazy(q, u);
    }
  };
  // phase 2
  // pk = P_{H-t}, sk = S_{H-t}; wa = word_at(H + t), wb = word_at(H - t + 1)
  auto phase2 = [&](int t, const C& pk, const C& sk, uint32_t wa, uint32_t wb) {
    const int ea = entry(wa), eb = entry(wb);
    C ga = P::mul_lazy(p, ld(ea + dd_off));
    if (t < H) ga = P::mul_lazy(ga, sk);
    C gb = P::mul_lazy(pk, ld(eb + dd_off));
    gb = P::mul_lazy(gb, q);
    p = P::mul_lazy(p, ld(ea));
    if (t < H) q = P::mul_lazy(q, ld(eb));
    rmw(wa, ga);
    rmw(wb, gb);
  };
  if constexpr (L == 2) {
#pragma unroll
    for (int t = 1; t <= H; ++t) phase1(t, word_at(t), word_at(K - t + 1));
#if PHC_DD_DEFER_RMW
    // the accumulator updates of step t are issued after the products of step t+1 (same
    // updates in the same order, so the same bits): the shared-memory read-modify-write
    // latency of a step overlaps the next step's arithmetic instead of stalling the warp
    uint32_t dwa = 0, dwb = 0;
    C dga, dgb;
#pragma unroll
    for (int t = 1; t <= H; ++t) {
      const uint32_t wa = word_at(H + t), wb = word_at(H - t + 1);
      const C pk = Pk[H - t], sk = t < H ? Sk[H - t] : P::one();
      const int ea = entry(wa), eb = entry(wb);
      C ga = P::mul_lazy(p, ld(ea + dd_off));
      if (t < H) ga = P::mul_lazy(ga, sk);
      C gb = P::mul_lazy(pk, ld(eb + dd_off));
      gb = P::mul_lazy(gb, q);
      p = P::mul_lazy(p, ld(ea));
      if (t < H) q = P::mul_lazy(q, ld(eb));
      if (t > 1) {
        rmw(dwa, dga);
        rmw(dwb, dgb);
      }
      dwa = wa, dwb = wb, dga = ga, dgb = gb;
    }
    rmw(dwa, dga);
    rmw(dwb, dgb);
#else
#pragma unroll
    for (int t = 1; t <= H; ++t)
      phase2(t, Pk[H - t], t < H ? Sk[H - t] : P::one(), word_at(H + t), word_at(H - t + 1));
#endif
  } else {
    // rolled loops (the QD body is thousands of instructions): the factor words are
    // fetched one step ahead, so the table gathers of a step do not wait on them
    uint32_t w1 = word_at(1), w2 = word_at(K);
#pragma unroll 1
    for (int t = 1; t <= H; ++t) {
      const uint32_t c1 = w1, c2 = w2;
      if (t < H) {
        w1 = word_at(t + 1);
        w2 = word_at(K - t);
      } else {
        w1 = word_at(H + 1);
        w2 = word_at(H);
      }
      phase1(t, c1, c2);
    }
    // the kept values live in local memory here: fetch them one step ahead
    C pk_n = Pk[H - 1], sk_n = (H > 1) ? Sk[H - 1] : P::one();
#pragma unroll 1
    for (int t = 1; t <= H; ++t) {
      const C pk = pk_n, sk = sk_n;
      const uint32_t wa = w1, wb = w2;
      if (t < H) {
        pk_n = Pk[H - t - 1];
        sk_n = (t + 1 < H) ? Sk[H - t - 1] : P::one();
        w1 = word_at(H + t + 1);
        w2 = word_at(H - t);
      }
      phase2(t, pk, sk, wa, wb);
    }
  }
  return warp_sum<L>(P::norm(p));
}

// Number of doubles of one warp's row accumulators (layout 2: n_var + PHC_JUNK_ROW rows per
// class, the spare one taking the padding slots' zero contributions).
__host__ __device__ inline size_t row_doubles(int layout, int R, int n_var, int L) {
  return layout == 2 ? (size_t)kClasses * (n_var + PHC_JUNK_ROW) * 2 * L : (size_t)R * n_var * 2 * L;
}

// Sum of a warp's accumulators for variable v (replicas r = 0..R-1 or classes, in a fixed
// order); lazy adds, NOT renormalised (the caller renormalises once).
template <int L, int LAYOUT>
PHC_DEV typename Prec<L>::C row_total(const double* rows, int R, int n_var, int v) {
  using P = Prec<L>;
  typename P::C acc;
  if constexpr (LAYOUT == 2) {
    // classes are visited in the order v, v+1, ... (mod 8): a fixed order per variable that
    // keeps the 8 lanes of a quarter-warp on 8 different banks
    const double2* rw = reinterpret_cast<const double2*>(rows);
    acc = cls_load<L>(rw, n_var + PHC_JUNK_ROW, v, v & (kClasses - 1));
    for (int c = 1; c < kClasses; ++c)
      acc = P::add_lazy(acc, cls_load<L>(rw, n_var + PHC_JUNK_ROW, v, (v + c) & (kClasses - 1)));
  } else {
    acc = row_ld<L>(rows, (size_t)v);
    for (int r = 1; r < R; ++r) acc = P::add_lazy(acc, row_ld<L>(rows, (size_t)r * n_var + v));
  }
  return acc;
}

// HOM: homotopy coefficients (NEXT-3) -- a separate instantiation, so the plain evaluation
// carries none of the blend's code or registers.
template <int L, int K, int LAYOUT, bool HOM>
__global__ void __launch_bounds__(block_warps(L, LAYOUT) * kWarp, 1)
block_kernel(const BlockArgs a) {
  using P = Prec<L>;
  using C = typename P::C;
  const int kBlockWarps = blockDim.x >> 5;  // the plan's warps per CTA
  extern __shared__ __align__(16) double smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int cd = 2 * L;
  const int twoE = 2 * a.E;
  const int64_t units_per_point =
      a.mode == 0 ? (a.n_eq + a.polys_per_cta - 1) / a.polys_per_cta : (int64_t)a.n_eq;
  const int64_t p = blockIdx.x / units_per_point;
  const int unit = (int)(blockIdx.x % units_per_point);
  if (p >= a.n_points) return;
  typename P::real tt = P::one().re, omt = P::one().re;
  if constexpr (HOM) {
    tt = P::rload(a.T + p * L);
    omt = P::one_minus(tt);
  }

  double* pt;
  double* rows_all;
  if constexpr (LAYOUT == 0) {
    pt = const_cast<double*>(a.PTg) + p * (int64_t)(a.n_var + 1) * twoE * cd;
    rows_all = smem;
    // dependent launch: the power table of the primary kernel is complete and visible
    asm volatile("griddepcontrol.wait;" ::: "memory");
  } else {
    pt = smem;
    const int NE = (a.n_var + 1) * twoE;
    rows_all = smem + (size_t)NE * cd * (LAYOUT == 2 ? kClasses : 1);
    if constexpr (LAYOUT == 1) {
      // one thread per variable: U = x^e and Dd = e x^(e-1) by repeated multiplication, stored
      // as swizzled entries (row_st, like the row accumulators); the dummy row is U = 1, Dd = 0
      for (int v = threadIdx.x; v <= a.n_var; v += blockDim.x) {
        const size_t e0 = (size_t)v * twoE;
        C pw = P::one();
        const C x = (v == a.n_var) ? P::one() : cload<L>(a.X + (p * a.n_var + v) * cd);
        for (int e = 1; e <= a.E; ++e) {
          C dd = (e == 1) ? pw : P::mul_int(pw, (double)e);
          pw = (e == 1) ? x : P::mul(pw, x);
          if (v == a.n_var) dd = P::zero();
          row_st<L>(pt, e0 + e - 1, pw);
          row_st<L>(pt, e0 + a.E + e - 1, dd);
        }
      }
    } else {
      // one thread per (variable, class): each computes the row (E-1 products; cheap)
      // and stores its class copy; the 8 threads of a quarter-warp write 8 classes of the
      // same entry, i.e. 8 different banks
      double2* pt2 = reinterpret_cast<double2*>(pt);
      for (int idx = threadIdx.x; idx < (a.n_var + 1) * kClasses; idx += blockDim.x) {
        const int v = idx / kClasses, c = idx % kClasses;
        C pw = P::one();
        const C x = (v == a.n_var) ? P::one() : cload<L>(a.X + (p * a.n_var + v) * cd);
        for (int e = 1; e <= a.E; ++e) {
          C dd = (e == 1) ? pw : P::mul_int(pw, (double)e);
          pw = (e == 1) ? x : P::mul(pw, x);
          if (v == a.n_var) dd = P::zero();
          cls_store<L>(pt2, NE, v * twoE + e - 1, c, pw);
          cls_store<L>(pt2, NE, v * twoE + a.E + e - 1, c, dd);
        }
      }
    }
  }
  const size_t row_elems = row_doubles(LAYOUT, a.R, a.n_var, L);
  double* rows = rows_all + warp * row_elems;
  double* fpart = rows_all + kBlockWarps * row_elems;  // mode B: per-warp F partials
  __syncthreads();

  // One loop for both modes, with a single call site of do_block (the QD instance is
  // thousands of instructions; two call sites would double the kernel's code footprint).
  //  mode A: warp w takes polynomials i0+w, i0+w+NW, ... and all their blocks;
  //  mode B: every warp takes polynomial `unit`, blocks blk[i]+w, blk[i]+w+NW, ...
  const bool mA = (a.mode == 0);
  const int i_first = mA ? unit * a.polys_per_cta + warp : unit;
  const int i_end = mA ? min(a.n_eq, (unit + 1) * a.polys_per_cta) : unit + 1;
  const int i_step = mA ? kBlockWarps : 1;
  for (int i = i_first; i < i_end; i += i_step) {
    for (size_t e = lane; e < row_elems / 2; e += kWarp) reinterpret_cast<double2*>(rows)[e] = make_double2(0.0, 0.0);
    __syncwarp();
    C fsum = P::zero();
    const int b_step = mA ? 1 : kBlockWarps;
    for (int b = a.blk[i] + (mA ? 0 : warp); b < a.blk[i + 1]; b += b_step) {
      C y = do_block<L, K, LAYOUT, HOM>(a, b, pt, rows, lane, omt, tt);
      fsum = P::add(fsum, y);
    }
    __syncwarp();
    double* jrow = a.J + (p * a.n_eq + i) * (int64_t)a.n_var * cd;
    if (mA) {
      if (lane == 0) cstore<L>(a.F + (p * a.n_eq + i) * cd, fsum);
      for (int v = lane; v < a.n_var; v += kWarp)
        cstore<L>(jrow + (size_t)v * cd, P::norm(row_total<L, LAYOUT>(rows, a.R, a.n_var, v)));
      __syncwarp();
    } else {
      if (lane == 0) sstore<L>(fpart + warp * cd, fsum);
      __syncthreads();
      if (threadIdx.x == 0) {
        C f = sload<L>(fpart);
        for (int w2 = 1; w2 < kBlockWarps; ++w2) f = P::add(f, sload<L>(fpart + w2 * cd));
        cstore<L>(a.F + (p * a.n_eq + i) * cd, f);
      }
      for (int v = threadIdx.x; v < a.n_var; v += blockDim.x) {
        C acc = row_total<L, LAYOUT>(rows_all, a.R, a.n_var, v);
        for (int w2 = 1; w2 < kBlockWarps; ++w2)
          acc = P::add_lazy(acc, row_total<L, LAYOUT>(rows_all + w2 * row_elems, a.R, a.n_var, v));
        cstore<L>(jrow + (size_t)v * cd, P::norm(acc));
      }
    }
  }
}

// ---------------------------------------------------------------------------
// host side: plan (blocks, edge colouring, packing), upload, launch
// ---------------------------------------------------------------------------
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, device) and size: the
// attribute call costs microseconds, and the tracker's corrector launches thousands of times.
inline cudaError_t ensure_smem(const void* func, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void*, int>, size_t> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  size_t& v = done[{func, dev}];
  if (v >= bytes) return cudaSuccess;
  const cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e == cudaSuccess) v = bytes;
  return e;
}

inline int compiled_K(int kmax) {
  static const int ks[] = {2, 4, 8, 12, 16, 20, 24, 32};
  for (int k : ks)
    if (kmax <= k) return k;
  return 0;
}

// Colour the edges (lane, var-replica) of one block with K colours so that no two edges
// at a lane or at a replica node share a colour (Konig: possible when every degree <= K).
// in: terms[lane] = list of (var, exp); out: slot[lane][j] for factor j, rep[lane][j].
inline bool colour_block(const std::vector<std::vector<std::pair<int, int>>>& terms, int n_var, int K, int R,
                         std::vector<std::vector<int>>* slot, std::vector<std::vector<int>>* rep) {
  const int nl = (int)terms.size();
  // replica assignment: round-robin over the occurrences of each variable (lane order)
  std::vector<int> seen(n_var, 0);
  rep->assign(nl, {});
  slot->assign(nl, {});
  for (int l = 0; l < nl; ++l) {
    for (auto& f : terms[l]) (*rep)[l].push_back(seen[f.first]++ % R);
    (*slot)[l].assign(terms[l].size(), -1);
  }
  const int nodes = n_var * R;
  std::vector<int> atL((size_t)nl * K, -1), atR((size_t)nodes * K, -1);  // colour -> neighbour
  std::vector<int> eL((size_t)nl * K, -1), eR((size_t)nodes * K, -1);    // colour -> factor index j
  for (int l = 0; l < nl; ++l) {
    for (int j = 0; j < (int)terms[l].size(); ++j) {
      const int w = terms[l][j].first * R + (*rep)[l][j];
      int ca = -1, cb = -1;
      for (int c = 0; c < K && ca < 0; ++c)
        if (atL[(size_t)l * K + c] < 0) ca = c;
      for (int c = 0; c < K && cb < 0; ++c)
        if (atR[(size_t)w * K + c] < 0) cb = c;
      if (ca < 0 || cb < 0) return false;
      if (atR[(size_t)w * K + ca] >= 0) {
        // flip the ca/cb alternating path starting at replica node w
        std::vector<std::pair<int, int>> path;  // (right node, left node) pairs along the path
        int rn = w, c = ca;
        while (true) {
          const int ln = atR[(size_t)rn * K + c];
          if (ln < 0) break;
          path.push_back({rn, ln});
          const int c2 = (c == ca) ? cb : ca;
          const int rn2 = atL[(size_t)ln * K + c2];
          if (rn2 < 0) break;
          path.push_back({rn2, ln});
          rn = rn2;
          c = (c2 == ca) ? cb : ca;
          if (path.size() > (size_t)4 * (nl + nodes)) return false;
        }
        // recolour every edge on the path: swap ca <-> cb
        struct Ed { int l, r, j, c; };
        std::vector<Ed> eds;
        for (size_t q = 0; q < path.size(); ++q) {
          const int rr = path[q].first, ll = path[q].second;
          const int cc = (q % 2 == 0) ? ca : cb;
          eds.push_back({ll, rr, eL[(size_t)ll * K + cc], cc});
        }
        for (auto& e : eds) {
          atL[(size_t)e.l * K + e.c] = -1;
          atR[(size_t)e.r * K + e.c] = -1;
          eL[(size_t)e.l * K + e.c] = -1;
          eR[(size_t)e.r * K + e.c] = -1;
        }
        for (auto& e : eds) {
          const int nc = (e.c == ca) ? cb : ca;
          atL[(size_t)e.l * K + nc] = e.r;
          atR[(size_t)e.r * K + nc] = e.l;
          eL[(size_t)e.l * K + nc] = e.j;
          eR[(size_t)e.r * K + nc] = e.j;
          (*slot)[e.l][e.j] = nc;
        }
        if (atR[(size_t)w * K + ca] >= 0 || atL[(size_t)l * K + ca] >= 0) return false;
      }
      atL[(size_t)l * K + ca] = w;
      atR[(size_t)w * K + ca] = l;
      eL[(size_t)l * K + ca] = j;
      eR[(size_t)w * K + ca] = j;
      (*slot)[l][j] = ca;
    }
  }
  return true;
}

// Lane placement for layout 2 with few slots: reorder the terms of every block over its lanes
// (lane l has class l % kClasses) so that each (class, var) occurs in at most Kc terms.
// Greedy, heaviest terms first, each to the class with free lanes that keeps its largest
// (class, var) count lowest (ties: most free lanes, then lowest class).  False when some
// block cannot be balanced.
template <class S>
bool balance_lane_classes(const S& s, const std::vector<std::vector<int64_t>>& bterms, int Kc,
                          std::vector<std::vector<int64_t>>* out) {
  std::vector<uint8_t> deg((size_t)kClasses * s.n_var, 0);
  out->assign(bterms.size(), {});
  for (size_t b = 0; b < bterms.size(); ++b) {
    const std::vector<int64_t>& ts = bterms[b];
    const int m = (int)ts.size();
    int cap[kClasses];
    for (int c = 0; c < kClasses; ++c) cap[c] = 0;
    for (int l = 0; l < m; ++l) cap[l % kClasses]++;
    std::vector<int> order(m);
    for (int j = 0; j < m; ++j) order[j] = j;
    std::stable_sort(order.begin(), order.end(), [&](int x, int y) {
      return s.term_ptr[ts[x] + 1] - s.term_ptr[ts[x]] > s.term_ptr[ts[y] + 1] - s.term_ptr[ts[y]];
    });
    std::vector<std::vector<int64_t>> by_class(kClasses);
    bool ok = true;
    for (int j : order) {
      const int64_t t = ts[j];
      int best = -1, best_cost = 1 << 30;
      for (int c = 0; c < kClasses; ++c) {
        if (!cap[c]) continue;
        int cost = 0;
        for (int64_t q = s.term_ptr[t]; q < s.term_ptr[t + 1]; ++q)
          cost = std::max(cost, deg[(size_t)c * s.n_var + (s.fac[q] & 0xffffu)] + 1);
        if (cost < best_cost || (cost == best_cost && cap[c] > cap[best])) {
          best = c;
          best_cost = cost;
        }
      }
      if (best < 0 || best_cost > Kc) {
        ok = false;
        break;
      }
      cap[best]--;
      by_class[best].push_back(t);
      for (int64_t q = s.term_ptr[t]; q < s.term_ptr[t + 1]; ++q) deg[(size_t)best * s.n_var + (s.fac[q] & 0xffffu)]++;
    }
    for (int c = 0; c < kClasses; ++c)  // reset the counts this block touched
      for (int64_t t : by_class[c])
        for (int64_t q = s.term_ptr[t]; q < s.term_ptr[t + 1]; ++q) deg[(size_t)c * s.n_var + (s.fac[q] & 0xffffu)] = 0;
    if (!ok) return false;
    std::vector<int64_t>& lanes = (*out)[b];
    lanes.resize(m);
    int taken[kClasses] = {0};
    for (int l = 0; l < m; ++l) {
      const int c = l % kClasses;
      lanes[l] = by_class[c][taken[c]++];
    }
  }
  return true;
}

template <class S>
void plan_blocks(const S& s, HostBlockPlan* plan) {
  plan->usable = false;
  const int L = s.L;
  const int E = s.E;
  const size_t cdb = (size_t)2 * L * sizeof(double);
  // layout 2 (class-interleaved, DD only) when it fits in shared memory
  const size_t pt1 = (size_t)(s.n_var + 1) * 2 * E * cdb;
  const int nw2 = block_warps(L, 2);
  const size_t l2_bytes = pt1 * kClasses + (size_t)nw2 * kClasses * (s.n_var + PHC_JUNK_ROW) * cdb + nw2 * cdb;
  const int layout = (L == 2 && l2_bytes <= (size_t)200 * 1024) ? 2 : 1;
  int K = compiled_K(std::max(s.kmax, layout == 2 ? 4 : 1));
  if (K == 0 || s.n_var >= (int)kDummyVar) return;
  // blocks
  std::vector<int32_t> blk(1, 0);
  std::vector<std::vector<int64_t>> bterms;
  int max_blocks_per_poly = 0;
  for (int i = 0; i < s.n_eq; ++i) {
    int nb = 0;
    for (int64_t t = s.poly_ptr[i]; t < s.poly_ptr[i + 1]; t += kWarp, ++nb) {
      std::vector<int64_t> ts;
      for (int64_t u = t; u < std::min<int64_t>(t + kWarp, s.poly_ptr[i + 1]); ++u) ts.push_back(u);
      bterms.push_back(ts);
    }
    blk.push_back((int32_t)bterms.size());
    max_blocks_per_poly = std::max(max_blocks_per_poly, nb);
  }
  const int64_t nb = (int64_t)bterms.size();
  // Layout 2 colours (lane, (class, var)) edges: an accumulator (class, var) is shared by the
  // 4 lanes of a class, so K >= 4 in general.  Systems with k <= 2 (quadratic systems, the
  // tracker's total-degree homotopies) can often do with K = 2 slots -- half the padded
  // products -- when the terms of each block are placed on lanes so that no (class, var)
  // is used by more than 2 of them (then a 2-edge-colouring exists, Koenig).  Greedy
  // placement; any block that does not balance keeps the plain order and K = 4.
  std::vector<std::vector<int64_t>> bterms2;
  const bool balanced = layout == 2 && s.kmax <= 2 && balance_lane_classes(s, bterms, 2, &bterms2);
  if (balanced) {
    bterms.swap(bterms2);
    K = 2;
  }
  // replicas needed: max over blocks and variables of ceil(d_v / K)
  int R = 1;
  for (auto& ts : bterms) {
    if (layout == 2) break;  // classes of 4 lanes: every (class, var) degree <= 4 <= K
    std::vector<int> d(s.n_var, 0);
    for (int64_t t : ts)
      for (int64_t q = s.term_ptr[t]; q < s.term_ptr[t + 1]; ++q) d[s.fac[q] & 0xffffu]++;
    for (int v = 0; v < s.n_var; ++v) R = std::max(R, (d[v] + K - 1) / K);
  }
  if (R > 255) return;
  std::vector<uint32_t> fac;
  std::vector<double> coef;
  std::vector<int64_t> slot_term;
  // slot assignment by edge colouring and packing; false when a block does not colour
  auto pack = [&]() -> bool {
    fac.assign((size_t)nb * K * kWarp, 0u);
    coef.assign((size_t)nb * kWarp * 2 * L, 0.0);
    slot_term.assign((size_t)nb * kWarp, -1);
    for (int64_t b = 0; b < nb; ++b) {
      std::vector<std::vector<std::pair<int, int>>> terms;
      for (int64_t t : bterms[b]) {
        std::vector<std::pair<int, int>> f;
        for (int64_t q = s.term_ptr[t]; q < s.term_ptr[t + 1]; ++q)
          f.push_back({(int)(s.fac[q] & 0xffffu), (int)((s.fac[q] >> 16) & 0xffu)});
        terms.push_back(f);
      }
      std::vector<std::vector<int>> slot, rep;
      if (layout == 2) {
        // right nodes are (class, var): lanes of different classes never share an accumulator
        auto cterms = terms;
        for (size_t l = 0; l < cterms.size(); ++l)
          for (auto& f : cterms[l]) f.first += s.n_var * (int)(l % kClasses);
        if (!colour_block(cterms, s.n_var * kClasses, K, 1, &slot, &rep)) return false;
      } else if (!colour_block(terms, s.n_var, K, R, &slot, &rep)) {
        return false;
      }
      const bool predecode = PHC_L2_PREDECODE && layout == 2 && PHC_JUNK_ROW;
      for (int l = 0; l < kWarp; ++l) {
        for (int q = 0; q < K; ++q)
          fac[((size_t)b * K + q) * kWarp + l] =
              predecode ? (PHC_L2_PREDECODE == 2 ? ((uint32_t)(s.n_var * 2 * E) << 7) | ((uint32_t)s.n_var << 24)
                                                 : (uint32_t)(s.n_var * 2 * E) | ((uint32_t)s.n_var << 16))
                        : kDummyVar | (1u << 16);
        if (l >= (int)terms.size()) continue;
        for (size_t j = 0; j < terms[l].size(); ++j) {
          const int q = slot[l][j];
          const uint32_t v = (uint32_t)terms[l][j].first, ex = (uint32_t)terms[l][j].second;
          fac[((size_t)b * K + q) * kWarp + l] =
              predecode ? (PHC_L2_PREDECODE == 2 ? ((v * 2 * E + ex - 1) << 7) | (v << 24) : (v * 2 * E + ex - 1) | (v << 16))
                        : v | (ex << 16) | ((uint32_t)rep[l][j] << 24);
        }
        const int64_t t = bterms[b][l];
        slot_term[(size_t)b * kWarp + l] = t;
        for (int c = 0; c < 2 * L; ++c) coef[((size_t)b * kWarp + l) * 2 * L + c] = s.coeff[(size_t)t * 2 * L + c];
      }
    }
    return true;
  };
  if (!pack()) {
    if (!balanced) return;
    bterms.swap(bterms2);  // the balanced placement did not colour with 2 slots: plain order, K = 4
    K = compiled_K(4);
    if (!pack()) return;
  }
  // mode A (a warp owns whole polynomials, the CTA's power table serves up to 4 nw of them)
  // or mode B (a CTA owns a polynomial, its warps split the blocks, one warp per block up to
  // 8).  Calls with few points take the latency path (kernels_scan.cuh), so this kernel
  // serves batches and large systems.  Mode B pays the power table once per polynomial:
  // worth it for long polynomials (>= 4 blocks) or heavy terms (K >= 12: c3 x 4,096 points
  // 7.1 -> 6.8 us/eval), not for light multi-block ones (a total-degree tracker system with
  // k <= 2: 141 -> 85 us per 1,024 points in mode A).
  plan->mode = (max_blocks_per_poly >= 4 || (max_blocks_per_poly >= 2 && K >= 12)) ? 1 : 0;
  const int nw = plan->mode == 1 ? std::min(max_blocks_per_poly, block_warps(L, layout)) : block_warps(L, layout);
  plan->nw = nw;
  if (layout == 2) {
    plan->layout = 2;
    plan->smem_bytes = pt1 * kClasses + (size_t)nw * kClasses * (s.n_var + PHC_JUNK_ROW) * cdb + nw * cdb;
  } else {
    const size_t rows_bytes = (size_t)nw * R * s.n_var * cdb + nw * cdb;
    plan->layout = pt1 + rows_bytes <= (size_t)160 * 1024 ? 1 : 0;
    plan->smem_bytes = (plan->layout == 1 ? pt1 : 0) + rows_bytes;
    if (plan->smem_bytes > (size_t)200 * 1024) return;
  }
  plan->polys_per_cta = 1;
  plan->K = K;
  plan->R = R;
  plan->E = E;
  plan->n_blocks = nb;
  plan->fac.swap(fac);
  plan->coeff.swap(coef);
  plan->blk.swap(blk);
  plan->slot_term.swap(slot_term);
  // operation counts per point (useful work: real terms and factors only)
  int64_t cm = (int64_t)s.n_var * std::max(0, E - 1);
  for (int64_t t = 0; t < s.n_terms; ++t) {
    const int64_t k = s.term_ptr[t + 1] - s.term_ptr[t];
    if (k >= 1) cm += 4 * k - 3;
  }
  plan->cm_per_point = cm;
  plan->ca_per_point = s.n_factors + s.n_terms +
                       (int64_t)s.n_eq * s.n_var * (plan->layout == 2 ? kClasses - 1 : R - 1);
  plan->launches = plan->layout == 0 ? 2 : 1;
  {
    const OpFlops f = op_flops(L);
    int64_t fl = (int64_t)s.n_var * std::max(0, E - 1) * (f.cm + f.ci);  // power table
    for (int64_t t = 0; t < s.n_terms; ++t) {
      const int64_t k = s.term_ptr[t + 1] - s.term_ptr[t];
      if (k >= 1) fl += (4 * k - 3) * f.cm_lazy + k * (f.ca_lazy + f.acc_norm);
    }
    fl += nb * kWarp * (2 * f.norm + 5 * f.ca_lazy);  // warp shuffle tree of each block's term values
    const int parts = plan->layout == 2 ? kClasses : R;
    fl += (int64_t)s.n_eq * s.n_var * (f.norm + (parts - 1) * f.ca_lazy);  // row totals
    fl += (int64_t)(nb - s.n_eq) * f.ca;  // block sums of F
    plan->exec_flops_per_point = fl;
  }
  plan->usable = true;
}

// NEXT-3: a coefficient table in term order ([n_terms][2][L]) packed like plan.coeff.
inline std::vector<double> pack_block_coeff(const HostBlockPlan& plan, const std::vector<double>& coeff, int L) {
  std::vector<double> out(plan.coeff.size(), 0.0);
  for (size_t q = 0; q < plan.slot_term.size(); ++q) {
    const int64_t t = plan.slot_term[q];
    if (t < 0) continue;
    for (int c = 0; c < 2 * L; ++c) out[q * 2 * L + c] = coeff[(size_t)t * 2 * L + c];
  }
  return out;
}

inline int upload_block_tables(const HostBlockPlan& plan, BlockTables* bt) {
  if (cudaMalloc(&bt->fac, std::max<size_t>(4, plan.fac.size() * 4)) != cudaSuccess) return -2;
  if (cudaMalloc(&bt->coeff, std::max<size_t>(8, plan.coeff.size() * 8)) != cudaSuccess) return -2;
  if (cudaMalloc(&bt->blk, plan.blk.size() * 4) != cudaSuccess) return -2;
  if (cudaMemcpy(bt->fac, plan.fac.data(), plan.fac.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess) return -3;
  if (cudaMemcpy(bt->coeff, plan.coeff.data(), plan.coeff.size() * 8, cudaMemcpyHostToDevice) != cudaSuccess) return -3;
  if (cudaMemcpy(bt->blk, plan.blk.data(), plan.blk.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess) return -3;
  return 0;
}

template <int L, int K, int LAYOUT>
int launch_block_k(const HostBlockPlan& plan, const BlockArgs& a, int64_t n_points, cudaStream_t st) {
  auto kern = a.coef2 ? block_kernel<L, K, LAYOUT, true> : block_kernel<L, K, LAYOUT, false>;
  if (plan.smem_bytes > 48 * 1024)
    if (ensure_smem((const void*)kern, plan.smem_bytes) != cudaSuccess)
      return -3;
  const int64_t units = a.mode == 0 ? (a.n_eq + a.polys_per_cta - 1) / a.polys_per_cta : a.n_eq;
  const int64_t max_grid = (int64_t)1 << 30;
  for (int64_t p0 = 0; p0 < n_points;) {
    const int64_t np = std::min<int64_t>(n_points - p0, max_grid / units);
    BlockArgs b = a;
    b.X = a.X + p0 * a.n_var * 2 * L;
    b.F = a.F + p0 * a.n_eq * 2 * L;
    b.J = a.J + p0 * (int64_t)a.n_eq * a.n_var * 2 * L;
    if (LAYOUT == 0) b.PTg = a.PTg + p0 * (int64_t)(a.n_var + 1) * 2 * a.E * 2 * L;
    if (a.T) b.T = a.T + p0 * L;
    b.n_points = np;
    if (LAYOUT == 0) {
      // programmatic dependent launch after block_power_table_kernel (same stream)
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3((unsigned)(np * units));
      cfg.blockDim = dim3(plan.nw * kWarp);
      cfg.dynamicSmemBytes = plan.smem_bytes;
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      if (cudaLaunchKernelEx(&cfg, kern, b) != cudaSuccess) return -3;
    } else {
      kern<<<(unsigned)(np * units), plan.nw * kWarp, plan.smem_bytes, st>>>(b);
    }
    if (cudaGetLastError() != cudaSuccess) return -3;
    p0 += np;
  }
  return 0;
}

// The block kernels are instantiated in separate translation units (generated by
// __graft_entry__.build(), compiled in parallel); everyone else sees extern declarations.
#define PHC_FOR_EACH_K(X, L, P) X(L, 2, P) X(L, 4, P) X(L, 8, P) X(L, 12, P) X(L, 16, P) X(L, 20, P) X(L, 24, P) X(L, 32, P)
#ifndef PHC_INSTANTIATE_BLOCK
#define PHC_EXTERN_K(L, K, P) \
  extern template int launch_block_k<L, K, P>(const HostBlockPlan&, const BlockArgs&, int64_t, cudaStream_t);
PHC_FOR_EACH_K(PHC_EXTERN_K, 2, 0)
PHC_FOR_EACH_K(PHC_EXTERN_K, 2, 1)
PHC_FOR_EACH_K(PHC_EXTERN_K, 2, 2)
PHC_FOR_EACH_K(PHC_EXTERN_K, 4, 0)
PHC_FOR_EACH_K(PHC_EXTERN_K, 4, 1)
#undef PHC_EXTERN_K
#endif

template <int L, int LAYOUT>
int launch_block_pts(const HostBlockPlan& plan, const BlockArgs& a, int64_t np, cudaStream_t st) {
  switch (plan.K) {
    case 2: return launch_block_k<L, 2, LAYOUT>(plan, a, np, st);
    case 4: return launch_block_k<L, 4, LAYOUT>(plan, a, np, st);
    case 8: return launch_block_k<L, 8, LAYOUT>(plan, a, np, st);
    case 12: return launch_block_k<L, 12, LAYOUT>(plan, a, np, st);
    case 16: return launch_block_k<L, 16, LAYOUT>(plan, a, np, st);
    case 20: return launch_block_k<L, 20, LAYOUT>(plan, a, np, st);
    case 24: return launch_block_k<L, 24, LAYOUT>(plan, a, np, st);
    case 32: return launch_block_k<L, 32, LAYOUT>(plan, a, np, st);
  }
  return -4;
}

// Runs the fused path for n_points points resident on the current device.
template <int L>
int run_block(const HostBlockPlan& plan, BlockTables& bt, int n_eq, int n_var, int64_t n_points, const double* x,
              const double* T, double* f, double* jac, cudaStream_t st) {
  BlockArgs a;
  a.fac = bt.fac;
  a.coef = bt.coeff;
  a.coef2 = T ? bt.coeff2 : nullptr;
  a.T = T;
  a.blk = bt.blk;
  a.X = x;
  a.PTg = nullptr;
  a.F = f;
  a.J = jac;
  a.n_points = n_points;
  a.n_eq = n_eq;
  a.n_var = n_var;
  a.E = plan.E;
  a.R = plan.R;
  a.mode = plan.mode;
  // mode A: results do not depend on how polynomials are grouped into CTAs (each warp
  // owns whole polynomials), so the grouping is chosen per call: one polynomial per warp
  // for few points (latency), up to 32 per CTA for batches (amortises the power table).
  const int nw = plan.nw;
#ifndef PHC_PPC_MULT
#define PHC_PPC_MULT 8
#endif
  a.polys_per_cta =
      plan.mode == 0 ? (n_points >= 4 * 148 ? std::min(n_eq, PHC_PPC_MULT * nw) : std::min(n_eq, nw)) : 1;
  if (plan.layout == 2) {
    if constexpr (L == 2) return launch_block_pts<L, 2>(plan, a, n_points, st);
    return -4;
  }
  if (plan.layout == 1) return launch_block_pts<L, 1>(plan, a, n_points, st);
  // global power table, in chunks of points that fit a 512 MiB scratch
  const int64_t per_point = (int64_t)(n_var + 1) * 2 * plan.E * 2 * L;
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(n_points, ((int64_t)64 << 20) / per_point));
  if (bt.pt_cap < chunk) {
    if (bt.PT) cudaFree(bt.PT);
    bt.PT = nullptr;
    bt.pt_cap = 0;
    if (cudaMalloc(&bt.PT, (size_t)(chunk * per_point * 8)) != cudaSuccess) return -2;
    bt.pt_cap = chunk;
  }
  for (int64_t p0 = 0; p0 < n_points; p0 += chunk) {
    const int64_t np = std::min(chunk, n_points - p0);
    const int64_t nth = np * (n_var + 1) * plan.E;
    block_power_table_kernel<L><<<(unsigned)((nth + 127) / 128), 128, 0, st>>>(x + p0 * n_var * 2 * L, n_var,
                                                                               plan.E, np, bt.PT);
    BlockArgs b = a;
    b.X = x + p0 * n_var * 2 * L;
    b.F = f + p0 * n_eq * 2 * L;
    b.J = jac + p0 * (int64_t)n_eq * n_var * 2 * L;
    b.PTg = bt.PT;
    if (T) b.T = T + p0 * L;
    b.n_points = np;
    int rc = launch_block_pts<L, 0>(plan, b, np, st);
    if (rc) return rc;
  }
  return 0;
}

}  // namespace phc
