// Device double-double (DD) and quad-double (QD) complex arithmetic core.
//
// The paper computes in complex double-double and complex quad-double arithmetic
// from QD-2.3.9 ("complex quad double"
// P:606).  This file restates the published error-free-transformation
// algorithms (Dekker / Knuth two_sum, FMA two_prod; the Hida-Li-Bailey DD and QD
// algorithms) for sm_100a.  Every floating-point step uses the __dadd_rn /
// __dmul_rn / __fma_rn intrinsics so that nvcc can neither contract nor reassociate
// an error-free transformation.
//
// Variants (reading C8): additions are the "sloppy" (normwise-accurate)
// forms, multiplications the standard FMA forms; the complex DD product is fused
// (one renormalisation per real part).  All are branch-free, so negation commutes
// with every operation (conjugation metamorphic test, P9) and warps never diverge.
#pragma once
#include <cstdint>

namespace phc {

#define PHC_DEV __device__ __forceinline__

// Device-side bounds checks of a debug build (-DPHC_CHECKS=1, __graft_entry__.build_checked):
// compute-sanitizer is not available on this pool, so indices into the power tables, the
// row accumulators and the term tables trap when out of range.  No-ops otherwise.
#if PHC_CHECKS
#define PHC_CHECK(cond) \
  do {                  \
    if (!(cond)) __trap(); \
  } while (0)
#else
#define PHC_CHECK(cond) \
  do {                  \
  } while (0)
#endif

// QD dot product summation shape (1 = balanced trees, 0 = the sequential chains)
#ifndef PHC_QD_TREE
#define PHC_QD_TREE 1
#endif

PHC_DEV double add_(double a, double b) { return __dadd_rn(a, b); }
PHC_DEV double sub_(double a, double b) { return __dadd_rn(a, -b); }
PHC_DEV double mul_(double a, double b) { return __dmul_rn(a, b); }
PHC_DEV double fma_(double a, double b, double c) { return __fma_rn(a, b, c); }

// s + e == a + b exactly (6 DADD).  (Ordering the operands by magnitude for a 3-DADD fast
// two-sum -- DSETP on |a|, |b| plus selects -- measured slower: batch DD -4%, large QD -5 to
// -10%; profiles/README.md.)
PHC_DEV void two_sum(double a, double b, double& s, double& e) {
  s = add_(a, b);
  double bb = sub_(s, a);
  e = add_(sub_(a, sub_(s, bb)), sub_(b, bb));
}
// s + e == a + b exactly when |a| >= |b| (3 DADD).
PHC_DEV void quick_two_sum(double a, double b, double& s, double& e) {
  s = add_(a, b);
  e = sub_(b, sub_(s, a));
}
// p + e == a * b exactly (DMUL + DFMA).
PHC_DEV void two_prod(double a, double b, double& p, double& e) {
  p = mul_(a, b);
  e = fma_(a, b, -p);
}

// ---------------------------------------------------------------------------
// double-double
// ---------------------------------------------------------------------------
struct dd {
  double x[2];
};

PHC_DEV dd dd_make(double h, double l) { dd r; r.x[0] = h; r.x[1] = l; return r; }
PHC_DEV dd dd_neg(const dd& a) { return dd_make(-a.x[0], -a.x[1]); }

// sloppy add: error <= ~2u^2 (|a| + |b|)  (normwise accurate)
PHC_DEV dd dd_add(const dd& a, const dd& b) {
  double s, e;
  two_sum(a.x[0], b.x[0], s, e);
  e = add_(e, add_(a.x[1], b.x[1]));
  dd r;
  quick_two_sum(s, e, r.x[0], r.x[1]);
  return r;
}
PHC_DEV dd dd_mul(const dd& a, const dd& b) {
  double p, e;
  two_prod(a.x[0], b.x[0], p, e);
  e = fma_(a.x[0], b.x[1], e);
  e = fma_(a.x[1], b.x[0], e);
  dd r;
  quick_two_sum(p, e, r.x[0], r.x[1]);
  return r;
}

// ---------------------------------------------------------------------------
// quad-double (Hida, Li, Bailey: sloppy add, sloppy mul, branch-free renormalisation)
// ---------------------------------------------------------------------------
struct qd {
  double x[4];
};

PHC_DEV qd qd_neg(const qd& a) { qd r; for (int i = 0; i < 4; ++i) r.x[i] = -a.x[i]; return r; }

// (a, b, c) <- three_sum(a, b, c): a + b + c exactly, a the leading term
PHC_DEV void three_sum(double& a, double& b, double& c) {
  double t1, t2, t3;
  two_sum(a, b, t1, t2);
  two_sum(c, t1, a, t3);
  two_sum(t2, t3, b, c);
}
// (a, b) <- leading two of a + b + c
PHC_DEV void three_sum2(double& a, double& b, double c) {
  double t1, t2, t3;
  two_sum(a, b, t1, t2);
  two_sum(c, t1, a, t3);
  b = add_(t2, t3);
}
// branch-free renormalisation of a 5-term expansion into 4 limbs
PHC_DEV qd renorm5(double c0, double c1, double c2, double c3, double c4) {
  double s, t0, t1, t2, t3;
  quick_two_sum(c3, c4, s, t3);
  quick_two_sum(c2, s, s, t2);
  quick_two_sum(c1, s, s, t1);
  qd r;
  quick_two_sum(c0, s, r.x[0], t0);
  quick_two_sum(t2, t3, s, t2);
  quick_two_sum(t1, s, s, t1);
  quick_two_sum(t0, s, r.x[1], t0);
  quick_two_sum(t1, t2, s, t1);
  quick_two_sum(t0, s, r.x[2], t0);
  r.x[3] = add_(t0, t1);
  return r;
}

PHC_DEV qd qd_add(const qd& a, const qd& b) {
  double s0, s1, s2, s3, t0, t1, t2, t3;
  two_sum(a.x[0], b.x[0], s0, t0);
  two_sum(a.x[1], b.x[1], s1, t1);
  two_sum(a.x[2], b.x[2], s2, t2);
  two_sum(a.x[3], b.x[3], s3, t3);
  two_sum(s1, t0, s1, t0);
  three_sum(s2, t0, t1);
  three_sum2(s3, t0, t2);
  t0 = add_(add_(t0, t1), t3);
  return renorm5(s0, s1, s2, s3, t0);
}

PHC_DEV qd qd_mul(const qd& a, const qd& b) {
  double p0, p1, p2, p3, p4, p5, q0, q1, q2, q3, q4, q5;
  two_prod(a.x[0], b.x[0], p0, q0);
  two_prod(a.x[0], b.x[1], p1, q1);
  two_prod(a.x[1], b.x[0], p2, q2);
  two_prod(a.x[0], b.x[2], p3, q3);
  two_prod(a.x[1], b.x[1], p4, q4);
  two_prod(a.x[2], b.x[0], p5, q5);
  // O(eps) terms
  three_sum(p1, p2, q0);
  // O(eps^2) terms: (p2, q1, q2) + (p3, p4, p5)
  three_sum(p2, q1, q2);
  three_sum(p3, p4, p5);
  double s0, s1, s2, t0, t1;
  two_sum(p2, p3, s0, t0);
  two_sum(q1, p4, s1, t1);
  s2 = add_(q2, p5);
  two_sum(s1, t0, s1, t0);
  s2 = add_(s2, add_(t0, t1));
  // O(eps^3) terms
  double o3 = mul_(a.x[0], b.x[3]);
  o3 = fma_(a.x[1], b.x[2], o3);
  o3 = fma_(a.x[2], b.x[1], o3);
  o3 = fma_(a.x[3], b.x[0], o3);
  o3 = add_(o3, add_(add_(q0, q3), add_(q4, q5)));
  s1 = add_(s1, o3);
  return renorm5(p0, p1, s0, s1, s2);
}

// Robust renormalisation of a 4-term sum of any magnitudes: an exact bottom-up two_sum
// sweep followed by a top-down two_sum sweep gives non-overlapping limbs in decreasing
// order even after cancellation (the quick_two_sum chain of renorm5 assumes ordered input).
PHC_DEV qd renorm4_robust(double a0, double a1, double a2, double a3) {
  double s, c0, c1, c2, c3;
  two_sum(a2, a3, s, c3);
  two_sum(a1, s, s, c2);
  two_sum(a0, s, c0, c1);
  qd r;
  double e;
  // two_sum(c0, c1) would return (c0, c1) unchanged: c1 is the rounding error of c0 = fl(.),
  // so |c1| <= ulp(c0)/2 and, on a tie, c0 is already even -- skipped (6 DADD per product)
  r.x[0] = c0;
  e = c1;
  two_sum(e, c2, r.x[1], e);
  two_sum(e, c3, r.x[2], r.x[3]);
  return r;
}

// QD dot product x*y + z*w (the real parts of a complex product), in the spirit of the
// Hida-Li-Bailey multiplication: all limb products of order <= 2 as exact two_prods, the
// order-3 products by FMA; level l collects the order-l terms with exact two_sum chains
// whose errors move to level l+1; level 3 is a plain sum.  Normwise error ~2^-208
// relative to |x||y| + |z||w| (checked in exact emulation).
// The levels' sums (a0, a1, a2, o) whose exact sum is x*y + z*w to ~2^-208 normwise, not yet
// renormalised: the "lazy" QD product (PHC_QD_LAZY) feeds them straight into the next product,
// whose limb levels only need |level l| <~ u^l N (N = |x0 y0| + |z0 w0|), which they satisfy by
// construction even after cancellation in a0; renorm4_robust makes them non-overlapping.
PHC_DEV qd qd_dot2_parts(const qd& x, const qd& y, const qd& z, const qd& w) {
  double p0, q0, r0, t0;
  two_prod(x.x[0], y.x[0], p0, q0);
  two_prod(z.x[0], w.x[0], r0, t0);
  double p1, q1, p2, q2, r1, t1, r2, t2;
  two_prod(x.x[0], y.x[1], p1, q1);
  two_prod(x.x[1], y.x[0], p2, q2);
  two_prod(z.x[0], w.x[1], r1, t1);
  two_prod(z.x[1], w.x[0], r2, t2);
  double p3, q3, p4, q4, p5, q5, r3, t3, r4, t4, r5, t5;
  two_prod(x.x[0], y.x[2], p3, q3);
  two_prod(x.x[1], y.x[1], p4, q4);
  two_prod(x.x[2], y.x[0], p5, q5);
  two_prod(z.x[0], w.x[2], r3, t3);
  two_prod(z.x[1], w.x[1], r4, t4);
  two_prod(z.x[2], w.x[0], r5, t5);
  // level 3 (plain): order-3 products and the errors of the order-2 products
  double o = mul_(x.x[0], y.x[3]);
  o = fma_(x.x[1], y.x[2], o);
  o = fma_(x.x[2], y.x[1], o);
  o = fma_(x.x[3], y.x[0], o);
  o = fma_(z.x[0], w.x[3], o);
  o = fma_(z.x[1], w.x[2], o);
  o = fma_(z.x[2], w.x[1], o);
  o = fma_(z.x[3], w.x[0], o);
  o = add_(o, add_(add_(add_(q3, q4), add_(q5, t3)), add_(t4, t5)));
  // level 0
  double a0, e;
  two_sum(p0, r0, a0, e);
#if PHC_QD_TREE
  // Same exact transformations as below, summed as balanced trees instead of chains: the
  // dependent-DADD depth per product falls from ~29 two_sums to ~14 (the profile's top
  // stall was the fixed-latency dependency wait).
  // level 1 (7 terms): e, q0, t0, p1, p2, r1, r2 -> a1, errors f1..f6 (order 2)
  double a1, f1, f2, f3, f4, f5, f6;
  {
    double u1, u2, u3, u4, u5;
    two_sum(e, q0, u1, f1);
    two_sum(t0, p1, u2, f2);
    two_sum(p2, r1, u3, f3);
    two_sum(u1, u2, u4, f4);
    two_sum(u3, r2, u5, f5);
    two_sum(u4, u5, a1, f6);
  }
  // level 2 (16 terms) -> a2; the 15 errors (order 3) are summed plainly into o
  double a2;
  {
    double v0, v1, v2, v3, v4, v5, v6, v7, g0, g1, g2, g3, g4, g5, g6, g7;
    two_sum(f1, f2, v0, g0);
    two_sum(f3, f4, v1, g1);
    two_sum(f5, f6, v2, g2);
    two_sum(q1, q2, v3, g3);
    two_sum(t1, t2, v4, g4);
    two_sum(p3, p4, v5, g5);
    two_sum(p5, r3, v6, g6);
    two_sum(r4, r5, v7, g7);
    double w0, w1, w2, w3, h0, h1, h2, h3;
    two_sum(v0, v1, w0, h0);
    two_sum(v2, v3, w1, h1);
    two_sum(v4, v5, w2, h2);
    two_sum(v6, v7, w3, h3);
    double z0, z1, k0, k1, k2;
    two_sum(w0, w1, z0, k0);
    two_sum(w2, w3, z1, k1);
    two_sum(z0, z1, a2, k2);
    const double gs = add_(add_(add_(g0, g1), add_(g2, g3)), add_(add_(g4, g5), add_(g6, g7)));
    const double hs = add_(add_(h0, h1), add_(h2, h3));
    o = add_(o, add_(add_(gs, hs), add_(add_(k0, k1), k2)));
  }
  qd r;
  r.x[0] = a0;
  r.x[1] = a1;
  r.x[2] = a2;
  r.x[3] = o;
  return r;
#else
  // level 1: e, q0, t0, p1, p2, r1, r2 -> a1, errors f1..f6 (order 2)
  double a1 = e, f1, f2, f3, f4, f5, f6;
  two_sum(a1, q0, a1, f1);
  two_sum(a1, t0, a1, f2);
  two_sum(a1, p1, a1, f3);
  two_sum(a1, p2, a1, f4);
  two_sum(a1, r1, a1, f5);
  two_sum(a1, r2, a1, f6);
  // level 2: f1..f6, q1, q2, t1, t2, p3, p4, p5, r3, r4, r5 -> a2, errors (order 3) into o
  double a2 = f1, g;
  two_sum(a2, f2, a2, g); o = add_(o, g);
  two_sum(a2, f3, a2, g); o = add_(o, g);
  two_sum(a2, f4, a2, g); o = add_(o, g);
  two_sum(a2, f5, a2, g); o = add_(o, g);
  two_sum(a2, f6, a2, g); o = add_(o, g);
  two_sum(a2, q1, a2, g); o = add_(o, g);
  two_sum(a2, q2, a2, g); o = add_(o, g);
  two_sum(a2, t1, a2, g); o = add_(o, g);
  two_sum(a2, t2, a2, g); o = add_(o, g);
  two_sum(a2, p3, a2, g); o = add_(o, g);
  two_sum(a2, p4, a2, g); o = add_(o, g);
  two_sum(a2, p5, a2, g); o = add_(o, g);
  two_sum(a2, r3, a2, g); o = add_(o, g);
  two_sum(a2, r4, a2, g); o = add_(o, g);
  two_sum(a2, r5, a2, g); o = add_(o, g);
  qd r;
  r.x[0] = a0;
  r.x[1] = a1;
  r.x[2] = a2;
  r.x[3] = o;
  return r;
#endif
}

// Level-wise sum of two lazy QD values (limb l bounded by c_l u^l N, as qd_dot2_parts leaves
// them): each level is summed exactly with two_sum, its errors moved to the next level, level 3
// plainly -- 41 DADD against 30 + 91 for renormalising the lazy operand and a qd_add.  The
// result is again lazy (bounds c_l grow with the number of operands summed); renorm4_robust
// when it is stored.
PHC_DEV qd qd_add_levels(const qd& a, const qd& b) {
  double s0, e0, t, f1, f2, s1, h1, h2, h3, s2;
  two_sum(a.x[0], b.x[0], s0, e0);
  two_sum(a.x[1], b.x[1], t, f1);
  two_sum(t, e0, s1, f2);
  two_sum(a.x[2], b.x[2], t, h1);
  two_sum(t, f1, t, h2);
  two_sum(t, f2, s2, h3);
  qd r;
  r.x[0] = s0;
  r.x[1] = s1;
  r.x[2] = s2;
  r.x[3] = add_(add_(a.x[3], b.x[3]), add_(add_(h1, h2), h3));
  return r;
}

PHC_DEV qd qd_dot2(const qd& x, const qd& y, const qd& z, const qd& w) {
  const qd t = qd_dot2_parts(x, y, z, w);
  return renorm4_robust(t.x[0], t.x[1], t.x[2], t.x[3]);
}

// ---------------------------------------------------------------------------
// division (NEXT-1 Newton step only: pivots and back substitution).  Long division
// q_j = r_j / b_0 with exact-ish remainders (the QD-library scheme, restated).
// ---------------------------------------------------------------------------
PHC_DEV dd dd_sub(const dd& a, const dd& b) { return dd_add(a, dd_neg(b)); }
PHC_DEV dd dd_mul_d(const dd& a, double b) {
  double p, e;
  two_prod(a.x[0], b, p, e);
  e = fma_(a.x[1], b, e);
  dd r;
  quick_two_sum(p, e, r.x[0], r.x[1]);
  return r;
}
PHC_DEV dd dd_div(const dd& a, const dd& b) {
  const double q1 = __ddiv_rn(a.x[0], b.x[0]);
  dd r = dd_sub(a, dd_mul_d(b, q1));
  const double q2 = __ddiv_rn(r.x[0], b.x[0]);
  r = dd_sub(r, dd_mul_d(b, q2));
  const double q3 = __ddiv_rn(r.x[0], b.x[0]);
  dd q;
  quick_two_sum(q1, q2, q.x[0], q.x[1]);
  return dd_add(q, dd_make(q3, 0.0));
}
PHC_DEV qd qd_from_d(double a) { qd r; r.x[0] = a; r.x[1] = r.x[2] = r.x[3] = 0.0; return r; }
PHC_DEV qd qd_sub(const qd& a, const qd& b) { return qd_add(a, qd_neg(b)); }
// QD x double: a_j s = p_j + e_j exactly (FMA two_prod), collected by order of magnitude
// (the QD library's mul_qd_d); ~4x cheaper than qd_mul with a promoted double.
PHC_DEV qd qd_mul_d(const qd& a, double s) {
  double p0, p1, p2, p3, e0, e1, e2;
  two_prod(a.x[0], s, p0, e0);
  two_prod(a.x[1], s, p1, e1);
  two_prod(a.x[2], s, p2, e2);
  p3 = mul_(a.x[3], s);
  double s1, t1;
  two_sum(p1, e0, s1, t1);  // O(eps)
  three_sum(p2, e1, t1);    // O(eps^2) -> p2, (e1, t1) O(eps^3)
  const double s3 = add_(add_(p3, e2), add_(e1, t1));
  return renorm5(p0, s1, p2, s3, 0.0);
}
// The same long divisions with each quotient digit formed as r_0 * (1 / b_0) -- one
// correctly rounded reciprocal (__drcp_rn) and a DMUL per digit instead of a DDIV per digit.
// A digit may be off by an ulp more; the remainders stay exact as before, so the next digit
// absorbs it and the last digit's error is ~2^-52 of a remainder already ~2^-104 (DD) /
// ~2^-208 (QD) of the quotient.
PHC_DEV dd dd_div_rc(const dd& a, const dd& b) {
  const double rc = __drcp_rn(b.x[0]);
  const double q1 = mul_(a.x[0], rc);
  dd r = dd_sub(a, dd_mul_d(b, q1));
  const double q2 = mul_(r.x[0], rc);
  r = dd_sub(r, dd_mul_d(b, q2));
  const double q3 = mul_(r.x[0], rc);
  dd q;
  quick_two_sum(q1, q2, q.x[0], q.x[1]);
  return dd_add(q, dd_make(q3, 0.0));
}
#ifndef PHC_QD_DIV_TAPER2
#define PHC_QD_DIV_TAPER2 1
#endif
// QD: the first two remainders are full QD updates; the later ones are ~2^-104 and ~2^-156 of
// |a| and only need ~2^-108 and ~2^-56 of their own size to keep the quotient at ~2^-212, so
// they are formed in two and one levels (two_prod / two_sum where an error could reach
// 2^-212 |a|, plain FMA below): dependent latency 2,050 -> 1,358 cycles, same maximum error
// over the arithmetic test's samples (profiles/op_latency_r02s3_taper.txt).
PHC_DEV qd qd_div_rc(const qd& a, const qd& b) {
  const double rc = __drcp_rn(b.x[0]);
  const double q0 = mul_(a.x[0], rc);
  qd r = qd_sub(a, qd_mul_d(b, q0));  // |r| ~ 2^-52 |a|
  const double q1 = mul_(r.x[0], rc);
#if PHC_QD_DIV_TAPER2
  {
    // r - q1 b (~2^-104 |a|, needed to ~2^-212 |a|): r0 - b0 q1 exact (Sterbenz), order-1 and
    // order-2 terms summed exactly, order-3 terms in one FMA-rounded double; then made
    // (nearly) normalised for the next digit's Sterbenz step
    double p0, e0, p1, e1, p2, e2;
    two_prod(b.x[0], q1, p0, e0);
    two_prod(b.x[1], q1, p1, e1);
    two_prod(b.x[2], q1, p2, e2);
    double u0, f1, f2, f3, u1, g1, g2, g3, g4, g5;
    two_sum(sub_(r.x[0], p0), r.x[1], u0, f1);
    two_sum(u0, -e0, u0, f2);
    two_sum(u0, -p1, u0, f3);
    two_sum(r.x[2], -e1, u1, g1);
    two_sum(u1, -p2, u1, g2);
    two_sum(u1, f1, u1, g3);
    two_sum(u1, f2, u1, g4);
    two_sum(u1, f3, u1, g5);
    const double u2 = add_(fma_(-q1, b.x[3], sub_(r.x[3], e2)), add_(add_(g1, g2), add_(add_(g3, g4), g5)));
    double v0, v1, v2, v3;
    two_sum(u0, u1, v0, v1);
    two_sum(v1, u2, v1, v2);
    two_sum(v0, v1, r.x[0], v3);
    two_sum(v3, v2, r.x[1], r.x[2]);
    r.x[3] = 0.0;
  }
#else
  r = qd_sub(r, qd_mul_d(b, q1));  // |r| ~ 2^-104 |a|, normalised
#endif
  const double q2 = mul_(r.x[0], rc);
  // t = r - q2 b (|t| ~ 2^-156 |a|): r0 - b0 q2 exact (Sterbenz: b0 q2 is within a few ulps of
  // r0), the order-1 terms summed exactly, the order-2 terms in one double
  double p0, e0, p1, e1;
  two_prod(b.x[0], q2, p0, e0);
  two_prod(b.x[1], q2, p1, e1);
  double t0, f1, f2, f3;
  two_sum(sub_(r.x[0], p0), r.x[1], t0, f1);
  two_sum(t0, -e0, t0, f2);
  two_sum(t0, -p1, t0, f3);
  const double t1 = add_(fma_(-q2, b.x[2], sub_(r.x[2], e1)), add_(add_(f1, f2), f3));
  const double q3 = mul_(add_(t0, t1), rc);
  // t - q3 b (~2^-208 |a|) in one double
  const double r4 = add_(fma_(-q3, b.x[0], t0), fma_(-q3, b.x[1], t1));
  const double q4 = mul_(r4, rc);
  return renorm5(q0, q1, q2, q3, q4);
}
PHC_DEV qd qd_div(const qd& a, const qd& b) {
  double q[5];
  qd r = a;
  for (int j = 0; j < 5; ++j) {
    q[j] = __ddiv_rn(r.x[0], b.x[0]);
    if (j < 4) r = qd_sub(r, qd_mul_d(b, q[j]));
  }
  return renorm5(q[0], q[1], q[2], q[3], q[4]);
}

// ---------------------------------------------------------------------------
// complex values, templated on the real type; Prec<L> traits below
// ---------------------------------------------------------------------------
template <class R>
struct cplx {
  R re, im;
};

using cdd = cplx<dd>;
using cqd = cplx<qd>;

template <int L> struct Prec;

// DD dot product x*y + z*w (one real part of a complex DD product), unnormalised:
// s + t with s = fl(x0 y0 + z0 w0) and t its error plus the cross terms.
// PHC_DD_DOT_TREE = 1 accumulates the cross terms in two chains started from the product
// errors (independent of the two_sum of the leading products), so the dependent depth
// falls from 11 to 7 operations at the same instruction count; 0 is the single chain.
#ifndef PHC_DD_DOT_TREE
#define PHC_DD_DOT_TREE 1
#endif
PHC_DEV void dd_dot2(double x0, double x1, double y0, double y1, double z0, double z1, double w0, double w1,
                     double& s, double& t) {
  double p1, e1, p2, e2;
  two_prod(x0, y0, p1, e1);
  two_prod(z0, w0, p2, e2);
  two_sum(p1, p2, s, t);
#if PHC_DD_DOT_TREE
  double c1 = fma_(x0, y1, e1);
  c1 = fma_(x1, y0, c1);
  double c2 = fma_(z0, w1, e2);
  c2 = fma_(z1, w0, c2);
  t = add_(t, add_(c1, c2));
#else
  t = add_(t, add_(e1, e2));
  t = fma_(x0, y1, t);
  t = fma_(x1, y0, t);
  t = fma_(z0, w1, t);
  t = fma_(z1, w0, t);
#endif
}

template <> struct Prec<2> {
  using real = dd;
  using C = cdd;
  static constexpr int L = 2;
  PHC_DEV static C zero() { C z; z.re = dd_make(0, 0); z.im = dd_make(0, 0); return z; }
  PHC_DEV static C one() { C z; z.re = dd_make(1, 0); z.im = dd_make(0, 0); return z; }
  PHC_DEV static C add(const C& a, const C& b) { C r; r.re = dd_add(a.re, b.re); r.im = dd_add(a.im, b.im); return r; }
  // real helpers (homotopy parameter t, NEXT-3)
  PHC_DEV static real rload(const double* p) { return dd_make(p[0], p[1]); }
  PHC_DEV static real one_minus(const real& t) { return dd_add(dd_make(1, 0), dd_neg(t)); }
  PHC_DEV static C mul_real(const C& a, const real& s) { C r; r.re = dd_mul(a.re, s); r.im = dd_mul(a.im, s); return r; }
  PHC_DEV static real rfrom(double d) { return dd_make(d, 0.0); }
  PHC_DEV static real radd(const real& a, const real& b) { return dd_add(a, b); }
  PHC_DEV static real rsub(const real& a, const real& b) { return dd_sub(a, b); }
  PHC_DEV static real rmul(const real& a, const real& b) { return dd_mul(a, b); }
  PHC_DEV static real rdiv(const real& a, const real& b) { return dd_div_rc(a, b); }
  PHC_DEV static void rstore(double* p, const real& a) { p[0] = a.x[0]; p[1] = a.x[1]; }
  // fused complex DD product: each real part is a 2-term dot product accumulated
  // in one error term, with one renormalisation (normwise error ~ u^2 |a||b|).
  PHC_DEV static C mul(const C& a, const C& b) {
    C r;
    double s, t;
    dd_dot2(a.re.x[0], a.re.x[1], b.re.x[0], b.re.x[1], -a.im.x[0], -a.im.x[1], b.im.x[0], b.im.x[1], s, t);
    quick_two_sum(s, t, r.re.x[0], r.re.x[1]);
    dd_dot2(a.re.x[0], a.re.x[1], b.im.x[0], b.im.x[1], a.im.x[0], a.im.x[1], b.re.x[0], b.re.x[1], s, t);
    quick_two_sum(s, t, r.im.x[0], r.im.x[1]);
    return r;
  }
  // "lazy" product: the same dot products, without the final renormalisation of each real
  // part, so (hi, lo) may have |lo| a few ulps of hi (or exceed hi after cancellation).
  // Every later product forms hi*hi exactly and the cross terms with FMA, so the
  // normwise error stays O(u^2 |a||b|).
  PHC_DEV static C mul_lazy(const C& a, const C& b) {
    C r;
    dd_dot2(a.re.x[0], a.re.x[1], b.re.x[0], b.re.x[1], -a.im.x[0], -a.im.x[1], b.im.x[0], b.im.x[1], r.re.x[0],
            r.re.x[1]);
    dd_dot2(a.re.x[0], a.re.x[1], b.im.x[0], b.im.x[1], a.im.x[0], a.im.x[1], b.re.x[0], b.re.x[1], r.im.x[0],
            r.im.x[1]);
    return r;
  }
  // lazy sum: exact two_sum of the leading parts, low parts summed without renormalising
  PHC_DEV static C add_lazy(const C& a, const C& b) {
    C r;
    double s, e;
    two_sum(a.re.x[0], b.re.x[0], s, e);
    r.re.x[0] = s;
    r.re.x[1] = add_(add_(a.re.x[1], b.re.x[1]), e);
    two_sum(a.im.x[0], b.im.x[0], s, e);
    r.im.x[0] = s;
    r.im.x[1] = add_(add_(a.im.x[1], b.im.x[1]), e);
    return r;
  }
  // accumulator update with a lazy product (the lazy sum takes unnormalised operands)
  PHC_DEV static C accum(const C& acc, const C& g) { return add_lazy(acc, g); }
  // renormalise a lazy value: (hi, lo) -> two_sum(hi, lo)
  PHC_DEV static C norm(const C& a) {
    C r;
    two_sum(a.re.x[0], a.re.x[1], r.re.x[0], r.re.x[1]);
    two_sum(a.im.x[0], a.im.x[1], r.im.x[0], r.im.x[1]);
    return r;
  }
  // multiply by a small positive integer s (exact in binary64): product exact via two_prod
  PHC_DEV static real mul_int_real(const real& a, double s) {
    double p, e;
    two_prod(a.x[0], s, p, e);
    e = fma_(a.x[1], s, e);
    real r;
    quick_two_sum(p, e, r.x[0], r.x[1]);
    return r;
  }
  PHC_DEV static C mul_int(const C& a, double s) { C r; r.re = mul_int_real(a.re, s); r.im = mul_int_real(a.im, s); return r; }
  PHC_DEV static C neg(const C& a) { C r; r.re = dd_neg(a.re); r.im = dd_neg(a.im); return r; }
  PHC_DEV static C sub(const C& a, const C& b) { return add(a, neg(b)); }
  // 1 / a = conj(a) / |a|^2
  // |a|^2 (the denominator of the reciprocal)
  PHC_DEV static real abs2(const C& a) { return dd_add(dd_mul(a.re, a.re), dd_mul(a.im, a.im)); }
  PHC_DEV static C recip(const C& a) {
    const dd d = abs2(a);
    C r;
    r.re = dd_div_rc(a.re, d);
    r.im = dd_neg(dd_div_rc(a.im, d));
    return r;
  }
  // |a|^2 from the leading limbs (pivot selection only)
  PHC_DEV static double abs2_hi(const C& a) { return a.re.x[0] * a.re.x[0] + a.im.x[0] * a.im.x[0]; }
};

template <> struct Prec<4> {
  using real = qd;
  using C = cqd;
  static constexpr int L = 4;
  PHC_DEV static C zero() { C z; for (int i = 0; i < 4; ++i) { z.re.x[i] = 0; z.im.x[i] = 0; } return z; }
  PHC_DEV static C one() { C z = zero(); z.re.x[0] = 1; return z; }
  PHC_DEV static C add(const C& a, const C& b) { C r; r.re = qd_add(a.re, b.re); r.im = qd_add(a.im, b.im); return r; }
  // real helpers (homotopy parameter t, NEXT-3)
  PHC_DEV static real rload(const double* p) { qd r; for (int i = 0; i < 4; ++i) r.x[i] = p[i]; return r; }
  PHC_DEV static real one_minus(const real& t) { return qd_add(qd_from_d(1.0), qd_neg(t)); }
  PHC_DEV static C mul_real(const C& a, const real& s) { C r; r.re = qd_mul(a.re, s); r.im = qd_mul(a.im, s); return r; }
  PHC_DEV static real rfrom(double d) { return qd_from_d(d); }
  PHC_DEV static real radd(const real& a, const real& b) { return qd_add(a, b); }
  PHC_DEV static real rsub(const real& a, const real& b) { return qd_sub(a, b); }
  PHC_DEV static real rmul(const real& a, const real& b) { return qd_mul(a, b); }
  PHC_DEV static real rdiv(const real& a, const real& b) { return qd_div_rc(a, b); }
  PHC_DEV static void rstore(double* p, const real& a) { for (int i = 0; i < 4; ++i) p[i] = a.x[i]; }
  // fused complex QD product: each real part is a QD dot product x*y + z*w evaluated in
  // one pass (qd_dot2), instead of two qd_mul and a qd_add (~440 vs ~680 FP64 instructions).
  PHC_DEV static C mul(const C& a, const C& b) {
    C r;
    r.re = qd_dot2(a.re, b.re, qd_neg(a.im), b.im);
    r.im = qd_dot2(a.re, b.im, a.im, b.re);
    return r;
  }
#ifndef PHC_QD_LAZY
#define PHC_QD_LAZY 1
#endif
#if PHC_QD_LAZY
  // lazy product: the dot products' level sums without the final renormalisation (qd_dot2_parts);
  // a lazy value may only feed another product, norm() or accum()
  PHC_DEV static C mul_lazy(const C& a, const C& b) {
    C r;
    r.re = qd_dot2_parts(a.re, b.re, qd_neg(a.im), b.im);
    r.im = qd_dot2_parts(a.re, b.im, a.im, b.re);
    return r;
  }
  PHC_DEV static C norm(const C& a) {
    C r;
    r.re = renorm4_robust(a.re.x[0], a.re.x[1], a.re.x[2], a.re.x[3]);
    r.im = renorm4_robust(a.im.x[0], a.im.x[1], a.im.x[2], a.im.x[3]);
    return r;
  }
#else
  PHC_DEV static C mul_lazy(const C& a, const C& b) { return mul(a, b); }
  PHC_DEV static C norm(const C& a) { return a; }
#endif
#ifndef PHC_QD_LAZY_ACC
#define PHC_QD_LAZY_ACC 1
#endif
#if PHC_QD_LAZY && PHC_QD_LAZY_ACC
  // lazy sums (accumulators, warp trees, row totals; every result is renormalised by norm()
  // before it is stored)
  PHC_DEV static C add_lazy(const C& a, const C& b) {
    C r;
    r.re = qd_add_levels(a.re, b.re);
    r.im = qd_add_levels(a.im, b.im);
    return r;
  }
  PHC_DEV static C accum(const C& acc, const C& g) { return add_lazy(acc, g); }
#else
  PHC_DEV static C add_lazy(const C& a, const C& b) { return add(a, b); }
  // accumulator update with a (possibly lazy) product: qd_add needs normalised operands
  PHC_DEV static C accum(const C& acc, const C& g) { return add(acc, norm(g)); }
#endif
  PHC_DEV static real mul_int_real(const real& a, double s) {
    // a_j * s = p_j + e_j exactly; collect by order of magnitude
    double p0, p1, p2, p3, e0, e1, e2;
    two_prod(a.x[0], s, p0, e0);
    two_prod(a.x[1], s, p1, e1);
    two_prod(a.x[2], s, p2, e2);
    p3 = mul_(a.x[3], s);
    double s1, t1;
    two_sum(p1, e0, s1, t1);      // O(eps)
    three_sum(p2, e1, t1);        // O(eps^2) -> p2, (e1, t1) O(eps^3)
    double s3 = add_(add_(p3, e2), add_(e1, t1));
    return renorm5(p0, s1, p2, s3, 0.0);
  }
  PHC_DEV static C mul_int(const C& a, double s) { C r; r.re = mul_int_real(a.re, s); r.im = mul_int_real(a.im, s); return r; }
  PHC_DEV static C neg(const C& a) { C r; r.re = qd_neg(a.re); r.im = qd_neg(a.im); return r; }
  PHC_DEV static C sub(const C& a, const C& b) { return add(a, neg(b)); }
  PHC_DEV static real abs2(const C& a) { return qd_dot2(a.re, a.re, a.im, a.im); }
  PHC_DEV static C recip(const C& a) {
    const qd d = abs2(a);
    C r;
    r.re = qd_div_rc(a.re, d);
    r.im = qd_neg(qd_div_rc(a.im, d));
    return r;
  }
  PHC_DEV static double abs2_hi(const C& a) { return a.re.x[0] * a.re.x[0] + a.im.x[0] * a.im.x[0]; }
};

// ---------------------------------------------------------------------------
// global-memory complex load/store in the [2][L] f64 layout (re limbs, im limbs).
// 256-bit vector accesses (LDG.E.ENL2.256 / STG.E.ENL2.256 on sm_100a).
// ---------------------------------------------------------------------------
PHC_DEV void ld4(const double* p, double& a, double& b, double& c, double& d) {
  asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}
PHC_DEV void ld4_rw(const double* p, double& a, double& b, double& c, double& d) {
  asm volatile("ld.global.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}
PHC_DEV void st4(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}

template <int L> PHC_DEV typename Prec<L>::C cload(const double* p);
template <int L> PHC_DEV void cstore(double* p, const typename Prec<L>::C& v);
template <int L> PHC_DEV typename Prec<L>::C cload_rw(const double* p);

template <> PHC_DEV cdd cload<2>(const double* p) {
  cdd v; ld4(p, v.re.x[0], v.re.x[1], v.im.x[0], v.im.x[1]); return v;
}
template <> PHC_DEV cdd cload_rw<2>(const double* p) {
  cdd v; ld4_rw(p, v.re.x[0], v.re.x[1], v.im.x[0], v.im.x[1]); return v;
}
template <> PHC_DEV void cstore<2>(double* p, const cdd& v) { st4(p, v.re.x[0], v.re.x[1], v.im.x[0], v.im.x[1]); }
template <> PHC_DEV cqd cload<4>(const double* p) {
  cqd v;
  ld4(p, v.re.x[0], v.re.x[1], v.re.x[2], v.re.x[3]);
  ld4(p + 4, v.im.x[0], v.im.x[1], v.im.x[2], v.im.x[3]);
  return v;
}
template <> PHC_DEV cqd cload_rw<4>(const double* p) {
  cqd v;
  ld4_rw(p, v.re.x[0], v.re.x[1], v.re.x[2], v.re.x[3]);
  ld4_rw(p + 4, v.im.x[0], v.im.x[1], v.im.x[2], v.im.x[3]);
  return v;
}
template <> PHC_DEV void cstore<4>(double* p, const cqd& v) {
  st4(p, v.re.x[0], v.re.x[1], v.re.x[2], v.re.x[3]);
  st4(p + 4, v.im.x[0], v.im.x[1], v.im.x[2], v.im.x[3]);
}

// 16-byte-vector complex access through a generic pointer (shared memory, or global memory
// written by the same kernel): LDS.128/STS.128 or LD/ST.128.
template <int L>
PHC_DEV typename Prec<L>::C sload(const double* p) {
  typename Prec<L>::C v;
  const double2* q = reinterpret_cast<const double2*>(p);
  if constexpr (L == 2) {
    double2 a = q[0], b = q[1];
    v.re.x[0] = a.x; v.re.x[1] = a.y; v.im.x[0] = b.x; v.im.x[1] = b.y;
  } else {
    double2 a = q[0], b = q[1], c = q[2], d = q[3];
    v.re.x[0] = a.x; v.re.x[1] = a.y; v.re.x[2] = b.x; v.re.x[3] = b.y;
    v.im.x[0] = c.x; v.im.x[1] = c.y; v.im.x[2] = d.x; v.im.x[3] = d.y;
  }
  return v;
}
template <int L>
PHC_DEV void sstore(double* p, const typename Prec<L>::C& v) {
  double2* q = reinterpret_cast<double2*>(p);
  if constexpr (L == 2) {
    q[0] = make_double2(v.re.x[0], v.re.x[1]);
    q[1] = make_double2(v.im.x[0], v.im.x[1]);
  } else {
    q[0] = make_double2(v.re.x[0], v.re.x[1]);
    q[1] = make_double2(v.re.x[2], v.re.x[3]);
    q[2] = make_double2(v.im.x[0], v.im.x[1]);
    q[3] = make_double2(v.im.x[2], v.im.x[3]);
  }
}

// Shared-memory complex arrays gathered by lanes at random entries (row accumulators and
// power tables of the block kernel's layouts 0/1, the latency path; entry idx, 2L doubles =
// L 16-byte units).  PHC_ROW_SWIZZLE rotates the units of entry idx by (idx >> s), s = log2(8 / L), so
// the lanes of a quarter-warp, which touch distinct entries, spread one LDS.128 over all 8
// bank groups instead of 2 (QD) or 4 (DD).
#ifndef PHC_ROW_SWIZZLE
#define PHC_ROW_SWIZZLE 1
#endif
template <int L>
PHC_DEV typename Prec<L>::C row_ld(const double* rows, size_t idx) {
  typename Prec<L>::C v;
  const double2* b = reinterpret_cast<const double2*>(rows) + idx * L;
  constexpr int sh = (L == 4) ? 1 : 2;
#pragma unroll
  for (int q = 0; q < L; ++q) {
    const int pos = PHC_ROW_SWIZZLE ? ((q + (int)(idx >> sh)) & (L - 1)) : q;
    const double2 d = b[pos];
    if (q < L / 2) {
      v.re.x[2 * q] = d.x;
      v.re.x[2 * q + 1] = d.y;
    } else {
      v.im.x[2 * q - L] = d.x;
      v.im.x[2 * q - L + 1] = d.y;
    }
  }
  return v;
}
template <int L>
PHC_DEV void row_st(double* rows, size_t idx, const typename Prec<L>::C& v) {
  double2* b = reinterpret_cast<double2*>(rows) + idx * L;
  constexpr int sh = (L == 4) ? 1 : 2;
#pragma unroll
  for (int q = 0; q < L; ++q) {
    const int pos = PHC_ROW_SWIZZLE ? ((q + (int)(idx >> sh)) & (L - 1)) : q;
    b[pos] = (q < L / 2) ? make_double2(v.re.x[2 * q], v.re.x[2 * q + 1])
                         : make_double2(v.im.x[2 * q - L], v.im.x[2 * q - L + 1]);
  }
}
}  // namespace phc
