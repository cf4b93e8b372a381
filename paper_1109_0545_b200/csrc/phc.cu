// Host runtime and C ABI (include/phc.h): validate and pack the system, own the
// per-device table replicas and scratch, select and launch the kernels, shard
// batches over devices and gather the results.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "runtime.h"
#include "kernels_generic.cuh"
#include "kernels_block.cuh"
#include "kernels_common.cuh"
#include "kernels_scan.cuh"

namespace phc_rt {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

cudaEvent_t pool_event(phc_system* s) {
  if (!s->pool.empty()) {
    cudaEvent_t e = s->pool.back();
    s->pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

int upload(void* dst, const void* src, size_t bytes) {
  if (bytes == 0) return PHC_OK;
  CUDA_TRY(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice));
  return PHC_OK;
}

// NEXT-3: the target coefficients on one device (term order for the generic path, packed for
// the block path).
int upload_target(const phc_system* s, DeviceState* d) {
  DeviceGuard g(d->dev);
  int rc;
  if (s->common) {
    if (!d->cT2 && (rc = dalloc(&d->cT2, s->cT2.size()))) return rc;
    return upload(d->cT2, s->cT2.data(), s->cT2.size() * 8);
  }
  if (!d->coeff2 && (rc = dalloc(&d->coeff2, s->coeff2.size()))) return rc;
  if ((rc = upload(d->coeff2, s->coeff2.data(), s->coeff2.size() * 8))) return rc;
  if (s->plan.usable) {
    const std::vector<double> packed = phc::pack_block_coeff(s->plan, s->coeff2, s->L);
    if (!d->bt.coeff2 && (rc = dalloc(&d->bt.coeff2, std::max<size_t>(1, packed.size())))) return rc;
    if ((rc = upload(d->bt.coeff2, packed.data(), packed.size() * 8))) return rc;
  }
  return PHC_OK;
}

int get_device_state(phc_system* s, int dev, DeviceState** out) {
  std::lock_guard<std::mutex> lk(s->mu);
  auto it = s->devs.find(dev);
  if (it != s->devs.end()) {
    *out = it->second.get();
    return PHC_OK;
  }
  DeviceGuard g(dev);
  std::unique_ptr<DeviceState> d(new DeviceState());
  d->dev = dev;
  CUDA_TRY(cudaStreamCreateWithFlags(&d->stream, cudaStreamNonBlocking));
  CUDA_TRY(cudaStreamCreateWithFlags(&d->stream2, cudaStreamNonBlocking));
  CUDA_TRY(cudaEventCreateWithFlags(&d->done, cudaEventDisableTiming));
  int rc;
  if ((rc = dalloc(&d->term_ptr, s->term_ptr.size()))) return rc;
  if ((rc = dalloc(&d->fac, s->fac.size()))) return rc;
  if ((rc = dalloc(&d->coeff, s->coeff.size()))) return rc;
  if ((rc = dalloc(&d->poly_ptr, s->poly_ptr.size()))) return rc;
  if ((rc = dalloc(&d->jptr, s->jptr.size()))) return rc;
  if ((rc = dalloc(&d->jidx, s->jidx.size()))) return rc;
  if ((rc = upload(d->term_ptr, s->term_ptr.data(), s->term_ptr.size() * 8))) return rc;
  if ((rc = upload(d->fac, s->fac.data(), s->fac.size() * 4))) return rc;
  if ((rc = upload(d->coeff, s->coeff.data(), s->coeff.size() * 8))) return rc;
  if ((rc = upload(d->poly_ptr, s->poly_ptr.data(), s->poly_ptr.size() * 8))) return rc;
  if ((rc = upload(d->jptr, s->jptr.data(), s->jptr.size() * 8))) return rc;
  if ((rc = upload(d->jidx, s->jidx.data(), s->jidx.size() * 8))) return rc;
  if (s->plan.usable) {
    if ((rc = phc::upload_block_tables(s->plan, &d->bt))) return fail(rc, "block table upload failed");
    d->have_block = true;
  }
  if (s->has_target && (rc = upload_target(s, d.get()))) return rc;
  if (s->common) {
    if ((rc = dalloc(&d->cl_ptr, s->cl_ptr.size()))) return rc;
    if ((rc = dalloc(&d->cl_j, s->cl_j.size()))) return rc;
    if ((rc = dalloc(&d->cl_q, s->cl_q.size()))) return rc;
    if ((rc = dalloc(&d->cT, s->cT.size()))) return rc;
    if ((rc = upload(d->cl_ptr, s->cl_ptr.data(), s->cl_ptr.size() * 8))) return rc;
    if ((rc = upload(d->cl_j, s->cl_j.data(), s->cl_j.size() * 4))) return rc;
    if ((rc = upload(d->cl_q, s->cl_q.data(), s->cl_q.size() * 8))) return rc;
    if ((rc = upload(d->cT, s->cT.data(), s->cT.size() * 8))) return rc;
  }
  *out = d.get();
  s->devs[dev] = std::move(d);
  return PHC_OK;
}

int ensure_scratch(const phc_system* s, DeviceState* d, int64_t want_points) {
  const int64_t pt_pp = (int64_t)(s->n_var + 1) * 2 * s->E;  // complex entries per point
  const int64_t per_point = (pt_pp + s->n_terms + s->n_factors) * (int64_t)cbytes(s);
  const int64_t budget = (int64_t)1 << 30;  // 1 GiB of scratch per device
  int64_t cap = std::max<int64_t>(1, std::min<int64_t>(want_points, budget / std::max<int64_t>(per_point, 1)));
  cap = std::min<int64_t>(cap, 65535);  // the generic kernels put the point on gridDim.y
  if (cap <= d->chunk_cap) return PHC_OK;
  DeviceGuard g(d->dev);
  cudaDeviceSynchronize();
  if (d->PT) cudaFree(d->PT);
  if (d->Y) cudaFree(d->Y);
  if (d->G) cudaFree(d->G);
  d->PT = d->Y = d->G = nullptr;
  d->chunk_cap = 0;
  int rc;
  const int64_t cd = 2 * s->L;
  if ((rc = dalloc(&d->PT, (size_t)(cap * pt_pp * cd)))) return rc;
  if ((rc = dalloc(&d->Y, (size_t)(cap * s->n_terms * cd)))) return rc;
  if ((rc = dalloc(&d->G, (size_t)(cap * s->n_factors * cd)))) return rc;
  d->chunk_cap = cap;
  return PHC_OK;
}

template <int L, int MAXK>
void launch_term(const phc_system* s, DeviceState* d, int64_t np, const double* T, cudaStream_t st) {
  dim3 grid((unsigned)((s->n_terms + 127) / 128), (unsigned)np);
  ProfScope ps(s, d->dev, 1, st);
  phc::term_kernel<L, MAXK><<<grid, 128, 0, st>>>(d->term_ptr, d->fac, d->coeff, T ? d->coeff2 : nullptr, T, d->PT,
                                                  s->n_var, s->E, s->n_terms, s->n_factors, np, d->Y, d->G);
}

template <int L>
int run_generic(const phc_system* s, DeviceState* d, int64_t n_points, const double* x, const double* T, double* f,
                double* jac, cudaStream_t st) {
  int rc = ensure_scratch(s, d, n_points);
  if (rc) return rc;
  const int64_t cd = 2 * L;
  for (int64_t p0 = 0; p0 < n_points; p0 += d->chunk_cap) {
    const int64_t np = std::min(d->chunk_cap, n_points - p0);
    const int64_t nth = np * (s->n_var + 1);
    {
    ProfScope ps(s, d->dev, 0, st);
    phc::power_table_kernel<L><<<(unsigned)((nth + 127) / 128), 128, 0, st>>>(x + p0 * s->n_var * cd, s->n_var, s->E,
                                                                              np, d->PT);
    }
    const double* Tc = T ? T + p0 * L : nullptr;
    if (s->kmax <= 8)
      launch_term<L, 8>(s, d, np, Tc, st);
    else if (s->kmax <= 16)
      launch_term<L, 16>(s, d, np, Tc, st);
    else if (s->kmax <= 32)
      launch_term<L, 32>(s, d, np, Tc, st);
    else
      launch_term<L, PHC_MAX_K>(s, d, np, Tc, st);
    const int64_t ne = (int64_t)s->n_eq * s->n_var + s->n_eq;
    dim3 grid((unsigned)((ne + 127) / 128), (unsigned)np);
    ProfScope ps(s, d->dev, 2, st);
    phc::reduce_kernel<L><<<grid, 128, 0, st>>>(d->jptr, d->jidx, d->poly_ptr, d->Y, d->G, s->n_eq, s->n_var,
                                                 s->n_terms, s->n_factors, np, f + p0 * s->n_eq * cd,
                                                 jac + p0 * (int64_t)s->n_eq * s->n_var * cd);
    CUDA_TRY(cudaGetLastError());
  }
  return PHC_OK;
}

// Latency path (kernels_scan.cuh) for calls with few points: one warp per term.
int split_scratch(const phc_system* s, DeviceState* d, int64_t n_points, int S, int64_t cd, cudaStream_t st,
                  phc::ScanArgs* a);

template <int L>
int run_scan(const phc_system* s, DeviceState* d, int64_t n_points, const double* x, const double* T, double* f,
             double* jac, cudaStream_t st) {
  const int64_t cd = 2 * L;
  phc::ScanArgs a;
  a.poly_ptr = d->poly_ptr;
  a.term_ptr = d->term_ptr;
  a.fac = d->fac;
  a.coeff = d->coeff;
  a.coeff2 = T ? d->coeff2 : nullptr;
  a.T = T;
  a.X = x;
  a.F = f;
  a.J = jac;
  a.n_eq = s->n_eq;
  a.n_var = s->n_var;
  a.E = s->E;
  a.S = s->scan_S;
  a.n_points = n_points;
  a.part = nullptr;
  a.count = nullptr;
  int rc = split_scratch(s, d, n_points, s->scan_S, cd, st, &a);
  if (rc) return rc;
  ProfScope ps(s, d->dev, 3, st);
  auto kern = phc::poly_scan_kernel<L>;
  if (s->scan_smem > 48 * 1024)
    CUDA_TRY(phc::ensure_smem((const void*)kern, s->scan_smem));
  const int64_t ctas = n_points * s->n_eq * s->scan_S;
  kern<<<(unsigned)ctas, s->scan_W * 32, s->scan_smem, st>>>(a);
  CUDA_TRY(cudaGetLastError());
  return PHC_OK;
}

// partial rows and arrival counters of an S-way split (latency paths)
int split_scratch(const phc_system* s, DeviceState* d, int64_t n_points, int S, int64_t cd, cudaStream_t st,
                  phc::ScanArgs* a) {
  if (S > 1) {
    const int64_t need = n_points * s->n_eq * S * (int64_t)(s->n_var + 1) * cd;
    if (need > d->part_cap) {
      cudaStreamSynchronize(st);
      if (d->part) cudaFree(d->part);
      d->part = nullptr;
      d->part_cap = 0;
      int rc = dalloc(&d->part, (size_t)need);
      if (rc) return rc;
      d->part_cap = need;
    }
    a->part = d->part;
    const int64_t nc = n_points * s->n_eq;
    if (nc > d->count_cap) {
      cudaStreamSynchronize(st);
      if (d->count) cudaFree(d->count);
      d->count = nullptr;
      d->count_cap = 0;
      int rc = dalloc(&d->count, (size_t)nc);
      if (rc) return rc;
      // zeroed on the caller's stream (ordered before the kernel that counts arrivals; the
      // legacy-stream cudaMemset is not ordered against non-blocking streams)
      CUDA_TRY(cudaMemsetAsync(d->count, 0, nc * sizeof(int), st));
      d->count_cap = nc;
    }
    a->count = d->count;
  }
  return PHC_OK;
}

// Segmented latency path (kernels_scan.cuh poly_seg_kernel): the power table of the call's
// points (block_power_table_kernel, global), then the segmented kernel as its programmatic
// dependent launch.
template <int L, int G>
int launch_seg(const phc_system* s, const phc::ScanArgs& a, const double* PT, int64_t n_points, cudaStream_t st) {
  auto kern = phc::poly_seg_kernel<L, G>;
  if (s->seg_smem > 48 * 1024) CUDA_TRY(phc::ensure_smem((const void*)kern, s->seg_smem));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(n_points * s->n_eq * s->seg_S));
  cfg.blockDim = dim3(s->seg_W * 32);
  cfg.dynamicSmemBytes = s->seg_smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, a, PT));
  return PHC_OK;
}

// segment widths G compiled for the segmented path (two factors per lane: k <= 2G);
// phc_system_create picks one
#define PHC_SEG_SHAPES(X) X(4) X(8) X(10) X(12) X(16)

template <int L>
int run_seg(const phc_system* s, DeviceState* d, int64_t n_points, const double* x, const double* T, double* f,
            double* jac, cudaStream_t st) {
  const int64_t cd = 2 * L;
  phc::ScanArgs a;
  a.poly_ptr = d->poly_ptr;
  a.term_ptr = d->term_ptr;
  a.fac = d->fac;
  a.coeff = d->coeff;
  a.coeff2 = T ? d->coeff2 : nullptr;
  a.T = T;
  a.X = x;
  a.F = f;
  a.J = jac;
  a.n_eq = s->n_eq;
  a.n_var = s->n_var;
  a.E = s->E;
  a.S = s->seg_S;
  a.n_points = n_points;
  a.part = nullptr;
  a.count = nullptr;
  int rc = split_scratch(s, d, n_points, s->seg_S, cd, st, &a);
  if (rc) return rc;
  const int64_t per_point = (int64_t)(s->n_var + 1) * 2 * s->E * cd;
  if (n_points * per_point > d->segPT_cap) {
    cudaStreamSynchronize(st);
    if (d->segPT) cudaFree(d->segPT);
    d->segPT = nullptr;
    d->segPT_cap = 0;
    rc = dalloc(&d->segPT, (size_t)(n_points * per_point));
    if (rc) return rc;
    d->segPT_cap = n_points * per_point;
  }
  ProfScope ps(s, d->dev, 3, st);
  const int64_t nth = n_points * (s->n_var + 1) * s->E;
  phc::block_power_table_kernel<L><<<(unsigned)((nth + 127) / 128), 128, 0, st>>>(x, s->n_var, s->E, n_points,
                                                                                 d->segPT);
  CUDA_TRY(cudaGetLastError());
#define PHC_SEG_CASE(G_) \
  if (s->seg_G == G_) return launch_seg<L, G_>(s, a, d->segPT, n_points, st);
  PHC_SEG_SHAPES(PHC_SEG_CASE)
#undef PHC_SEG_CASE
  return fail(PHC_EUNSUPPORTED, "segmented latency path: no kernel for G = %d", s->seg_G);
}

// NEXT-2 two-stage path: power table, monomial stage V (the term kernel with unit
// coefficients), coefficient product Y = C [V | D].
// split: the latency variant of the coefficient product, chosen per CALL from the call's total
// point count (so a sharded call and an unsharded one use the same variant).
inline bool common_split(const phc_system* s, int64_t call_points) {
  const int TI = s->L == 2 ? 8 : 4;
  return call_points * (s->n_var + 1) * ((s->n_eq + TI - 1) / TI) < 148 * 128;
}

template <int L>
int run_common(const phc_system* s, DeviceState* d, int64_t n_points, const double* x, const double* T, double* f,
               double* jac, bool split, cudaStream_t st) {
  int rc = ensure_scratch(s, d, n_points);
  if (rc) return rc;
  const int64_t cd = 2 * L;
  constexpr int TI = L == 2 ? 8 : 4;
  for (int64_t p0 = 0; p0 < n_points; p0 += d->chunk_cap) {
    const int64_t np = std::min(d->chunk_cap, n_points - p0);
    const int64_t nth = np * (s->n_var + 1);
    {
      ProfScope ps(s, d->dev, 0, st);
      phc::power_table_kernel<L><<<(unsigned)((nth + 127) / 128), 128, 0, st>>>(x + p0 * s->n_var * cd, s->n_var,
                                                                                s->E, np, d->PT);
    }
    if (split && s->kmax <= 32) {
      ProfScope ps1(s, d->dev, 1, st);
      const int64_t nwarps = np * s->n_terms;
      phc::monomial_scan_kernel<L><<<(unsigned)((nwarps * 32 + 127) / 128), 128, 0, st>>>(
          d->term_ptr, d->fac, d->PT, s->n_var, s->E, s->n_terms, s->n_factors, np, d->Y, d->G);
    } else {
      // point-fastest monomial stage with transposed outputs (see coef_product_pt_kernel)
      ProfScope ps1(s, d->dev, 1, st);
      const dim3 grid((unsigned)((np + 127) / 128), (unsigned)s->n_terms);
      if (s->kmax <= 8)
        phc::term_kernel<L, 8, true><<<grid, 128, 0, st>>>(d->term_ptr, d->fac, d->coeff, nullptr, nullptr, d->PT,
                                                          s->n_var, s->E, s->n_terms, s->n_factors, np, d->Y, d->G);
      else if (s->kmax <= 16)
        phc::term_kernel<L, 16, true><<<grid, 128, 0, st>>>(d->term_ptr, d->fac, d->coeff, nullptr, nullptr, d->PT,
                                                           s->n_var, s->E, s->n_terms, s->n_factors, np, d->Y, d->G);
      else if (s->kmax <= 32)
        phc::term_kernel<L, 32, true><<<grid, 128, 0, st>>>(d->term_ptr, d->fac, d->coeff, nullptr, nullptr, d->PT,
                                                           s->n_var, s->E, s->n_terms, s->n_factors, np, d->Y, d->G);
      else
        phc::term_kernel<L, PHC_MAX_K, true><<<grid, 128, 0, st>>>(d->term_ptr, d->fac, d->coeff, nullptr, nullptr,
                                                                  d->PT, s->n_var, s->E, s->n_terms, s->n_factors, np,
                                                                  d->Y, d->G);
    }
    const int64_t tiles = (s->n_eq + TI - 1) / TI;
    const int64_t nthr = np * (s->n_var + 1) * tiles;
    ProfScope ps(s, d->dev, 2, st);
    if (split) {
      const int64_t nwarps = np * (s->n_var + 1) * s->n_eq;
      phc::coef_product_split_kernel<L><<<(unsigned)((nwarps * 32 + 255) / 256), 256, 0, st>>>(
          d->cl_ptr, d->cl_j, d->cl_q, d->cT, T ? d->cT2 : nullptr, T ? T + p0 * L : nullptr, d->Y, d->G, s->n_eq,
          s->n_var, s->n_terms, s->n_factors, np, f + p0 * s->n_eq * cd, jac + p0 * (int64_t)s->n_eq * s->n_var * cd);
    } else {
      (void)nthr;
      const dim3 grid((unsigned)((np + 127) / 128), (unsigned)((s->n_var + 1) * tiles));
      phc::coef_product_pt_kernel<L, TI><<<grid, 128, 0, st>>>(
          d->cl_ptr, d->cl_j, d->cl_q, d->cT, T ? d->cT2 : nullptr, T ? T + p0 * L : nullptr, d->Y, d->G, s->n_eq,
          s->n_var, np, f + p0 * s->n_eq * cd, jac + p0 * (int64_t)s->n_eq * s->n_var * cd);
    }
    CUDA_TRY(cudaGetLastError());
  }
  return PHC_OK;
}

// Evaluate n_points points resident on device d, on stream st.  T (t per point, device d)
// selects the homotopy coefficients (NEXT-3); nullptr evaluates the system's own coefficients.
int run_on_device(const phc_system* s, DeviceState* d, int64_t n_points, const double* x, const double* T, double* f,
                  double* jac, cudaStream_t st, int64_t call_points) {
  if (n_points <= 0) return PHC_OK;
  if (s->common) {
    const bool split = common_split(s, call_points < 0 ? n_points : call_points);
    return s->L == 2 ? run_common<2>(s, d, n_points, x, T, f, jac, split, st)
                     : run_common<4>(s, d, n_points, x, T, f, jac, split, st);
  }
  static const bool no_latency = getenv("PHC_DEBUG_NO_LATENCY_PATH") != nullptr;  // A/B hook
  if (s->scan_ok && !no_latency && (call_points < 0 ? n_points : call_points) * s->n_terms <= kScanMaxTerms)
    return s->seg_ok ? run_seg<4>(s, d, n_points, x, T, f, jac, st)
           : s->L == 2 ? run_scan<2>(s, d, n_points, x, T, f, jac, st)
                       : run_scan<4>(s, d, n_points, x, T, f, jac, st);
  if (d->have_block) {
    ProfScope ps(s, d->dev, 3, st);
    int rc = s->L == 2 ? phc::run_block<2>(s->plan, d->bt, s->n_eq, s->n_var, n_points, x, T, f, jac, st)
                       : phc::run_block<4>(s->plan, d->bt, s->n_eq, s->n_var, n_points, x, T, f, jac, st);
    if (rc) return fail(PHC_ECUDA, "block kernel launch failed: %s", cudaGetErrorString(cudaGetLastError()));
    return PHC_OK;
  }
  return s->L == 2 ? run_generic<2>(s, d, n_points, x, T, f, jac, st) : run_generic<4>(s, d, n_points, x, T, f, jac, st);
}

int ensure_stage(const phc_system* s, DeviceState* d, int64_t np) {
  if (np <= d->stage_cap) return PHC_OK;
  DeviceGuard g(d->dev);
  cudaDeviceSynchronize();
  if (d->xs) cudaFree(d->xs);
  if (d->fs) cudaFree(d->fs);
  if (d->js) cudaFree(d->js);
  if (d->ts) cudaFree(d->ts);
  d->xs = d->fs = d->js = d->ts = nullptr;
  d->stage_cap = 0;
  const int64_t cd = 2 * s->L;
  int rc;
  if ((rc = dalloc(&d->ts, (size_t)(np * s->L)))) return rc;
  if ((rc = dalloc(&d->xs, (size_t)(np * s->n_var * cd)))) return rc;
  if ((rc = dalloc(&d->fs, (size_t)(np * s->n_eq * cd)))) return rc;
  if ((rc = dalloc(&d->js, (size_t)(np * (int64_t)s->n_eq * s->n_var * cd)))) return rc;
  d->stage_cap = np;
  return PHC_OK;
}

// Shared body of the batch calls: T = t per point [n_points][L] (homotopy) or nullptr.
int eval_batch_impl(const phc_system* cs, int64_t n_points, const double* x, const double* T, double* f,
                           double* jac, const int32_t* devices, int32_t n_devices, void* stream) {
  g_err.clear();
  phc_system* s = const_cast<phc_system*>(cs);
  if (!s) return fail(PHC_EINVAL, "NULL system");
  if (n_points < 0) return fail(PHC_EINVAL, "n_points < 0");
  if (n_points == 0) return PHC_OK;
  if (!x || !f || !jac) return fail(PHC_EINVAL, "NULL x/f/jac");
  if ((((uintptr_t)x) | ((uintptr_t)f) | ((uintptr_t)jac)) & 31) return fail(PHC_EINVAL, "x/f/jac must be 32-byte aligned");
  cudaStream_t st = (cudaStream_t)stream;
  if (!devices || n_devices <= 0 || (n_devices == 1 && devices[0] == s->home)) {
    // the common case, on the home device (no device-list bookkeeping on the latency path)
    DeviceGuard g(s->home);
    DeviceState* d;
    int rc = get_device_state(s, s->home, &d);
    if (rc) return rc;
    return run_on_device(s, d, n_points, x, T, f, jac, st);
  }
  std::vector<int> devs(devices, devices + n_devices);
  static const int ndev = [] {
    int c = 0;
    cudaGetDeviceCount(&c);
    return c;
  }();
  for (int dv : devs)
    if (dv < 0 || dv >= ndev) return fail(PHC_EINVAL, "device %d out of range", dv);
  DeviceGuard g(s->home);
  const int64_t cd = 2 * s->L;
  const int64_t G = (int64_t)devs.size();
  // sharded: contiguous equal ranges [g P / G, (g+1) P / G)
  cudaEvent_t start;
  CUDA_TRY(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
  CUDA_TRY(cudaEventRecord(start, st));
  std::vector<cudaEvent_t> dones;
  int rc = PHC_OK;
  for (int64_t gi = 0; gi < G && rc == PHC_OK; ++gi) {
    const int64_t p0 = gi * n_points / G, p1 = (gi + 1) * n_points / G;
    const int64_t np = p1 - p0;
    if (np == 0) continue;
    const int dv = devs[gi];
    DeviceState* d;
    if ((rc = get_device_state(s, dv, &d))) break;
    // PHC_DEBUG_REMOTE=staged|fused (test hook): shards on the home device take the remote
    // branches below, so the one-GPU test boxes exercise the scatter / gather bookkeeping
    const char* dbg = getenv("PHC_DEBUG_REMOTE");
    const int debug_remote = !dbg ? 0 : (strcmp(dbg, "fused") == 0 ? 2 : (strcmp(dbg, "staged") == 0 ? 1 : 0));
    if (dv == s->home && !debug_remote) {
      rc = run_on_device(s, d, np, x + p0 * s->n_var * cd, T ? T + p0 * s->L : nullptr, f + p0 * s->n_eq * cd,
                         jac + p0 * (int64_t)s->n_eq * s->n_var * cd, st, n_points);
      continue;
    }
    DeviceGuard gd(dv);
    int can = 0;
    if (dv == s->home)
      can = debug_remote == 2;  // own memory: "peer" pointers are plain device pointers
    else
      cudaDeviceCanAccessPeer(&can, dv, s->home);
    if (can && dv != s->home) {
      cudaError_t pe = cudaDeviceEnablePeerAccess(s->home, 0);
      if (pe == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
      } else if (pe != cudaSuccess) {
        cudaGetLastError();
        can = 0;
      }
    }
    if (can && s->fused_gather) {
      // fused scatter/compute/gather (SURVEY.md §8(e) option 1): with peer access the
      // kernels of device dv read their points and t from the home device and store F and J
      // straight into the caller's home-device buffers over NVLink -- no staging buffers,
      // no copies; the stores of a point's rows overlap the evaluation of the next points.
      if (cudaStreamWaitEvent(d->stream, start, 0) != cudaSuccess) { rc = fail(PHC_ECUDA, "wait event"); break; }
      if ((rc = run_on_device(s, d, np, x + p0 * s->n_var * cd, T ? T + p0 * s->L : nullptr, f + p0 * s->n_eq * cd,
                              jac + p0 * (int64_t)s->n_eq * s->n_var * cd, d->stream, n_points)))
        break;
      cudaEvent_t e;
      cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
      cudaEventRecord(e, d->stream);
      dones.push_back(e);
      continue;
    }
    if ((rc = ensure_stage(s, d, np))) break;
    if (cudaStreamWaitEvent(d->stream, start, 0) != cudaSuccess) { rc = fail(PHC_ECUDA, "wait event"); break; }
    // a device listed more than once reuses its staging buffers: the next shard's scatter and
    // evaluation wait for the previous shard's gathers (recorded on d->done)
    if (cudaStreamWaitEvent(d->stream, d->done, 0) != cudaSuccess) { rc = fail(PHC_ECUDA, "wait event"); break; }
    if (cudaMemcpyPeerAsync(d->xs, dv, x + p0 * s->n_var * cd, s->home, np * s->n_var * cd * 8, d->stream) != cudaSuccess) {
      rc = fail(PHC_ECUDA, "scatter copy failed");
      break;
    }
    if (T && cudaMemcpyPeerAsync(d->ts, dv, T + p0 * s->L, s->home, np * s->L * 8, d->stream) != cudaSuccess) {
      rc = fail(PHC_ECUDA, "scatter copy (t) failed");
      break;
    }
    // the shard in chunks: evaluation of chunk c on d->stream, its gather to the home device
    // over NVLink on d->stream2, so the gather overlaps the evaluation of the next chunks
    // (SURVEY.md §8(e) option 2).  call_points = the call's total: same regime, same bits.
    const int64_t nch = np >= 8192 ? 4 : 1;
    for (int64_t c = 0; c < nch && rc == PHC_OK; ++c) {
      const int64_t q0 = c * np / nch, q1 = (c + 1) * np / nch, nq = q1 - q0;
      if (nq == 0) continue;
      if ((rc = run_on_device(s, d, nq, d->xs + q0 * s->n_var * cd, T ? d->ts + q0 * s->L : nullptr,
                              d->fs + q0 * s->n_eq * cd, d->js + q0 * (int64_t)s->n_eq * s->n_var * cd, d->stream,
                              n_points)))
        break;
      cudaEvent_t ce;
      cudaEventCreateWithFlags(&ce, cudaEventDisableTiming);
      cudaEventRecord(ce, d->stream);
      cudaStreamWaitEvent(d->stream2, ce, 0);
      cudaEventDestroy(ce);
      if (cudaMemcpyPeerAsync(f + (p0 + q0) * s->n_eq * cd, s->home, d->fs + q0 * s->n_eq * cd, dv,
                              nq * s->n_eq * cd * 8, d->stream2) != cudaSuccess ||
          cudaMemcpyPeerAsync(jac + (p0 + q0) * (int64_t)s->n_eq * s->n_var * cd, s->home,
                              d->js + q0 * (int64_t)s->n_eq * s->n_var * cd, dv,
                              nq * (int64_t)s->n_eq * s->n_var * cd * 8, d->stream2) != cudaSuccess) {
        rc = fail(PHC_ECUDA, "gather copy failed");
        break;
      }
    }
    if (rc) break;
    cudaEventRecord(d->done, d->stream2);
    cudaEvent_t e;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    cudaEventRecord(e, d->stream2);
    dones.push_back(e);
  }
  for (cudaEvent_t e : dones) {
    cudaStreamWaitEvent(st, e, 0);
    cudaEventDestroy(e);
  }
  cudaEventDestroy(start);
  return rc;
}

}  // namespace phc_rt

using namespace phc_rt;

extern "C" {

const char* phc_last_error(void) { return g_err.c_str(); }
const char* phc_version(void) { return "phc-b200 0.1 (sm_100a)"; }

int phc_system_create(phc_system** out, int32_t n_eq, int32_t n_var, int32_t limbs, int64_t n_terms,
                      const int64_t* poly_ptr, const int64_t* term_ptr, const int32_t* var_idx,
                      const int32_t* exponent, const double* coeff, int32_t device) {
  g_err.clear();
  if (!out) return fail(PHC_EINVAL, "out is NULL");
  *out = nullptr;
  if (n_eq < 1 || n_var < 1) return fail(PHC_EINVAL, "n_eq and n_var must be >= 1 (got %d, %d)", n_eq, n_var);
  if (limbs != 2 && limbs != 4) return fail(PHC_EUNSUPPORTED, "limbs must be 2 (DD) or 4 (QD), got %d", limbs);
  if (n_var > PHC_MAX_VARS) return fail(PHC_EUNSUPPORTED, "n_var %d exceeds %d", n_var, PHC_MAX_VARS);
  if (n_terms < 0) return fail(PHC_EINVAL, "n_terms < 0");
  if (!poly_ptr || !term_ptr || (n_terms > 0 && !coeff)) return fail(PHC_EINVAL, "NULL array");
  if (poly_ptr[0] != 0 || poly_ptr[n_eq] != n_terms) return fail(PHC_EINVAL, "poly_ptr must start at 0 and end at n_terms");
  for (int i = 0; i < n_eq; ++i)
    if (poly_ptr[i + 1] < poly_ptr[i]) return fail(PHC_EINVAL, "poly_ptr not monotone at %d", i);
  if (term_ptr[0] != 0) return fail(PHC_EINVAL, "term_ptr[0] must be 0");
  for (int64_t t = 0; t < n_terms; ++t)
    if (term_ptr[t + 1] < term_ptr[t]) return fail(PHC_EINVAL, "term_ptr not monotone at %lld", (long long)t);
  const int64_t n_factors = term_ptr[n_terms];
  if (n_factors > 0 && (!var_idx || !exponent)) return fail(PHC_EINVAL, "NULL var_idx/exponent");
  int kmax = 0, emax = 1;
  for (int64_t t = 0; t < n_terms; ++t) {
    const int64_t a = term_ptr[t], b = term_ptr[t + 1];
    if (b - a > PHC_MAX_K) return fail(PHC_EUNSUPPORTED, "term %lld has k = %lld > %d", (long long)t, (long long)(b - a), PHC_MAX_K);
    kmax = std::max<int>(kmax, (int)(b - a));
    for (int64_t q = a; q < b; ++q) {
      if (var_idx[q] < 0 || var_idx[q] >= n_var)
        return fail(PHC_EINVAL, "term %lld: variable index %d out of range [0, %d)", (long long)t, var_idx[q], n_var);
      if (q > a && var_idx[q] <= var_idx[q - 1])
        return fail(PHC_EINVAL, "term %lld: variable indices must be strictly increasing", (long long)t);
      if (exponent[q] < 1) return fail(PHC_EINVAL, "term %lld: exponent %d < 1", (long long)t, exponent[q]);
      if (exponent[q] > PHC_MAX_EXP) return fail(PHC_EUNSUPPORTED, "exponent %d > %d", exponent[q], PHC_MAX_EXP);
      emax = std::max(emax, exponent[q]);
    }
  }
  for (int64_t q = 0; q < n_terms * 2 * limbs; ++q)
    if (!std::isfinite(coeff[q])) return fail(PHC_EINVAL, "coefficient limb %lld is not finite", (long long)q);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(PHC_ECUDA, "no CUDA device available");
  }
  if (device < 0 || device >= ndev) return fail(PHC_EINVAL, "device %d out of range (have %d)", device, ndev);

  std::unique_ptr<phc_system> s(new phc_system());
  s->n_eq = n_eq;
  s->n_var = n_var;
  s->L = limbs;
  s->home = device;
  s->n_terms = n_terms;
  s->n_factors = n_factors;
  s->kmax = kmax;
  s->E = emax;
  s->poly_ptr.assign(poly_ptr, poly_ptr + n_eq + 1);
  s->term_ptr.assign(term_ptr, term_ptr + n_terms + 1);
  s->fac.resize(n_factors);
  for (int64_t q = 0; q < n_factors; ++q) s->fac[q] = (uint32_t)var_idx[q] | ((uint32_t)exponent[q] << 16);
  s->coeff.assign(coeff, coeff + n_terms * 2 * limbs);
  // Jacobian CSR: for (i, v) the factor slots of terms of f_i on x_v, in factor order.
  std::vector<int64_t> cnt((size_t)n_eq * n_var + 1, 0);
  for (int i = 0; i < n_eq; ++i)
    for (int64_t t = poly_ptr[i]; t < poly_ptr[i + 1]; ++t)
      for (int64_t q = term_ptr[t]; q < term_ptr[t + 1]; ++q) cnt[(size_t)i * n_var + var_idx[q] + 1]++;
  for (size_t e = 1; e < cnt.size(); ++e) {
    if (cnt[e]) s->nnz++;
    cnt[e] += cnt[e - 1];
  }
  s->jptr = cnt;
  s->jidx.resize(n_factors);
  {
    std::vector<int64_t> pos(cnt.begin(), cnt.end() - 1);
    for (int i = 0; i < n_eq; ++i)
      for (int64_t t = poly_ptr[i]; t < poly_ptr[i + 1]; ++t)
        for (int64_t q = term_ptr[t]; q < term_ptr[t + 1]; ++q) s->jidx[pos[(size_t)i * n_var + var_idx[q]]++] = q;
  }
  // operation counts actually performed per point (generic path: 4k-3 CM per term with k >= 1,
  // (E-1) CM + (E-1) integer scalings per variable in the power table)
  for (int64_t t = 0; t < n_terms; ++t) {
    const int64_t k = term_ptr[t + 1] - term_ptr[t];
    if (k >= 1) s->cm_per_point += 4 * k - 3;
  }
  s->cm_per_point += (int64_t)n_var * std::max(0, s->E - 1);
  s->ca_per_point = n_factors + n_terms;  // one add per contribution into a zero-initialised sum
  phc::plan_blocks(*s, &s->plan);
  {
    // latency path eligibility and its fixed split (independent of the call: reproducibility)
    int64_t max_terms = 0;
    for (int i = 0; i < n_eq; ++i) max_terms = std::max<int64_t>(max_terms, poly_ptr[i + 1] - poly_ptr[i]);
    const int W = s->scan_W;
    s->scan_smem = ((size_t)n_var * 2 * s->E + (size_t)W * n_var + W) * 2 * limbs * sizeof(double);
    s->scan_S = (int)std::max<int64_t>(1, std::min<int64_t>(148 / n_eq, (max_terms + W - 1) / W));
    // only for terms long enough that the block kernel's per-lane chain (4k - 3 products) is
    // the latency: measured kernel times tiny (k = 4) 9.2 us block vs 10.7 us latency path,
    // c2 (k = 10) 12.6 vs 12.5, c3 (k = 20) 75 vs 47 (tools/regime_ab.sh); k <= 2 tracker
    // systems: the block path is as fast or faster and steadier (tools/track_regime.py)
    s->scan_ok = kmax >= 12 && kmax <= 32 && s->scan_smem <= (size_t)200 * 1024 && max_terms > 0;
    // segmented latency path (QD): the segment width G (lanes per term, two factors per lane)
    // with the fewest products on the busiest scheduler, 8 + 2 ceil(log2 G) per lane times the
    // warp-tasks per scheduler (592 on a B200); W = 2 warps per CTA (more when the CTA count
    // would exceed two per SM), S splits so that each warp takes about one task
    if (s->scan_ok && limbs == 4) {  // DD: the warp-scan kernel is faster (batch config 13.0 vs 16.3 us)
      static const int widths[] = {4, 8, 10, 12, 16};
      int bestG = 0;
      double best = 1e300;
      const char* env = getenv("PHC_SEG");  // A/B hook: "G" forces a width, "0" the warp-scan path
      const int eg = env ? atoi(env) : -1;
      for (int G : widths) {
        if (2 * G < kmax) continue;
        if (eg >= 0 && G != eg) continue;
        int lg = 0;
        while ((1 << lg) < G) ++lg;
        int64_t tasks = 0;
        for (int i = 0; i < n_eq; ++i) tasks += (poly_ptr[i + 1] - poly_ptr[i] + 32 / G - 1) / (32 / G);
        const double est = (8.0 + 2 * lg) * std::max<double>(1.0, std::ceil(tasks / 592.0));
        if (est < best) best = est, bestG = G;
      }
      if (bestG > 0) {
        const int TPW = 32 / bestG;
        int W = 2;
        int64_t S = (max_terms + W * TPW - 1) / (W * TPW);
        while (n_eq * S > 2 * 148 && W < phc::kSegMaxWarps) {
          W *= 2;
          S = (max_terms + W * TPW - 1) / (W * TPW);
        }
        if (const char* ew = getenv("PHC_SEG_W")) {  // A/B hook: warps per CTA
          W = std::max(1, std::min(phc::kSegMaxWarps, atoi(ew)));
          S = (max_terms + W * TPW - 1) / (W * TPW);
        }
        if (const char* es = getenv("PHC_SEG_S")) S = std::max(1, atoi(es));  // test hook: splits
        s->seg_G = bestG;
        s->seg_W = W;
        s->seg_S = (int)std::max<int64_t>(1, S);
        s->seg_smem = (size_t)W * TPW * (n_var + 1) * 2 * limbs * sizeof(double);
        s->seg_ok = s->seg_smem <= (size_t)200 * 1024;
      }
    }
  }
  s->ca_per_point = s->plan.usable ? s->plan.ca_per_point : s->ca_per_point;
  DeviceState* d;
  int rc = get_device_state(s.get(), device, &d);
  if (rc) return rc;
  *out = s.release();
  return PHC_OK;
}

int phc_system_create_common(phc_system** out, int32_t n_eq, int32_t n_var, int32_t limbs, int64_t n_mono,
                             const int64_t* mono_ptr, const int32_t* var_idx, const int32_t* exponent,
                             const double* coeff, int32_t device) {
  g_err.clear();
  if (!out) return fail(PHC_EINVAL, "out is NULL");
  *out = nullptr;
  if (n_eq < 1 || n_var < 1) return fail(PHC_EINVAL, "n_eq and n_var must be >= 1 (got %d, %d)", n_eq, n_var);
  if (limbs != 2 && limbs != 4) return fail(PHC_EUNSUPPORTED, "limbs must be 2 (DD) or 4 (QD), got %d", limbs);
  if (n_mono < 1) return fail(PHC_EINVAL, "n_mono must be >= 1");
  if (n_mono > INT32_MAX) return fail(PHC_EUNSUPPORTED, "n_mono too large");
  if (!mono_ptr || !coeff) return fail(PHC_EINVAL, "NULL array");
  const size_t nc = (size_t)n_eq * n_mono * 2 * limbs;
  for (size_t q = 0; q < nc; ++q)
    if (!std::isfinite(coeff[q])) return fail(PHC_EINVAL, "coefficient limb %zu is not finite", q);
  // the monomials as a one-polynomial system with unit coefficients: validation, packing and
  // the monomial stage are those of an ordinary system (phc_system_create)
  std::vector<int64_t> pp(n_eq + 1, 0);
  pp[0] = 0;
  for (int i = 1; i <= n_eq; ++i) pp[i] = n_mono;  // polynomial 0 owns every monomial
  std::vector<double> ones((size_t)n_mono * 2 * limbs, 0.0);
  for (int64_t j = 0; j < n_mono; ++j) ones[(size_t)j * 2 * limbs] = 1.0;
  phc_system* s = nullptr;
  int rc = phc_system_create(&s, n_eq, n_var, limbs, n_mono, pp.data(), mono_ptr, var_idx, exponent, ones.data(),
                             device);
  if (rc) return rc;
  s->common = true;
  s->plan = phc::HostBlockPlan();  // the fused per-polynomial path does not apply
  {
    std::lock_guard<std::mutex> lk(s->mu);
    for (auto& kv : s->devs) kv.second->have_block = false;
  }
  // C^T [M][n_eq][2][L]
  const int cd = 2 * limbs;
  s->cT.resize(nc);
  for (int i = 0; i < n_eq; ++i)
    for (int64_t j = 0; j < n_mono; ++j)
      for (int c = 0; c < cd; ++c) s->cT[((size_t)j * n_eq + i) * cd + c] = coeff[((size_t)i * n_mono + j) * cd + c];
  // column lists: c = 0 every monomial (F), c = v + 1 the factor slots on variable v (J)
  std::vector<std::vector<std::pair<int32_t, int64_t>>> cols(n_var + 1);
  for (int64_t j = 0; j < n_mono; ++j) {
    cols[0].push_back({(int32_t)j, -1});
    for (int64_t q = mono_ptr[j]; q < mono_ptr[j + 1]; ++q) cols[var_idx[q] + 1].push_back({(int32_t)j, q});
  }
  s->cl_ptr.assign(1, 0);
  for (auto& c : cols) {
    for (auto& e : c) {
      s->cl_j.push_back(e.first);
      s->cl_q.push_back(e.second);
    }
    s->cl_ptr.push_back((int64_t)s->cl_j.size());
  }
  // counts: monomial stage (4k - 3 CM per monomial, power table) + coefficient product
  int64_t nz_vars = 0;
  for (int v = 0; v < n_var; ++v) nz_vars += cols[v + 1].empty() ? 0 : 1;
  s->nnz = (int64_t)n_eq * nz_vars;
  const int64_t cma = (int64_t)n_eq * (n_mono + s->n_factors);
  s->cm_per_point += cma;
  s->ca_per_point = cma;
  DeviceState* d;
  if ((rc = get_device_state(s, s->home, &d))) {
    phc_system_destroy(s);
    return rc;
  }
  // the home replica was made before the common tables existed: add them now
  {
    DeviceGuard g(s->home);
    if ((rc = dalloc(&d->cl_ptr, s->cl_ptr.size())) || (rc = dalloc(&d->cl_j, s->cl_j.size())) ||
        (rc = dalloc(&d->cl_q, s->cl_q.size())) || (rc = dalloc(&d->cT, s->cT.size())) ||
        (rc = upload(d->cl_ptr, s->cl_ptr.data(), s->cl_ptr.size() * 8)) ||
        (rc = upload(d->cl_j, s->cl_j.data(), s->cl_j.size() * 4)) ||
        (rc = upload(d->cl_q, s->cl_q.data(), s->cl_q.size() * 8)) ||
        (rc = upload(d->cT, s->cT.data(), s->cT.size() * 8))) {
      phc_system_destroy(s);
      return rc;
    }
  }
  *out = s;
  return PHC_OK;
}

void phc_system_destroy(phc_system* s) {
  if (!s) return;
  {
    DeviceGuard g(s->home);
    if (s->hx) cudaFree(s->hx);
    if (s->hf) cudaFree(s->hf);
    if (s->hj) cudaFree(s->hj);
    if (s->hstream) cudaStreamDestroy(s->hstream);
    if (s->hstream2) cudaStreamDestroy(s->hstream2);
  }
  s->devs.clear();
  {
    DeviceGuard g(s->home);
    for (auto& r : s->recs) { cudaEventDestroy(r.a); cudaEventDestroy(r.b); }
    for (auto e : s->pool) cudaEventDestroy(e);
  }
  delete s;
}

int phc_eval_jacobian_batch(const phc_system* s, int64_t n_points, const double* x, double* f, double* jac,
                            const int32_t* devices, int32_t n_devices, void* stream) {
  return eval_batch_impl(s, n_points, x, nullptr, f, jac, devices, n_devices, stream);
}

int phc_eval_jacobian_batch_range(const phc_system* cs, int64_t n_points, int64_t p_begin, int64_t p_end,
                                  const double* x, double* f, double* jac, void* stream) {
  g_err.clear();
  phc_system* s = const_cast<phc_system*>(cs);
  if (!s) return fail(PHC_EINVAL, "NULL system");
  if (n_points < 0 || p_begin < 0 || p_end < p_begin || p_end > n_points)
    return fail(PHC_EINVAL, "need 0 <= p_begin <= p_end <= n_points (got %lld, %lld, %lld)", (long long)p_begin,
                (long long)p_end, (long long)n_points);
  if (p_end == p_begin) return PHC_OK;
  if (!x || !f || !jac) return fail(PHC_EINVAL, "NULL x/f/jac");
  if ((((uintptr_t)x) | ((uintptr_t)f) | ((uintptr_t)jac)) & 31) return fail(PHC_EINVAL, "x/f/jac must be 32-byte aligned");
  const int64_t cd = 2 * s->L;
  DeviceGuard g(s->home);
  DeviceState* d;
  int rc = get_device_state(s, s->home, &d);
  if (rc) return rc;
  // call_points = n_points: the regime of the whole call, so the rows are bitwise those of
  // phc_eval_jacobian_batch over all n_points (determinism, phc.h)
  return run_on_device(s, d, p_end - p_begin, x + p_begin * s->n_var * cd, nullptr, f + p_begin * s->n_eq * cd,
                       jac + p_begin * (int64_t)s->n_eq * s->n_var * cd, (cudaStream_t)stream, n_points);
}

// cuMemGetAddressRange through the runtime's driver entry point (no link-time libcuda, so the
// library still loads on hosts without a driver)
typedef int (*phc_get_range_fn)(unsigned long long*, size_t*, unsigned long long);

int phc_ipc_get_handle(const void* dev_ptr, void* handle, int64_t* offset) {
  g_err.clear();
  if (!dev_ptr || !handle || !offset) return fail(PHC_EINVAL, "NULL argument");
  static phc_get_range_fn range = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      fn = nullptr;
    return (phc_get_range_fn)fn;
  }();
  if (!range) return fail(PHC_ECUDA, "cuMemGetAddressRange not available");
  unsigned long long base = 0;
  size_t size = 0;
  if (range(&base, &size, (unsigned long long)(uintptr_t)dev_ptr) != 0) return fail(PHC_EINVAL, "not a device allocation");
  CUDA_TRY(cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(handle), (void*)(uintptr_t)base));
  *offset = (int64_t)((uintptr_t)dev_ptr - (uintptr_t)base);
  return PHC_OK;
}

static int check_device(int32_t device) {
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) return fail(PHC_ECUDA, "cudaGetDeviceCount failed");
  if (device < 0 || device >= c) return fail(PHC_EINVAL, "device %d out of range (%d devices)", device, c);
  return PHC_OK;
}

int phc_ipc_open(const void* handle, int32_t device, void** base) {
  g_err.clear();
  if (!handle || !base) return fail(PHC_EINVAL, "NULL argument");
  if (int rc = check_device(device)) return rc;
  DeviceGuard g(device);
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof(h));
  CUDA_TRY(cudaIpcOpenMemHandle(base, h, cudaIpcMemLazyEnablePeerAccess));
  return PHC_OK;
}

int phc_ipc_close(void* base, int32_t device) {
  g_err.clear();
  if (!base) return PHC_OK;
  if (int rc = check_device(device)) return rc;
  DeviceGuard g(device);
  CUDA_TRY(cudaIpcCloseMemHandle(base));
  return PHC_OK;
}

int phc_eval_homotopy_batch(const phc_system* s, int64_t n_points, const double* x, const double* t, double* f,
                            double* jac, const int32_t* devices, int32_t n_devices, void* stream) {
  g_err.clear();
  if (!s) return fail(PHC_EINVAL, "NULL system");
  if (!s->has_target) return fail(PHC_EINVAL, "no target coefficients: call phc_system_set_target first");
  if (n_points > 0 && !t) return fail(PHC_EINVAL, "NULL t");
  return eval_batch_impl(s, n_points, x, t, f, jac, devices, n_devices, stream);
}

int phc_system_set_target(phc_system* s, const double* coeff_target) {
  g_err.clear();
  if (!s) return fail(PHC_EINVAL, "NULL system");
  if (s->n_terms > 0 && !coeff_target) return fail(PHC_EINVAL, "NULL coeff_target");
  if (s->common) {  // dense target matrix [n_eq][n_mono][2][L], stored transposed
    const int cd = 2 * s->L;
    const size_t nc = (size_t)s->n_eq * s->n_terms * cd;
    for (size_t q = 0; q < nc; ++q)
      if (!std::isfinite(coeff_target[q])) return fail(PHC_EINVAL, "target coefficient limb %zu is not finite", q);
    {
      DeviceGuard g(s->home);
      cudaDeviceSynchronize();
    }
    s->cT2.resize(nc);
    for (int i = 0; i < s->n_eq; ++i)
      for (int64_t j = 0; j < s->n_terms; ++j)
        for (int c = 0; c < cd; ++c)
          s->cT2[((size_t)j * s->n_eq + i) * cd + c] = coeff_target[((size_t)i * s->n_terms + j) * cd + c];
    s->has_target = true;
    std::lock_guard<std::mutex> lk(s->mu);
    for (auto& kv : s->devs) {
      int rc = upload_target(s, kv.second.get());
      if (rc) return rc;
    }
    return PHC_OK;
  }
  const size_t nc = (size_t)s->n_terms * 2 * s->L;
  for (size_t q = 0; q < nc; ++q)
    if (!std::isfinite(coeff_target[q])) return fail(PHC_EINVAL, "target coefficient limb %zu is not finite", q);
  {
    DeviceGuard g(s->home);
    cudaDeviceSynchronize();  // no evaluation may be reading the previous target
  }
  s->coeff2.assign(coeff_target, coeff_target + nc);
  if (nc == 0) s->coeff2.assign(1, 0.0);
  s->has_target = true;
  std::lock_guard<std::mutex> lk(s->mu);
  for (auto& kv : s->devs) {
    int rc = upload_target(s, kv.second.get());
    if (rc) return rc;
  }
  return PHC_OK;
}

int phc_homotopy_old_create(phc_system** out, int32_t n_eq, int32_t n_var, int32_t limbs, int64_t n_terms,
                            const int64_t* poly_ptr, const int64_t* term_ptr, const int32_t* var_idx,
                            const int32_t* exponent, const double* coeff_start, const double* coeff_target,
                            int32_t device) {
  g_err.clear();
  if (!out) return fail(PHC_EINVAL, "out is NULL");
  *out = nullptr;
  if (n_eq < 1 || n_var < 1 || n_terms < 0 || !poly_ptr || !term_ptr) return fail(PHC_EINVAL, "malformed input");
  if (limbs != 2 && limbs != 4) return fail(PHC_EUNSUPPORTED, "limbs must be 2 or 4");
  if (n_terms > 0 && (!coeff_start || !coeff_target)) return fail(PHC_EINVAL, "NULL coefficients");
  if (n_terms > 0 && term_ptr[n_terms] > 0 && (!var_idx || !exponent)) return fail(PHC_EINVAL, "NULL var_idx/exponent");
  if (poly_ptr[0] != 0 || poly_ptr[n_eq] != n_terms || term_ptr[0] != 0)
    return fail(PHC_EINVAL, "poly_ptr/term_ptr must start at 0 and poly_ptr end at n_terms");
  for (int i = 0; i < n_eq; ++i)
    if (poly_ptr[i + 1] < poly_ptr[i]) return fail(PHC_EINVAL, "poly_ptr not monotone at %d", i);
  for (int64_t t = 0; t < n_terms; ++t)
    if (term_ptr[t + 1] < term_ptr[t]) return fail(PHC_EINVAL, "term_ptr not monotone at %lld", (long long)t);
  // each term c x^a of h = (1 - t) c_s x^a + t c_f x^a becomes c_s x^a, -c_s t x^a, c_f t x^a,
  // with t the variable n_var ("t treated as just another variable")
  const int cd = 2 * limbs;
  std::vector<int64_t> pp(1, 0), tp(1, 0);
  std::vector<int32_t> vi, ex;
  std::vector<double> cf;
  for (int i = 0; i < n_eq; ++i) {
    for (int64_t t = poly_ptr[i]; t < poly_ptr[i + 1]; ++t) {
      for (int copy = 0; copy < 3; ++copy) {
        for (int64_t q = term_ptr[t]; q < term_ptr[t + 1]; ++q) {
          vi.push_back(var_idx ? var_idx[q] : 0);
          ex.push_back(exponent ? exponent[q] : 0);
        }
        if (copy > 0) {
          vi.push_back(n_var);
          ex.push_back(1);
        }
        tp.push_back((int64_t)vi.size());
        const double* c = (copy == 2 ? coeff_target : coeff_start) + t * cd;
        for (int j = 0; j < cd; ++j) cf.push_back(copy == 1 ? -c[j] : c[j]);
      }
    }
    pp.push_back((int64_t)tp.size() - 1);
  }
  return phc_system_create(out, n_eq, n_var + 1, limbs, (int64_t)tp.size() - 1, pp.data(), tp.data(), vi.data(),
                           ex.data(), cf.data(), device);
}

int phc_eval_jacobian(const phc_system* s, const double* x, double* f, double* jac, void* stream) {
  return phc_eval_jacobian_batch(s, 1, x, f, jac, nullptr, 0, stream);
}

int phc_eval_jacobian_batch_host(const phc_system* cs, int64_t n_points, const double* x_host, double* f_host,
                                 double* jac_host, const int32_t* devices, int32_t n_devices) {
  g_err.clear();
  phc_system* s = const_cast<phc_system*>(cs);
  if (!s) return fail(PHC_EINVAL, "NULL system");
  if (n_points < 0) return fail(PHC_EINVAL, "n_points < 0");
  if (n_points == 0) return PHC_OK;
  if (!x_host || !f_host || !jac_host) return fail(PHC_EINVAL, "NULL host pointer");
  DeviceGuard g(s->home);
  const int64_t cd = 2 * s->L;
  if (!s->hstream) CUDA_TRY(cudaStreamCreateWithFlags(&s->hstream, cudaStreamNonBlocking));
  if (n_points > s->h_cap) {
    cudaStreamSynchronize(s->hstream);
    if (s->hx) cudaFree(s->hx);
    if (s->hf) cudaFree(s->hf);
    if (s->hj) cudaFree(s->hj);
    s->hx = s->hf = s->hj = nullptr;
    s->h_cap = 0;
    int rc;
    if ((rc = dalloc(&s->hx, (size_t)(n_points * s->n_var * cd)))) return rc;
    if ((rc = dalloc(&s->hf, (size_t)(n_points * s->n_eq * cd)))) return rc;
    if ((rc = dalloc(&s->hj, (size_t)(n_points * (int64_t)s->n_eq * s->n_var * cd)))) return rc;
    s->h_cap = n_points;
  }
  const bool single = !devices || n_devices <= 0 || (n_devices == 1 && devices[0] == s->home);
  if (!single) {
    CUDA_TRY(cudaMemcpyAsync(s->hx, x_host, n_points * s->n_var * cd * 8, cudaMemcpyHostToDevice, s->hstream));
    int rc = phc_eval_jacobian_batch(s, n_points, s->hx, s->hf, s->hj, devices, n_devices, s->hstream);
    if (rc) return rc;
    CUDA_TRY(cudaMemcpyAsync(f_host, s->hf, n_points * s->n_eq * cd * 8, cudaMemcpyDeviceToHost, s->hstream));
    CUDA_TRY(cudaMemcpyAsync(jac_host, s->hj, n_points * (int64_t)s->n_eq * s->n_var * cd * 8,
                             cudaMemcpyDeviceToHost, s->hstream));
    CUDA_TRY(cudaStreamSynchronize(s->hstream));
    return PHC_OK;
  }
  // one device: a pipeline over chunks of points -- H2D and evaluation of chunk c on
  // hstream, its D2H on a second stream, so the output copies (the bulk of the bytes: J)
  // overlap the evaluation of the following chunks.  Every chunk is evaluated with the
  // call's total point count as its regime (run_on_device call_points), so the results are
  // bitwise those of the unchunked call.
  if (!s->hstream2) CUDA_TRY(cudaStreamCreateWithFlags(&s->hstream2, cudaStreamNonBlocking));
  DeviceState* d;
  int rc = get_device_state(s, s->home, &d);
  if (rc) return rc;
  // chunks of ~128 MiB of output (the last chunk's copy is the exposed tail), at least 256
  // points each (a chunk must still fill the GPU), at most 64
  const int64_t out_bytes = n_points * (int64_t)s->n_eq * (s->n_var + 1) * cd * 8;
  int64_t chunks = std::min<int64_t>(64, std::max<int64_t>(1, out_bytes >> 27));
  chunks = std::max<int64_t>(1, std::min<int64_t>(chunks, n_points / 256));
  std::vector<cudaEvent_t> evs;
  for (int64_t c = 0; c < chunks; ++c) {
    const int64_t p0 = c * n_points / chunks, p1 = (c + 1) * n_points / chunks, np = p1 - p0;
    if (np == 0) continue;
    CUDA_TRY(cudaMemcpyAsync(s->hx + p0 * s->n_var * cd, x_host + p0 * s->n_var * cd, np * s->n_var * cd * 8,
                             cudaMemcpyHostToDevice, s->hstream));
    if ((rc = run_on_device(s, d, np, s->hx + p0 * s->n_var * cd, nullptr, s->hf + p0 * s->n_eq * cd,
                            s->hj + p0 * (int64_t)s->n_eq * s->n_var * cd, s->hstream, n_points)))
      break;
    cudaEvent_t e;
    CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    evs.push_back(e);
    CUDA_TRY(cudaEventRecord(e, s->hstream));
    CUDA_TRY(cudaStreamWaitEvent(s->hstream2, e, 0));
    CUDA_TRY(cudaMemcpyAsync(f_host + p0 * s->n_eq * cd, s->hf + p0 * s->n_eq * cd, np * s->n_eq * cd * 8,
                             cudaMemcpyDeviceToHost, s->hstream2));
    CUDA_TRY(cudaMemcpyAsync(jac_host + p0 * (int64_t)s->n_eq * s->n_var * cd,
                             s->hj + p0 * (int64_t)s->n_eq * s->n_var * cd,
                             np * (int64_t)s->n_eq * s->n_var * cd * 8, cudaMemcpyDeviceToHost, s->hstream2));
  }
  cudaStreamSynchronize(s->hstream);
  cudaStreamSynchronize(s->hstream2);
  for (cudaEvent_t e : evs) cudaEventDestroy(e);
  if (rc) return rc;
  CUDA_TRY(cudaGetLastError());
  return PHC_OK;
}

int phc_profile_enable(const phc_system* cs, int enable) {
  phc_system* s = const_cast<phc_system*>(cs);
  if (!s) return fail(PHC_EINVAL, "NULL system");
  s->prof = enable != 0;
  return PHC_OK;
}

int phc_profile_read(const phc_system* cs, double ms[4], int64_t launches[4], int reset) {
  phc_system* s = const_cast<phc_system*>(cs);
  if (!s || !ms || !launches) return fail(PHC_EINVAL, "NULL argument");
  DeviceGuard g(s->home);
  for (auto& r : s->recs) {
    CUDA_TRY(cudaEventSynchronize(r.b));
    float t = 0;
    CUDA_TRY(cudaEventElapsedTime(&t, r.a, r.b));
    s->prof_ms[r.cls] += t;
    s->prof_n[r.cls] += 1;
    s->pool.push_back(r.a);
    s->pool.push_back(r.b);
  }
  s->recs.clear();
  for (int c = 0; c < 4; ++c) {
    ms[c] = s->prof_ms[c];
    launches[c] = s->prof_n[c];
    if (reset) { s->prof_ms[c] = 0; s->prof_n[c] = 0; }
  }
  return PHC_OK;
}

int phc_system_stats(const phc_system* s, int64_t out[PHC_STATS_LEN]) {
  if (!s || !out) return fail(PHC_EINVAL, "NULL argument");
  out[0] = s->n_terms;
  out[1] = s->n_factors;
  out[2] = s->kmax;
  out[3] = s->E;
  out[4] = s->nnz;
  out[5] = s->plan.usable ? s->plan.cm_per_point : s->cm_per_point;
  out[6] = s->ca_per_point;
  out[7] = s->plan.usable ? s->plan.launches : 3;  // generic and common paths: 3 kernels
  if (s->plan.usable) {
    out[8] = s->plan.exec_flops_per_point;
  } else if (s->common) {
    const phc::OpFlops f = phc::op_flops(s->L);
    const int64_t mono_cm = s->cm_per_point - s->ca_per_point;  // monomial stage + power table products
    out[8] = mono_cm * f.cm + (int64_t)s->n_var * std::max(0, s->E - 1) * f.ci + s->ca_per_point * (f.cm_lazy + f.ca_lazy + f.acc_norm) +
             (int64_t)s->n_eq * (s->n_var + 1) * f.norm;
  } else {
    const phc::OpFlops f = phc::op_flops(s->L);
    out[8] = s->cm_per_point * f.cm + s->ca_per_point * f.ca + (int64_t)s->n_var * std::max(0, s->E - 1) * f.ci;
  }
  out[9] = s->plan.usable ? 1 : 0;
  out[10] = s->plan.usable ? s->plan.layout : -1;
  out[11] = s->plan.usable ? s->plan.K : s->kmax;
  {
    // latency path (kernels_scan.cuh): per term 1 + 10 + 2 complex products on all 32 lanes
    // (normalised), k + 1 additions; per CTA the power table (<= 2 log2(E) + 1 products and
    // one integer scaling per entry), n_eq * S CTAs per point
    const phc::OpFlops f = phc::op_flops(s->L);
    int64_t fl = 0;
    if (s->seg_ok && !s->common) {
      // segmented path: per warp-task (32 / G terms) 8 + 2 ceil(log2 G) lazy products on all
      // 32 lanes (the first task of a slot stores its partials, no addition); the global power
      // table once per point (<= 2 log2(E) + 1 products and one integer scaling per entry); the
      // epilogue's lazy additions and one renormalisation per stored entry
      int lg = 0, lgE = 0;
      while ((1 << lg) < s->seg_G) ++lg;
      while ((1 << lgE) < s->E) ++lgE;
      const int TPW = 32 / s->seg_G;
      for (int i = 0; i < s->n_eq; ++i) {
        const int64_t nt = s->poly_ptr[i + 1] - s->poly_ptr[i];
        fl += (nt + TPW - 1) / TPW * 32 * (8 + 2 * lg) * (int64_t)f.cm_lazy;
      }
      fl += (int64_t)(s->n_var + 1) * s->E * ((2 * lgE + 1) * (int64_t)f.cm + f.ci);
      fl += (int64_t)s->n_eq * s->seg_S * (s->n_var + 1) * (s->seg_W * TPW - 1) * (int64_t)f.ca_lazy;
      fl += (int64_t)s->n_eq * (s->seg_S - 1) * (s->n_var + 1) * (int64_t)f.ca_lazy;
      fl += (int64_t)s->n_eq * (s->n_var + 1) * (int64_t)f.norm;
    } else if (s->scan_ok && !s->common) {
      for (int64_t t = 0; t < s->n_terms; ++t) {
        const int64_t k = s->term_ptr[t + 1] - s->term_ptr[t];
        fl += 32 * 13 * (int64_t)f.cm + (k + 1) * f.ca;
      }
      int lg = 0;
      while ((1 << lg) < s->E) ++lg;
      fl += (int64_t)s->n_eq * s->scan_S * s->n_var * s->E * ((2 * lg + 1) * (int64_t)f.cm + f.ci);
      fl += (int64_t)s->n_eq * s->scan_S * (s->n_var + 1) * (s->scan_W - 1) * (int64_t)f.ca;
    }
    out[12] = fl;
    out[13] = s->scan_ok && !s->common ? kScanMaxTerms : 0;
    out[14] = s->common ? 1 : 0;
    const bool lat = s->scan_ok && !s->common;
    out[15] = !lat ? 0 : s->seg_ok ? 2 : 1;
    out[16] = lat && s->seg_ok ? s->seg_G : 0;
    out[17] = !lat ? 0 : s->seg_ok ? 2 : 1;  // segmented: the power table, then the kernel
  }
  return PHC_OK;
}

#if PHC_SEG_TRACE
// diagnostic builds only (PHC_SEG_TRACE): the per-CTA phase stamps of the last segmented call
int phc_debug_seg_trace(unsigned long long* out, int n_ctas) {
  if (cudaDeviceSynchronize() != cudaSuccess) return PHC_ECUDA;
  n_ctas = std::min(n_ctas, 4096);
  if (cudaMemcpyFromSymbol(out, phc::g_seg_trace, (size_t)n_ctas * 8 * sizeof(unsigned long long)) != cudaSuccess)
    return PHC_ECUDA;
  return PHC_OK;
}
#endif

}  // extern "C"
