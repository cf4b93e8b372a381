// Internal runtime of the C ABI (include/phc.h), shared by the library's translation units:
// the system handle, the per-device replicas and scratch, error reporting, the launch
// dispatch of the evaluation paths.  Not installed; nothing here is part of the ABI.
#pragma once
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/phc.h"
#include "kernels_block.cuh"

namespace phc_rt {

extern thread_local std::string g_err;

int fail(int code, const char* fmt, ...);

#define CUDA_TRY(expr)                                                                         \
  do {                                                                                         \
    cudaError_t e_ = (expr);                                                                   \
    if (e_ != cudaSuccess) return fail(PHC_ECUDA, "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

template <class T>
int dalloc(T** p, size_t n) {
  if (n == 0) n = 1;
  cudaError_t e = cudaMalloc((void**)p, n * sizeof(T));
  if (e != cudaSuccess) {
    *p = nullptr;
    cudaGetLastError();
    return fail(PHC_ENOMEM, "cudaMalloc(%zu bytes): %s", n * sizeof(T), cudaGetErrorString(e));
  }
  return PHC_OK;
}

// Per-device replica of the packed tables plus scratch (tables
// replicated once per device at first use).
struct DeviceState {
  int dev = -1;
  cudaStream_t stream = nullptr;   // internal stream for non-home shards
  cudaStream_t stream2 = nullptr;  // gather stream of the non-home shards
  cudaEvent_t done = nullptr;
  // generic path tables
  int64_t* term_ptr = nullptr;
  uint32_t* fac = nullptr;
  double* coeff = nullptr;
  double* coeff2 = nullptr;  // NEXT-3 homotopy target coefficients (term order)
  int64_t* poly_ptr = nullptr;
  int64_t* jptr = nullptr;
  int64_t* jidx = nullptr;
  // common-support tables (NEXT-2): column lists and C transposed
  int64_t* cl_ptr = nullptr;
  int32_t* cl_j = nullptr;
  int64_t* cl_q = nullptr;
  double* cT = nullptr;
  double* cT2 = nullptr;  // homotopy target of a common-support system
  // block path tables
  phc::BlockTables bt{};
  bool have_block = false;
  // scratch
  double* PT = nullptr;
  double* Y = nullptr;
  double* G = nullptr;
  int64_t chunk_cap = 0;
  // Newton-step workspace (evaluation outputs and the global elimination matrix)
  double* nF = nullptr;
  double* nJ = nullptr;
  double* nM = nullptr;
  int64_t n_cap = 0, nM_cap = 0;
  double* nAux = nullptr;  // cooperative elimination: per-CTA residuals, row permutation, flag
  int64_t naux_cap = 0;
  // latency (warp-scan) path: partial rows of the S splits
  double* part = nullptr;
  int64_t part_cap = 0;
  int* count = nullptr;  // arrival counters (zeroed at allocation; each call leaves them zero)
  int64_t count_cap = 0;
  // segmented latency path: the global power table of the call's points
  double* segPT = nullptr;
  int64_t segPT_cap = 0;
  // staging buffers for remote shards
  double* xs = nullptr;
  double* fs = nullptr;
  double* js = nullptr;
  double* ts = nullptr;  // t per point (homotopy shards)
  int64_t stage_cap = 0;
  ~DeviceState() {
    DeviceGuard g(dev);
    for (void* p : {(void*)term_ptr, (void*)fac, (void*)coeff, (void*)poly_ptr, (void*)jptr, (void*)jidx, (void*)PT,
                    (void*)Y, (void*)G, (void*)xs, (void*)fs, (void*)js, (void*)ts, (void*)bt.fac, (void*)bt.coeff,
                    (void*)bt.blk, (void*)bt.PT, (void*)coeff2, (void*)bt.coeff2, (void*)cl_ptr, (void*)cl_j,
                    (void*)cl_q, (void*)cT, (void*)part, (void*)count, (void*)cT2, (void*)nF, (void*)nJ,
                    (void*)nM, (void*)nAux, (void*)segPT})
      if (p) cudaFree(p);
    if (stream) cudaStreamDestroy(stream);
    if (stream2) cudaStreamDestroy(stream2);
    if (done) cudaEventDestroy(done);
  }
};


}  // namespace phc_rt

struct phc_system {
  int32_t n_eq = 0, n_var = 0, L = 0, home = 0;
  int64_t n_terms = 0, n_factors = 0;
  int kmax = 0, E = 1;
  int64_t nnz = 0;
  int64_t cm_per_point = 0, ca_per_point = 0;
  // host copies
  std::vector<int64_t> poly_ptr, term_ptr;
  std::vector<uint32_t> fac;
  std::vector<double> coeff;
  std::vector<double> coeff2;  // NEXT-3: homotopy target coefficients (empty: not a homotopy)
  // NEXT-2 common-support system: "terms" are the M shared monomials (unit coefficients),
  // C^T [M][n_eq][2][L] and the per-column lists of the coefficient product
  bool common = false;
  bool fused_gather = true;   // remote shards write F, J into home memory over NVLink (else staged copies)
  bool has_target = false;    // NEXT-3 target attached (coeff2, or cT2 for common systems)
  std::vector<double> cT2;    // common systems: target C^T [M][n_eq][2][L]
  // latency path (kernels_scan.cuh): eligible when k <= 32 and the CTA's table + rows fit
  bool scan_ok = false;
  int scan_S = 1, scan_W = 8;
  size_t scan_smem = 0;
  // segmented latency path (kernels_scan.cuh poly_seg_kernel, QD): G lanes per term (two
  // factors per lane), W warps per CTA, S splits per polynomial; takes the place of the
  // warp-scan path when seg_ok
  bool seg_ok = false;
  int seg_G = 0, seg_W = 2, seg_S = 1;
  size_t seg_smem = 0;
  std::vector<int64_t> cl_ptr, cl_q;
  std::vector<int32_t> cl_j;
  std::vector<double> cT;
  std::vector<int64_t> jptr, jidx;
  phc::HostBlockPlan plan;  // warp-per-block layout (kernels_block.cuh)
  std::mutex mu;
  std::map<int, std::unique_ptr<phc_rt::DeviceState>> devs;
  // host-API staging on the home device
  double *hx = nullptr, *hf = nullptr, *hj = nullptr;
  int64_t h_cap = 0;
  cudaStream_t hstream = nullptr;
  cudaStream_t hstream2 = nullptr;  // D2H stream of the pipelined host call
  // kernel timing (phc_profile_*): events on the launch stream, home device only
  bool prof = false;
  struct Rec { int cls; cudaEvent_t a, b; };
  std::vector<Rec> recs;
  std::vector<cudaEvent_t> pool;
  double prof_ms[4] = {0, 0, 0, 0};
  int64_t prof_n[4] = {0, 0, 0, 0};
};

namespace phc_rt {

cudaEvent_t pool_event(phc_system* s);

// Brackets one kernel launch with events on its stream when profiling is on.
struct ProfScope {
  phc_system* s;
  int cls;
  cudaStream_t st;
  cudaEvent_t a = nullptr;
  ProfScope(const phc_system* cs, int dev, int cls_, cudaStream_t st_) : s(const_cast<phc_system*>(cs)), cls(cls_), st(st_) {
    if (!s->prof || dev != s->home) { s = nullptr; return; }
    a = pool_event(s);
    cudaEventRecord(a, st);
  }
  ~ProfScope() {
    if (!s) return;
    cudaEvent_t b = pool_event(s);
    cudaEventRecord(b, st);
    s->recs.push_back({cls, a, b});
  }
};

inline size_t cbytes(const phc_system* s) { return (size_t)2 * s->L * sizeof(double); }


constexpr int64_t kScanMaxTerms = 148 * 32;  // call_points * n_terms at or below: latency path

int upload(void* dst, const void* src, size_t bytes);
int upload_target(const phc_system* s, DeviceState* d);
int get_device_state(phc_system* s, int dev, DeviceState** out);
int ensure_scratch(const phc_system* s, DeviceState* d, int64_t want_points);
int ensure_stage(const phc_system* s, DeviceState* d, int64_t np);
// Evaluate n_points points resident on device d (T: t per point for the homotopy, or nullptr);
// call_points = the caller's total point count (regime selection), -1 = n_points.
int run_on_device(const phc_system* s, DeviceState* d, int64_t n_points, const double* x, const double* T, double* f,
                  double* jac, cudaStream_t st, int64_t call_points = -1);
// Shared bodies of the batch evaluation and Newton calls (T = t per point or nullptr).
int eval_batch_impl(const phc_system* s, int64_t n_points, const double* x, const double* T, double* f, double* jac,
                    const int32_t* devices, int32_t n_devices, void* stream);
int newton_impl(const phc_system* s, int64_t n_points, const double* x, const double* T, double* x_new,
                double* residual, int32_t* status, void* stream);

template <class T>
struct HostBuf {  // RAII pinned host buffer (the tracker's per-step exchange arrays)
  T* p = nullptr;
  int alloc(size_t n) {
    if (cudaMallocHost((void**)&p, std::max<size_t>(n, 1) * sizeof(T)) != cudaSuccess) {
      p = nullptr;
      cudaGetLastError();
      return fail(PHC_ENOMEM, "cudaMallocHost(%zu bytes) failed", n * sizeof(T));
    }
    return PHC_OK;
  }
  T& operator[](size_t i) { return p[i]; }
  ~HostBuf() { if (p) cudaFreeHost(p); }
};

template <class T>
struct DevBuf {  // RAII device buffer (the tracker's workspace)
  T* p = nullptr;
  ~DevBuf() { if (p) cudaFree(p); }
};


}  // namespace phc_rt
