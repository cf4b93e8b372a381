// NEXT-1 host side: one Newton iteration per point (Alg. 2) -- the
// evaluation (run_on_device) followed by the elimination kernels of kernels_newton.cuh.
#include "runtime.h"
#include "kernels_newton.cuh"

namespace phc_rt {

constexpr int64_t kCoopMaxPoints = 4;  // cooperative elimination up to this many points per call

// Multi-kernel elimination (kernels_newton.cuh) for matrices beyond shared memory.
template <int L>
void newton_multi(const phc::NewtonArgs& a, int64_t np, cudaStream_t st) {
  const int n = a.n;
  phc::newton_load_kernel<L><<<(unsigned)np, 256, 0, st>>>(a);
  for (int k = 0; k < n; ++k) {
    phc::newton_pivot_kernel<L><<<(unsigned)np, 256, 0, st>>>(a, k);
    const int64_t work = (int64_t)(n - k - 1) * (n - k);
    if (work > 0) phc::newton_update_kernel<L><<<dim3((unsigned)((work + 255) / 256), (unsigned)np), 256, 0, st>>>(a, k);
  }
  phc::newton_backsub_kernel<L><<<(unsigned)np, 256, 0, st>>>(a);
}

// One cooperative launch per chunk (kernels_newton.cuh newton_coop_kernel): one CTA per SM.
template <int L>
int newton_coop(const phc::NewtonArgs& a, DeviceState* d, cudaStream_t st) {
  static std::mutex mu;
  static std::map<int, int> sms;  // device -> SM count (cooperative grid size)
  int G;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = sms.find(d->dev);
    if (it == sms.end()) {
      int nsm = 0;
      CUDA_TRY(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, d->dev));
      it = sms.emplace(d->dev, nsm).first;
    }
    G = it->second;
  }
  if (const char* e = getenv("PHC_NEWTON_COOP_CTAS")) G = std::max(2, std::min(G, atoi(e)));  // A/B hook
  const size_t smem = phc::coop_smem_bytes(a.n, L);
  if (smem > 48 * 1024) CUDA_TRY(phc::ensure_smem((const void*)phc::newton_coop_kernel<L>, smem));
  int nb = 0;
  CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, phc::newton_coop_kernel<L>, phc::kCoopThreads, smem));
  if (nb < 1) return fail(PHC_ECUDA, "cooperative elimination kernel does not fit an SM");
  const int64_t need = G + a.n + 2;
  if (d->naux_cap < need) {
    cudaStreamSynchronize(st);
    if (d->nAux) cudaFree(d->nAux);
    d->nAux = nullptr;
    d->naux_cap = 0;
    int rc = dalloc(&d->nAux, (size_t)need);
    if (rc) return rc;
    d->naux_cap = need;
  }
  double* red = d->nAux;
  int32_t* perm = reinterpret_cast<int32_t*>(d->nAux + G);
  int32_t* flag = perm + 2 * a.n;
  phc::NewtonArgs args = a;
  void* kargs[] = {(void*)&args, (void*)&perm, (void*)&red, (void*)&flag};
  CUDA_TRY(cudaLaunchCooperativeKernel((const void*)phc::newton_coop_kernel<L>, dim3((unsigned)G), dim3(phc::kCoopThreads), kargs, smem, st));
  return PHC_OK;
}

int newton_impl(const phc_system* cs, int64_t n_points, const double* x, const double* T, double* x_new,
                       double* residual, int32_t* status, void* stream) {
  g_err.clear();
  phc_system* s = const_cast<phc_system*>(cs);
  if (!s) return fail(PHC_EINVAL, "NULL system");
  if (s->n_eq != s->n_var) return fail(PHC_EINVAL, "Newton needs a square system (n_eq %d != n_var %d)", s->n_eq, s->n_var);
  if (n_points < 0) return fail(PHC_EINVAL, "n_points < 0");
  if (n_points == 0) return PHC_OK;
  if (!x || !x_new || !residual || !status) return fail(PHC_EINVAL, "NULL pointer");
  if ((((uintptr_t)x) | ((uintptr_t)x_new)) & 31) return fail(PHC_EINVAL, "x/x_new must be 32-byte aligned");
  DeviceGuard g(s->home);
  DeviceState* d;
  int rc = get_device_state(s, s->home, &d);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  const int n = s->n_eq, L = s->L;
  const int64_t cd = 2 * L;
  const size_t mat = ((size_t)n * (n + 1) + n) * cd * sizeof(double);  // [J | -F] + pivot reciprocals
  const size_t smat = phc::solve_smem_bytes(n, L);                                     // + permutations
  const bool smem = smat <= (size_t)200 * 1024 && !getenv("PHC_NEWTON_GLOBAL");  // (test hook: global-memory paths)
  const int64_t per_point = (int64_t)n * n * cd * 8 + (smem ? 0 : (int64_t)mat);
  const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(n_points, ((int64_t)512 << 20) / per_point));
  if (d->n_cap < chunk) {
    cudaStreamSynchronize(st);
    for (double** q : {&d->nF, &d->nJ}) {
      if (*q) cudaFree(*q);
      *q = nullptr;
    }
    d->n_cap = 0;
    if ((rc = dalloc(&d->nF, (size_t)(chunk * n * cd)))) return rc;
    if ((rc = dalloc(&d->nJ, (size_t)(chunk * n * n * cd)))) return rc;
    d->n_cap = chunk;
  }
  if (!smem && d->nM_cap < chunk) {  // global elimination matrices, sized separately
    cudaStreamSynchronize(st);
    if (d->nM) cudaFree(d->nM);
    d->nM = nullptr;
    d->nM_cap = 0;
    if ((rc = dalloc(&d->nM, (size_t)chunk * mat / sizeof(double)))) return rc;
    d->nM_cap = chunk;
  }
  // few points: 512 threads spread one elimination over the whole SM; batches: 128-256 per point
  const char* th_env = getenv("PHC_NEWTON_THREADS");  // A/B hook (CTA eliminations)
  const int threads = th_env ? std::max(64, std::min(512, atoi(th_env) / 32 * 32))  // the kernels' launch bounds
                             : (n_points < 148 ? 512 : (n <= 48 ? 128 : 256));
  for (int64_t p0 = 0; p0 < n_points; p0 += chunk) {
    const int64_t np = std::min(chunk, n_points - p0);
    if ((rc = run_on_device(s, d, np, x + p0 * n * cd, T ? T + p0 * L : nullptr, d->nF, d->nJ, st, n_points)))
      return rc;
    phc::NewtonArgs a;
    a.X = x + p0 * n * cd;
    a.F = d->nF;
    a.J = d->nJ;
    a.Xnew = x_new + p0 * n * cd;
    a.resid = residual + p0;
    a.status = status + p0;
    a.Mg = d->nM;
    a.n = n;
    a.n_points = np;
    ProfScope ps(s, d->dev, 2, st);
    // small systems: one warp per point (bitwise the same step as the CTA kernel)
    const size_t per_warp = (size_t)n * (n + 1) * cd * sizeof(double);
    const int warp_env = getenv("PHC_NEWTON_WARP") ? atoi(getenv("PHC_NEWTON_WARP")) : -1;  // A/B hook
    const bool warp_kernel = warp_env >= 0 ? (n <= 32 && warp_env == 1) : (n <= 32 && (n <= 16 || n_points < 4096));
    if (warp_kernel) {
      const int wpc = per_warp * 4 <= (size_t)160 * 1024 ? 4 : (per_warp * 2 <= (size_t)160 * 1024 ? 2 : 1);
      const size_t sm = per_warp * wpc;
      const unsigned grid = (unsigned)((np + wpc - 1) / wpc);
      if (L == 2) {
        if (sm > 48 * 1024) CUDA_TRY(phc::ensure_smem((const void*)phc::newton_warp_kernel<2>, sm));
        phc::newton_warp_kernel<2><<<grid, wpc * 32, sm, st>>>(a);
      } else {
        if (sm > 48 * 1024) CUDA_TRY(phc::ensure_smem((const void*)phc::newton_warp_kernel<4>, sm));
        phc::newton_warp_kernel<4><<<grid, wpc * 32, sm, st>>>(a);
      }
      CUDA_TRY(cudaGetLastError());
      continue;
    }
    // matrices beyond shared memory: one cooperative launch for few points (the points one
    // after another, each over all SMs), the multi-kernel path (all points at once) otherwise
    const int coop_env = getenv("PHC_NEWTON_COOP") ? atoi(getenv("PHC_NEWTON_COOP")) : -1;  // A/B hook
    const bool coop_ok = n <= 1 + phc::kCoopRows * phc::kCoopThreads && phc::coop_smem_bytes(n, L) <= (size_t)200 * 1024;
    const bool coop = coop_ok && (coop_env >= 0 ? coop_env == 1 : np <= kCoopMaxPoints);
    if (L == 2) {
      if (smem) {
        if (smat > 48 * 1024) CUDA_TRY(phc::ensure_smem((const void*)phc::newton_solve_kernel<2>, smat));
        phc::newton_solve_kernel<2><<<(unsigned)np, threads, smat, st>>>(a);
      } else if (coop) {
        if ((rc = newton_coop<2>(a, d, st))) return rc;
      } else {
        newton_multi<2>(a, np, st);
      }
    } else {
      if (smem) {
        if (smat > 48 * 1024) CUDA_TRY(phc::ensure_smem((const void*)phc::newton_solve_kernel<4>, smat));
        phc::newton_solve_kernel<4><<<(unsigned)np, threads, smat, st>>>(a);
      } else if (coop) {
        if ((rc = newton_coop<4>(a, d, st))) return rc;
      } else {
        newton_multi<4>(a, np, st);
      }
    }
    CUDA_TRY(cudaGetLastError());
  }
  return PHC_OK;
}

}  // namespace phc_rt

using namespace phc_rt;

extern "C" {

int phc_newton_step_batch(const phc_system* s, int64_t n_points, const double* x, double* x_new, double* residual,
                          int32_t* status, void* stream) {
  return newton_impl(s, n_points, x, nullptr, x_new, residual, status, stream);
}

int phc_newton_step_homotopy_batch(const phc_system* s, int64_t n_points, const double* x, const double* t,
                                   double* x_new, double* residual, int32_t* status, void* stream) {
  g_err.clear();
  if (!s) return fail(PHC_EINVAL, "NULL system");
  if (!s->has_target) return fail(PHC_EINVAL, "no target coefficients: call phc_system_set_target first");
  if (n_points > 0 && !t) return fail(PHC_EINVAL, "NULL t");
  return newton_impl(s, n_points, x, t, x_new, residual, status, stream);
}

int phc_newton_solve_batch(const phc_system* s, int64_t n_points, const double* x, const double* t, double tol,
                           int32_t max_it, double* x_out, double* residual, int32_t* iterations, int32_t* status,
                           void* stream) {
  g_err.clear();
  if (!s) return fail(PHC_EINVAL, "NULL system");
  if (!(tol >= 0.0) || max_it < 0) return fail(PHC_EINVAL, "tol >= 0 and max_it >= 0 required");
  if (t && !s->has_target) return fail(PHC_EINVAL, "no target coefficients: call phc_system_set_target first");
  if (s->n_eq != s->n_var) return fail(PHC_EINVAL, "Newton needs a square system (n_eq %d != n_var %d)", s->n_eq, s->n_var);
  if (n_points < 0) return fail(PHC_EINVAL, "n_points < 0");
  if (n_points == 0) return PHC_OK;
  if (!x || !x_out || !residual || !iterations || !status) return fail(PHC_EINVAL, "NULL pointer");
  if ((((uintptr_t)x) | ((uintptr_t)x_out)) & 31) return fail(PHC_EINVAL, "x/x_out must be 32-byte aligned");
  DeviceGuard g(s->home);
  cudaStream_t st = (cudaStream_t)stream;
  const int n = s->n_var, L = s->L;
  const int64_t cd = 2 * L, P = n_points;
  int rc;
  DevBuf<double> xw, res;
  DevBuf<int32_t> stt, active;
  if ((rc = dalloc(&xw.p, (size_t)(P * n * cd))) || (rc = dalloc(&res.p, (size_t)P)) ||
      (rc = dalloc(&stt.p, (size_t)P)) || (rc = dalloc(&active.p, (size_t)(2 * P))))
    return rc;
  CUDA_TRY(cudaMemcpyAsync(xw.p, x, (size_t)(P * n * cd) * sizeof(double), cudaMemcpyDeviceToDevice, st));
  auto grid = [](int64_t nth) { return (unsigned)((nth + 127) / 128); };
  phc::newton_solve_init_kernel<<<grid(P), 128, 0, st>>>(P, active.p, residual, iterations, status, tol, max_it);
  // x_out := x for points that never enter the loop (max_it = 0, or tol >= 1 = the initial
  // ||h||); the exit kernel overwrites the entries of every point that runs
  if (x_out != x)
    CUDA_TRY(cudaMemcpyAsync(x_out, x, (size_t)(P * n * cd) * sizeof(double), cudaMemcpyDeviceToDevice, st));
  CUDA_TRY(cudaGetLastError());
  if (!(1.0 > tol)) max_it = 0;  // the loop condition ||h|| > tol fails before the first iteration
  HostBuf<int32_t> act;
  if ((rc = act.alloc((size_t)P))) return rc;
  constexpr int kCheck = 4;  // iterations between host checks for an early end of the batch
  for (int k = 0; k < max_it; ++k) {
    if ((rc = newton_impl(s, P, xw.p, t, xw.p, res.p, stt.p, st))) return rc;
    if (L == 2)
      phc::newton_exit_kernel<2><<<grid(P * n), 128, 0, st>>>(n, P, k, max_it, tol, res.p, stt.p, xw.p,
                                                             active.p + (k & 1) * P, active.p + ((k + 1) & 1) * P,
                                                             x_out, residual, iterations, status);
    else
      phc::newton_exit_kernel<4><<<grid(P * n), 128, 0, st>>>(n, P, k, max_it, tol, res.p, stt.p, xw.p,
                                                             active.p + (k & 1) * P, active.p + ((k + 1) & 1) * P,
                                                             x_out, residual, iterations, status);
    CUDA_TRY(cudaGetLastError());
    if ((k + 1) % kCheck == 0 && k + 1 < max_it) {
      CUDA_TRY(cudaMemcpyAsync(act.p, active.p + ((k + 1) & 1) * P, (size_t)P * 4, cudaMemcpyDeviceToHost, st));
      CUDA_TRY(cudaStreamSynchronize(st));
      bool any = false;
      for (int64_t p = 0; p < P && !any; ++p) any = act[p] != 0;
      if (!any) break;
    }
  }
  CUDA_TRY(cudaStreamSynchronize(st));
  return PHC_OK;
}

}  // extern "C"
