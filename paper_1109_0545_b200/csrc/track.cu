// NEXT-4 host side: the predictor entry point and the batched path tracker (Alg. 1,
// P:191-238; the quadratic predictor of §5), driving the kernels of
// kernels_track.cuh and the Newton corrector (newton.cu).
#include "runtime.h"
#include "kernels_track.cuh"

using namespace phc_rt;

namespace {
// the tracker's private stream, its ordering event and the window graph
struct TrackStream {
  cudaStream_t s = nullptr;
  cudaEvent_t e = nullptr;
  cudaGraphExec_t ex = nullptr;
  ~TrackStream() {
    if (s) cudaStreamSynchronize(s);
    if (ex) cudaGraphExecDestroy(ex);
    if (e) cudaEventDestroy(e);
    if (s) cudaStreamDestroy(s);
  }
};
}  // namespace

extern "C" {

int phc_predict_batch(int32_t limbs, int32_t n_var, int64_t n_paths, int32_t order, const int32_t* n_hist,
                      const double* t_hist, const double* x_hist, const double* t_new, double* x_out, void* stream) {
  g_err.clear();
  if (limbs != 2 && limbs != 4) return fail(PHC_EUNSUPPORTED, "limbs must be 2 or 4");
  if (n_var < 1 || n_paths < 0) return fail(PHC_EINVAL, "n_var >= 1 and n_paths >= 0 required");
  if (order < 0 || order > 2) return fail(PHC_EINVAL, "order must be 0, 1 or 2");
  if (n_paths == 0) return PHC_OK;
  if (!n_hist || !t_hist || !x_hist || !t_new || !x_out) return fail(PHC_EINVAL, "NULL pointer");
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t nth = n_paths * n_var;
  const unsigned grid = (unsigned)((nth + 127) / 128);
  if (limbs == 2)
    phc::predict_kernel<2><<<grid, 128, 0, st>>>(n_var, n_paths, nullptr, n_hist, t_hist, x_hist, nullptr, t_new, order,
                                                 nullptr, x_out, nullptr);
  else
    phc::predict_kernel<4><<<grid, 128, 0, st>>>(n_var, n_paths, nullptr, n_hist, t_hist, x_hist, nullptr, t_new, order,
                                                 nullptr, x_out, nullptr);
  CUDA_TRY(cudaGetLastError());
  return PHC_OK;
}

int phc_track_paths(const phc_system* cs, int64_t n_paths, double* x, const phc_track_params* prm, int32_t* status,
                    double* path_stats, double* t_end, void* stream) {
  g_err.clear();
  phc_system* s = const_cast<phc_system*>(cs);
  if (!s || !prm) return fail(PHC_EINVAL, "NULL argument");
  if (!s->has_target) return fail(PHC_EINVAL, "no target coefficients: call phc_system_set_target first");
  if (s->n_eq != s->n_var) return fail(PHC_EINVAL, "tracking needs a square system");
  if (n_paths < 0) return fail(PHC_EINVAL, "n_paths < 0");
  if (n_paths == 0) return PHC_OK;
  if (!x || !status) return fail(PHC_EINVAL, "NULL x/status");
  const phc_track_params& q = *prm;
  if (!(q.step_min > 0 && q.step_min <= q.step_init && q.step_init <= q.step_max && q.step_max <= 1.0) ||
      !(q.contract > 0 && q.contract < 1 && q.expand >= 1) || !(q.tol > 0) || q.max_newton < 1 || q.max_steps < 1 ||
      q.end_newton < 0 || q.predictor < 0 || q.predictor > 2)
    return fail(PHC_EINVAL, "invalid tracker parameters");
  DeviceGuard g(s->home);
  // the tracker runs on a private stream ordered after the caller's (`stream` may be the
  // legacy default stream, which cannot be captured into a graph); it is synchronous
  TrackStream ts_guard;
  {
    cudaStream_t user = (cudaStream_t)stream;
    CUDA_TRY(cudaStreamCreateWithFlags(&ts_guard.s, cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(&ts_guard.e, cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(ts_guard.e, user));
    CUDA_TRY(cudaStreamWaitEvent(ts_guard.s, ts_guard.e, 0));
  }
  cudaStream_t st = ts_guard.s;
  const int n = s->n_var, L = s->L;
  const int64_t cd = 2 * L, P = n_paths;
  int rc;
  DevBuf<double> t_hist, x_hist, lam_d, tc, xc, res_d, minst_d, sumst_d;
  DevBuf<int32_t> n_hist, idx_d, clip_d, acc_d, nst_d, stat_d;
  DevBuf<int64_t> steps_d, succ_d, iters_d;
  if ((rc = dalloc(&t_hist.p, (size_t)(P * 3 * L))) || (rc = dalloc(&x_hist.p, (size_t)(P * 3 * n * cd))) ||
      (rc = dalloc(&lam_d.p, (size_t)P)) || (rc = dalloc(&tc.p, (size_t)(P * L))) ||
      (rc = dalloc(&xc.p, (size_t)(P * n * cd))) || (rc = dalloc(&res_d.p, (size_t)P * q.max_newton)) ||
      (rc = dalloc(&minst_d.p, (size_t)P)) || (rc = dalloc(&sumst_d.p, (size_t)P)) ||
      (rc = dalloc(&n_hist.p, (size_t)P)) || (rc = dalloc(&idx_d.p, (size_t)P)) || (rc = dalloc(&clip_d.p, (size_t)P)) ||
      (rc = dalloc(&acc_d.p, (size_t)P)) || (rc = dalloc(&nst_d.p, (size_t)P * q.max_newton)) ||
      (rc = dalloc(&stat_d.p, (size_t)P)) || (rc = dalloc(&steps_d.p, (size_t)P)) || (rc = dalloc(&succ_d.p, (size_t)P)) ||
      (rc = dalloc(&iters_d.p, (size_t)P)))
    return rc;
  auto grid = [](int64_t nth) { return (unsigned)((nth + 127) / 128); };
  if (L == 2)
    phc::track_init_kernel<2><<<grid(P * n), 128, 0, st>>>(n, P, x, n_hist.p, t_hist.p, x_hist.p);
  else
    phc::track_init_kernel<4><<<grid(P * n), 128, 0, st>>>(n, P, x, n_hist.p, t_hist.p, x_hist.p);
  CUDA_TRY(cudaGetLastError());
  // Per-path control state (Alg. 1 step_size_control / stop_criterion) lives on the device
  // and is updated by control_kernel after every step, so W steps are enqueued back to back
  // with no host synchronisation; the host reads the statuses once per window and re-compacts
  // the active paths.  A path that stops inside a window is skipped by the control kernel
  // for the rest of it (its predictor/corrector work there is wasted, not used), so the
  // window changes no decision: the result is that of a host check after every step.
  HostBuf<double> lam, minst;
  HostBuf<int32_t> idx, stat;
  if ((rc = lam.alloc(P)) || (rc = minst.alloc(P)) || (rc = idx.alloc(P)) || (rc = stat.alloc(P))) return rc;
  for (int64_t p = 0; p < P; ++p) {
    lam[p] = q.step_init;
    minst[p] = 1e300;
    stat[p] = 0;
  }
  CUDA_TRY(cudaMemcpyAsync(lam_d.p, lam.p, P * 8, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemcpyAsync(minst_d.p, minst.p, P * 8, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaMemsetAsync(sumst_d.p, 0, P * 8, st));
  CUDA_TRY(cudaMemsetAsync(stat_d.p, 0, P * 4, st));
  CUDA_TRY(cudaMemsetAsync(steps_d.p, 0, P * 8, st));
  CUDA_TRY(cudaMemsetAsync(succ_d.p, 0, P * 8, st));
  CUDA_TRY(cudaMemsetAsync(iters_d.p, 0, P * 8, st));
  const phc::TrackCtl ctl{q.step_min, q.step_max, q.expand, q.contract, q.tol, q.max_newton, q.max_steps};
  const char* wenv = getenv("PHC_TRACK_WINDOW");
  const int window = wenv ? std::max(1, atoi(wenv)) : 8;
  // W tracker steps over the A active paths of idx_d
  auto enqueue_window = [&](int64_t A) -> int {
    for (int w = 0; w < window; ++w) {
      // predict: t_try = min(t + lambda, 1), z_guess by the secant / quadratic predictor (§5)
      if (L == 2)
        phc::predict_kernel<2><<<grid(A * n), 128, 0, st>>>(n, A, idx_d.p, n_hist.p, t_hist.p, x_hist.p, lam_d.p,
                                                             nullptr, q.predictor, tc.p, xc.p, clip_d.p);
      else
        phc::predict_kernel<4><<<grid(A * n), 128, 0, st>>>(n, A, idx_d.p, n_hist.p, t_hist.p, x_hist.p, lam_d.p,
                                                             nullptr, q.predictor, tc.p, xc.p, clip_d.p);
      CUDA_TRY(cudaGetLastError());
      // correct: Alg. 2 on h(., t_try).  All max_newton iterations are enqueued back to back;
      // iteration k records its residual and status in row k.  A path is corrected at the
      // first iteration whose residual passes tol (Alg. 2 applies that iteration's update
      // too); the iterations after it only refine the point further (documented deviation,
      // DESIGN.md reading T1).
      for (int k = 0; k < q.max_newton; ++k)
        if ((rc = newton_impl(s, A, xc.p, tc.p, xc.p, res_d.p + (size_t)k * A, nst_d.p + (size_t)k * A, st)))
          return rc;
      // step-size control, step back, stop criterion (Alg. 1), then the history shift of the
      // accepted steps
      phc::control_kernel<<<grid(A), 128, 0, st>>>(A, idx_d.p, ctl, res_d.p, nst_d.p, clip_d.p, acc_d.p, stat_d.p,
                                                   lam_d.p, steps_d.p, succ_d.p, iters_d.p, minst_d.p, sumst_d.p);
      if (L == 2)
        phc::accept_kernel<2><<<grid(A * n), 128, 0, st>>>(n, A, idx_d.p, acc_d.p, tc.p, xc.p, n_hist.p, t_hist.p,
                                                            x_hist.p);
      else
        phc::accept_kernel<4><<<grid(A * n), 128, 0, st>>>(n, A, idx_d.p, acc_d.p, tc.p, xc.p, n_hist.p, t_hist.p,
                                                            x_hist.p);
      CUDA_TRY(cudaGetLastError());
    }
    return PHC_OK;
  };
  // After a first window of plain launches (it also sizes every workspace), a window is one
  // CUDA graph launch: captured once per active-path count A (cudaGraphExecUpdate when the
  // topology allows), so a window of ~11 W kernels costs one launch on the host.  The
  // few-path tracker is launch-bound without it.  PHC_TRACK_GRAPH=0 disables the graphs.
  bool use_graph = !(getenv("PHC_TRACK_GRAPH") && atoi(getenv("PHC_TRACK_GRAPH")) == 0);
  bool warmed = false;
  int64_t graph_A = -1;
  while (true) {
    int64_t A = 0;
    for (int64_t p = 0; p < P; ++p)
      if (stat[p] == 0) idx[A++] = (int32_t)p;
    if (A == 0) break;
    CUDA_TRY(cudaMemcpyAsync(idx_d.p, idx.p, A * 4, cudaMemcpyHostToDevice, st));
    if (use_graph && warmed && A != graph_A) {
      cudaGraph_t gr = nullptr;
      CUDA_TRY(cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed));
      const int rc_cap = enqueue_window(A);
      const cudaError_t ce = cudaStreamEndCapture(st, &gr);
      if (rc_cap != PHC_OK || ce != cudaSuccess || gr == nullptr) {
        if (gr) cudaGraphDestroy(gr);
        cudaGetLastError();
        g_err.clear();
        use_graph = false;  // not capturable here: plain launches from now on
      } else {
        bool ok = false;
        if (ts_guard.ex) {
          cudaGraphExecUpdateResultInfo info;
          ok = cudaGraphExecUpdate(ts_guard.ex, gr, &info) == cudaSuccess;
          if (!ok) {
            cudaGetLastError();
            cudaGraphExecDestroy(ts_guard.ex);
            ts_guard.ex = nullptr;
          }
        }
        if (!ok) {
          const cudaError_t ie = cudaGraphInstantiate(&ts_guard.ex, gr, 0);
          if (ie != cudaSuccess) {
            cudaGetLastError();
            ts_guard.ex = nullptr;
            use_graph = false;
          }
        }
        cudaGraphDestroy(gr);
        graph_A = use_graph ? A : -1;
      }
    }
    if (use_graph && warmed && graph_A == A) {
      CUDA_TRY(cudaGraphLaunch(ts_guard.ex, st));
    } else {
      if ((rc = enqueue_window(A))) return rc;
      warmed = true;
    }
    CUDA_TRY(cudaMemcpyAsync(stat.p, stat_d.p, P * 4, cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
  }
  std::vector<int32_t> stat_v(stat.p, stat.p + P);
  if (L == 2)
    phc::track_finish_kernel<2><<<grid(P * n), 128, 0, st>>>(n, P, t_hist.p, x_hist.p, x, t_end);
  else
    phc::track_finish_kernel<4><<<grid(P * n), 128, 0, st>>>(n, P, t_hist.p, x_hist.p, x, t_end);
  CUDA_TRY(cudaGetLastError());
  // end refinement at t = 1 of the paths that arrived (Newton on the target system)
  int64_t A = 0;
  for (int64_t p = 0; p < P; ++p)
    if (stat_v[p] == 1) idx[A++] = (int32_t)p;
  if (q.end_newton > 0 && A > 0) {
    CUDA_TRY(cudaMemcpyAsync(idx_d.p, idx.p, A * 4, cudaMemcpyHostToDevice, st));
    std::vector<double> ones((size_t)A * L, 0.0);
    for (int64_t a = 0; a < A; ++a) ones[(size_t)a * L] = 1.0;
    CUDA_TRY(cudaMemcpyAsync(tc.p, ones.data(), A * L * 8, cudaMemcpyHostToDevice, st));
    phc::gather_rows_kernel<<<grid(A * n * cd), 128, 0, st>>>(A, n * cd, idx_d.p, x, xc.p);
    for (int k = 0; k < q.end_newton; ++k)
      if ((rc = newton_impl(s, A, xc.p, tc.p, xc.p, res_d.p, nst_d.p, st))) return rc;
    phc::scatter_rows_kernel<<<grid(A * n * cd), 128, 0, st>>>(A, n * cd, idx_d.p, xc.p, x);
    CUDA_TRY(cudaGetLastError());
  }
  std::vector<int64_t> steps((size_t)P), succ((size_t)P), iters((size_t)P);
  std::vector<double> min_step((size_t)P), sum_step((size_t)P);
  CUDA_TRY(cudaMemcpyAsync(steps.data(), steps_d.p, P * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(succ.data(), succ_d.p, P * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(iters.data(), iters_d.p, P * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(min_step.data(), minst_d.p, P * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaMemcpyAsync(sum_step.data(), sumst_d.p, P * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  for (int64_t p = 0; p < P; ++p) {
    status[p] = stat_v[p];
    if (path_stats) {
      path_stats[p * 5 + 0] = (double)succ[p];
      path_stats[p * 5 + 1] = (double)steps[p];
      path_stats[p * 5 + 2] = (double)iters[p];
      path_stats[p * 5 + 3] = succ[p] ? min_step[p] : 0.0;
      path_stats[p * 5 + 4] = succ[p] ? sum_step[p] / succ[p] : 0.0;
    }
  }
  return PHC_OK;
}

}  // extern "C"
