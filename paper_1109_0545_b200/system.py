"""Object wrapper over the C ABI taking torch tensors (device memory) and torch streams."""
from __future__ import annotations

import ctypes

import numpy as np

from . import _lib


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data) if isinstance(a, np.ndarray) else ctypes.c_void_p(a.data_ptr())

def _stream_handle(stream, device):
    """cudaStream_t of `stream`, else of the current stream of `device` (the raw-pointer query
    when this torch build has it: a few microseconds cheaper per call than
    torch.cuda.current_stream(), which matters for single small evaluations)."""
    if stream is not None:
        return stream.cuda_stream
    idx = device.index if device.index is not None else 0
    if _RAW_STREAM is not None:
        return _RAW_STREAM(idx)
    import torch
    return torch.cuda.current_stream(device).cuda_stream


try:
    import torch as _torch
    _RAW_STREAM = getattr(_torch._C, "_cuda_getCurrentRawStream", None)
except Exception:  # torch without CUDA support: the handle-creating calls fail later anyway
    _RAW_STREAM = None



class System:
    """A system handle: ``System(arrays, device=0)`` with ``arrays`` having the attributes
    n_eq, n_var, limbs, poly_ptr, term_ptr, var_idx, exponent, coeff (include/phc.h layout)."""

    def __init__(self, arrays, device: int = 0, coeff_target=None, old_homotopy: bool = False):
        """``coeff_target`` [n_terms][2][L] attaches homotopy target coefficients (NEXT-3,
        phc_system_set_target).  ``old_homotopy=True`` instead builds the paper's "old"
        t-as-variable system (phc_homotopy_old_create): n_var + 1 variables, t last."""
        self.n_eq = int(arrays.n_eq)
        self.n_var = int(arrays.n_var)
        self.limbs = int(arrays.limbs)
        self.device = int(device)
        pp = np.ascontiguousarray(getattr(arrays, "poly_ptr", np.zeros(1)), dtype=np.int64)
        tp = np.ascontiguousarray(getattr(arrays, "term_ptr", getattr(arrays, "mono_ptr", None)), dtype=np.int64)
        vi = np.ascontiguousarray(arrays.var_idx, dtype=np.int32)
        ex = np.ascontiguousarray(arrays.exponent, dtype=np.int32)
        cf = np.ascontiguousarray(arrays.coeff, dtype=np.float64)
        self.n_terms = int(tp.shape[0] - 1)
        self._h = None
        self.homotopy = False
        self.common = False
        if hasattr(arrays, "mono_ptr"):
            # NEXT-2 common-support system: arrays.coeff is the dense [n_eq][n_mono][2][L] matrix
            mp = np.ascontiguousarray(arrays.mono_ptr, dtype=np.int64)
            self.n_terms = int(mp.shape[0] - 1)
            self._h = _lib.phc_system_create_common(self.n_eq, self.n_var, self.limbs, self.n_terms, _ptr(mp),
                                                    _ptr(vi), _ptr(ex), _ptr(cf), self.device)
            self.common = True
            if coeff_target is not None:
                self.set_target(coeff_target)
            return
        if old_homotopy:
            ct = np.ascontiguousarray(coeff_target, dtype=np.float64)
            self._h = _lib.phc_homotopy_old_create(self.n_eq, self.n_var, self.limbs, self.n_terms, _ptr(pp),
                                                   _ptr(tp), _ptr(vi), _ptr(ex), _ptr(cf), _ptr(ct), self.device)
            self.n_var += 1
            self.n_terms *= 3
            return
        self._h = _lib.phc_system_create(self.n_eq, self.n_var, self.limbs, self.n_terms, _ptr(pp), _ptr(tp),
                                         _ptr(vi), _ptr(ex), _ptr(cf), self.device)
        if coeff_target is not None:
            self.set_target(coeff_target)

    def set_target(self, coeff_target):
        ct = np.ascontiguousarray(coeff_target, dtype=np.float64)
        want = (self.n_eq, self.n_terms, 2, self.limbs) if self.common else (self.n_terms, 2, self.limbs)
        if ct.shape != want:
            raise ValueError(f"coeff_target must have shape {want}")
        _lib.phc_system_set_target(self._h, _ptr(ct))
        self.homotopy = True

    def close(self):
        if self._h is not None:
            _lib.phc_system_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def stats(self):
        keys = ("n_terms", "n_factors", "kmax", "D", "nnz_J", "cm_per_point", "ca_per_point", "launches",
                "exec_flops_per_point", "path", "layout", "K", "latency_exec_flops_per_point", "latency_bound",
                "common", "latency_kernel", "latency_G", "latency_launches")
        return dict(zip(keys, _lib.phc_system_stats(self._h)))

    def _check(self, t, shape):
        import torch

        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
            raise ValueError("expected a contiguous float64 CUDA tensor")
        if t.device.index != self.device:
            # the C ABI takes device pointers on the handle's home device; a pointer on another
            # GPU would fault inside the kernels (a sticky context error), so refuse it here
            raise ValueError(f"tensor on cuda:{t.device.index}, the system's home device is cuda:{self.device}")
        if tuple(t.shape) != tuple(shape):
            raise ValueError(f"expected shape {tuple(shape)}, got {tuple(t.shape)}")

    def eval(self, x, f=None, jac=None, stream=None):
        """x: [n_var, 2, L] float64 on the home device -> (f [n_eq,2,L], jac [n_eq,n_var,2,L])."""
        import torch

        L = self.limbs
        self._check(x, (self.n_var, 2, L))
        if f is None:
            f = torch.empty((self.n_eq, 2, L), dtype=torch.float64, device=x.device)
        if jac is None:
            jac = torch.empty((self.n_eq, self.n_var, 2, L), dtype=torch.float64, device=x.device)
        self._check(f, (self.n_eq, 2, L))
        self._check(jac, (self.n_eq, self.n_var, 2, L))
        st = _stream_handle(stream, x.device)
        _lib.phc_eval_jacobian(self._h, _ptr(x), _ptr(f), _ptr(jac), ctypes.c_void_p(st))
        return f, jac

    def eval_batch(self, X, F=None, J=None, devices=None, stream=None):
        """X: [P, n_var, 2, L] on the home device -> (F [P,n_eq,2,L], J [P,n_eq,n_var,2,L])."""
        import torch

        L = self.limbs
        P = int(X.shape[0])
        self._check(X, (P, self.n_var, 2, L))
        if F is None:
            F = torch.empty((P, self.n_eq, 2, L), dtype=torch.float64, device=X.device)
        if J is None:
            J = torch.empty((P, self.n_eq, self.n_var, 2, L), dtype=torch.float64, device=X.device)
        self._check(F, (P, self.n_eq, 2, L))
        self._check(J, (P, self.n_eq, self.n_var, 2, L))
        st = _stream_handle(stream, X.device)
        if devices:
            dv = (ctypes.c_int32 * len(devices))(*devices)
            nd = len(devices)
        else:
            dv, nd = None, 0
        _lib.phc_eval_jacobian_batch(self._h, P, _ptr(X), _ptr(F), _ptr(J), dv, nd, ctypes.c_void_p(st))
        return F, J

    def eval_batch_range(self, X, p_begin, p_end, F, J, stream=None):
        """Points [p_begin, p_end) of the len(X)-point batch call (phc_eval_jacobian_batch_range):
        X [P, n_var, 2, L] on the home device (only those rows are read); F [P, n_eq, 2, L] and
        J [P, n_eq, n_var, 2, L] receive those rows, bitwise what eval_batch writes for all P.
        F and J are tensors on the home device or raw device pointers (int) to such arrays,
        e.g. another process's buffers mapped with phc_ipc_open (the gather fused into the
        kernels' stores)."""
        L = self.limbs
        P = int(X.shape[0])
        self._check(X, (P, self.n_var, 2, L))
        ptrs = []
        for a, shape in ((F, (P, self.n_eq, 2, L)), (J, (P, self.n_eq, self.n_var, 2, L))):
            if isinstance(a, int):
                ptrs.append(ctypes.c_void_p(a))
            else:
                self._check(a, shape)
                ptrs.append(_ptr(a))
        st = _stream_handle(stream, X.device)
        _lib.phc_eval_jacobian_batch_range(self._h, P, int(p_begin), int(p_end), _ptr(X), ptrs[0], ptrs[1],
                                           ctypes.c_void_p(st))

    def newton_step(self, X, X_new=None, stream=None):
        """One Newton iteration per point (NEXT-1): X [P, n, 2, L] on the home device ->
        (X_new, residual [P] float64, status [P] int32).  X_new may be X (in place)."""
        import torch

        L = self.limbs
        P = int(X.shape[0])
        self._check(X, (P, self.n_var, 2, L))
        if X_new is None:
            X_new = torch.empty_like(X)
        self._check(X_new, (P, self.n_var, 2, L))
        res = torch.empty(P, dtype=torch.float64, device=X.device)
        status = torch.empty(P, dtype=torch.int32, device=X.device)
        st = _stream_handle(stream, X.device)
        _lib.phc_newton_step_batch(self._h, P, _ptr(X), _ptr(X_new), _ptr(res), _ptr(status), ctypes.c_void_p(st))
        return X_new, res, status

    def newton_solve(self, X, tol, max_it, T=None, X_out=None, stream=None):
        """Alg. 2 to tolerance per point (phc_newton_solve_batch): X [P, n, 2, L] (and T [P, L]
        for the homotopy h(., t)) on the home device -> (X_out, residual [P] float64,
        iterations [P] int32, status [P] int32: 0 converged, 1 failed, 2 singular)."""
        import torch

        L = self.limbs
        P = int(X.shape[0])
        self._check(X, (P, self.n_var, 2, L))
        if T is not None:
            self._check(T, (P, L))
        if X_out is None:
            X_out = torch.empty_like(X)
        self._check(X_out, (P, self.n_var, 2, L))
        res = torch.empty(P, dtype=torch.float64, device=X.device)
        its = torch.empty(P, dtype=torch.int32, device=X.device)
        status = torch.empty(P, dtype=torch.int32, device=X.device)
        st = _stream_handle(stream, X.device)
        _lib.phc_newton_solve_batch(self._h, P, _ptr(X), _ptr(T) if T is not None else None, float(tol), int(max_it),
                                    _ptr(X_out), _ptr(res), _ptr(its), _ptr(status), ctypes.c_void_p(st))
        return X_out, res, its, status

    def eval_homotopy_batch(self, X, T, F=None, J=None, devices=None, stream=None):
        """h(., t_p) at X [P, n_var, 2, L] with T [P, L] (real t limbs), both on the home
        device -> (F, J) as eval_batch (NEXT-3)."""
        import torch

        L = self.limbs
        P = int(X.shape[0])
        self._check(X, (P, self.n_var, 2, L))
        self._check(T, (P, L))
        if F is None:
            F = torch.empty((P, self.n_eq, 2, L), dtype=torch.float64, device=X.device)
        if J is None:
            J = torch.empty((P, self.n_eq, self.n_var, 2, L), dtype=torch.float64, device=X.device)
        self._check(F, (P, self.n_eq, 2, L))
        self._check(J, (P, self.n_eq, self.n_var, 2, L))
        st = _stream_handle(stream, X.device)
        if devices:
            dv = (ctypes.c_int32 * len(devices))(*devices)
            nd = len(devices)
        else:
            dv, nd = None, 0
        _lib.phc_eval_homotopy_batch(self._h, P, _ptr(X), _ptr(T), _ptr(F), _ptr(J), dv, nd, ctypes.c_void_p(st))
        return F, J

    def newton_step_homotopy(self, X, T, X_new=None, stream=None):
        """One Newton iteration on h(., t_p) = 0 per point: X [P, n, 2, L], T [P, L]."""
        import torch

        L = self.limbs
        P = int(X.shape[0])
        self._check(X, (P, self.n_var, 2, L))
        self._check(T, (P, L))
        if X_new is None:
            X_new = torch.empty_like(X)
        self._check(X_new, (P, self.n_var, 2, L))
        res = torch.empty(P, dtype=torch.float64, device=X.device)
        status = torch.empty(P, dtype=torch.int32, device=X.device)
        st = _stream_handle(stream, X.device)
        _lib.phc_newton_step_homotopy_batch(self._h, P, _ptr(X), _ptr(T), _ptr(X_new), _ptr(res), _ptr(status),
                                            ctypes.c_void_p(st))
        return X_new, res, status

    def track(self, X, stream=None, t_end=False, **params):
        """Track the paths starting at X [P, n, 2, L] (solutions of h(., 0) = 0, on the home
        device) to t = 1 (NEXT-4, phc_track_paths).  ``params`` override the phc_track_params
        defaults (reading T1).  Returns (X_end, status [P] numpy int32: 1 arrived,
        2 failed, stats [P, 5] numpy: accepted, corrector calls, Newton iterations, min step,
        mean step[, T_end [P, L]])."""
        import torch

        L = self.limbs
        P = int(X.shape[0])
        self._check(X, (P, self.n_var, 2, L))
        prm = default_track_params(L)
        for k, v in params.items():
            setattr(prm, k, v)
        Xe = X.clone()
        status = np.zeros(P, dtype=np.int32)
        stats = np.zeros((P, 5))
        te = torch.empty((P, L), dtype=torch.float64, device=X.device) if t_end else None
        st = _stream_handle(stream, X.device)
        _lib.phc_track_paths(self._h, P, _ptr(Xe), prm, _ptr(status), _ptr(stats),
                             _ptr(te) if te is not None else None, ctypes.c_void_p(st))
        return (Xe, status, stats, te) if t_end else (Xe, status, stats)

    def eval_batch_host(self, X, F=None, J=None, devices=None):
        """Host arrays (numpy or pinned CPU tensors) in and out; synchronous."""
        L = self.limbs
        P = int(X.shape[0])
        if F is None:
            F = np.empty((P, self.n_eq, 2, L))
        if J is None:
            J = np.empty((P, self.n_eq, self.n_var, 2, L))
        for a, shape in ((X, (P, self.n_var, 2, L)), (F, (P, self.n_eq, 2, L)), (J, (P, self.n_eq, self.n_var, 2, L))):
            if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous):
                raise ValueError("expected C-contiguous float64 numpy arrays (host memory)")
            if a.shape != shape:
                raise ValueError(f"expected shape {shape}, got {a.shape}")
        if devices:
            dv = (ctypes.c_int32 * len(devices))(*devices)
            nd = len(devices)
        else:
            dv, nd = None, 0
        _lib.phc_eval_jacobian_batch_host(self._h, P, _ptr(X), _ptr(F), _ptr(J), dv, nd)
        return F, J


def default_track_params(limbs):
    """Tracker defaults (reading T1; SPEC tracker/corrector decisions): lambda_0 = 0.01,
    contraction 0.5, expansion 2 after every success, lambda_max = 0.1, lambda_min = 1e-8
    (DD) / 1e-12 (QD), corrector tolerance 1e-24 (DD) / 1e-48 (QD) with Max_It = 4, 4 end
    iterations at t = 1, quadratic predictor."""
    return _lib.TrackParams(step_init=0.01, step_min=1e-8 if limbs == 2 else 1e-12, step_max=0.1, expand=2.0,
                            contract=0.5, tol=1e-24 if limbs == 2 else 1e-48, max_newton=4, max_steps=100000,
                            end_newton=4, predictor=2)


def predict_batch(order, n_hist, t_hist, x_hist, t_new, out=None, stream=None):
    """phc_predict_batch on torch tensors: n_hist [P] int32, t_hist [P, 3, L], x_hist [P, 3, n, 2, L],
    t_new [P, L] (all on one device) -> x_out [P, n, 2, L]."""
    import torch

    P, _, n, _, L = x_hist.shape
    if out is None:
        out = torch.empty((P, n, 2, L), dtype=torch.float64, device=x_hist.device)
    st = _stream_handle(stream, x_hist.device)
    _lib.phc_predict_batch(L, n, P, order, _ptr(n_hist), _ptr(t_hist), _ptr(x_hist), _ptr(t_new), _ptr(out),
                           ctypes.c_void_p(st))
    return out
