"""ctypes binding of the C ABI declared in include/phc.h (argument marshalling only).

Every function here has the C name; every step of the evaluation runs in the CUDA
kernels of libphc.so.  There is no fallback: if the shared library is missing the
import fails loudly.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PHC_LIB") or os.path.join(_HERE, "libphc.so")

PHC_OK = 0
PHC_EINVAL = -1
PHC_ENOMEM = -2
PHC_ECUDA = -3
PHC_EUNSUPPORTED = -4
PHC_MAX_K = 64
PHC_MAX_EXP = 255

EXPORTED = (
    "phc_system_create",
    "phc_system_destroy",
    "phc_eval_jacobian",
    "phc_eval_jacobian_batch",
    "phc_eval_jacobian_batch_host",
    "phc_eval_jacobian_batch_range",
    "phc_ipc_get_handle",
    "phc_ipc_open",
    "phc_ipc_close",
    "phc_newton_step_batch",
    "phc_system_set_target",
    "phc_system_create_common",
    "phc_predict_batch",
    "phc_arith_test",
    "phc_track_paths",
    "phc_eval_homotopy_batch",
    "phc_newton_step_homotopy_batch",
    "phc_newton_solve_batch",
    "phc_homotopy_old_create",
    "phc_system_stats",
    "phc_fp64_peak",
    "phc_profile_enable",
    "phc_profile_read",
    "phc_last_error",
    "phc_version",
)


class TrackParams(ctypes.Structure):
    """phc_track_params (include/phc.h); defaults: DESIGN.md reading T1."""
    _fields_ = [("step_init", ctypes.c_double), ("step_min", ctypes.c_double), ("step_max", ctypes.c_double),
                ("expand", ctypes.c_double), ("contract", ctypes.c_double), ("tol", ctypes.c_double),
                ("max_newton", ctypes.c_int32), ("max_steps", ctypes.c_int32), ("end_newton", ctypes.c_int32),
                ("predictor", ctypes.c_int32)]


class PhcError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"phc error {code}: {msg}")
        self.code = code


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the CUDA extension is required; there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.c_void_p
    i32, i64 = ctypes.c_int32, ctypes.c_int64
    lib.phc_system_create.argtypes = [ctypes.POINTER(P), i32, i32, i32, i64, P, P, P, P, P, i32]
    lib.phc_system_create.restype = ctypes.c_int
    lib.phc_system_destroy.argtypes = [P]
    lib.phc_system_destroy.restype = None
    lib.phc_eval_jacobian.argtypes = [P, P, P, P, P]
    lib.phc_eval_jacobian.restype = ctypes.c_int
    lib.phc_eval_jacobian_batch.argtypes = [P, i64, P, P, P, P, i32, P]
    lib.phc_eval_jacobian_batch.restype = ctypes.c_int
    lib.phc_eval_jacobian_batch_host.argtypes = [P, i64, P, P, P, P, i32]
    lib.phc_eval_jacobian_batch_host.restype = ctypes.c_int
    lib.phc_eval_jacobian_batch_range.argtypes = [P, i64, i64, i64, P, P, P, P]
    lib.phc_eval_jacobian_batch_range.restype = ctypes.c_int
    lib.phc_ipc_get_handle.argtypes = [P, P, ctypes.POINTER(i64)]
    lib.phc_ipc_get_handle.restype = ctypes.c_int
    lib.phc_ipc_open.argtypes = [P, i32, ctypes.POINTER(P)]
    lib.phc_ipc_open.restype = ctypes.c_int
    lib.phc_ipc_close.argtypes = [P, i32]
    lib.phc_ipc_close.restype = ctypes.c_int
    lib.phc_newton_step_batch.argtypes = [P, i64, P, P, P, P, P]
    lib.phc_newton_step_batch.restype = ctypes.c_int
    lib.phc_system_create_common.argtypes = [ctypes.POINTER(P), i32, i32, i32, i64, P, P, P, P, i32]
    lib.phc_system_create_common.restype = ctypes.c_int
    lib.phc_arith_test.argtypes = [i32, i32, i64, P, P, P, P]
    lib.phc_arith_test.restype = ctypes.c_int
    lib.phc_predict_batch.argtypes = [i32, i32, i64, i32, P, P, P, P, P, P]
    lib.phc_predict_batch.restype = ctypes.c_int
    lib.phc_track_paths.argtypes = [P, i64, P, ctypes.POINTER(TrackParams), P, P, P, P]
    lib.phc_track_paths.restype = ctypes.c_int
    lib.phc_system_set_target.argtypes = [P, P]
    lib.phc_system_set_target.restype = ctypes.c_int
    lib.phc_eval_homotopy_batch.argtypes = [P, i64, P, P, P, P, P, i32, P]
    lib.phc_eval_homotopy_batch.restype = ctypes.c_int
    lib.phc_newton_step_homotopy_batch.argtypes = [P, i64, P, P, P, P, P, P]
    lib.phc_newton_step_homotopy_batch.restype = ctypes.c_int
    lib.phc_newton_solve_batch.argtypes = [P, i64, P, P, ctypes.c_double, i32, P, P, P, P, P]
    lib.phc_newton_solve_batch.restype = ctypes.c_int
    lib.phc_homotopy_old_create.argtypes = [ctypes.POINTER(P), i32, i32, i32, i64, P, P, P, P, P, P, i32]
    lib.phc_homotopy_old_create.restype = ctypes.c_int
    lib.phc_system_stats.argtypes = [P, P]
    lib.phc_system_stats.restype = ctypes.c_int
    lib.phc_fp64_peak.argtypes = [i32, ctypes.c_double, ctypes.POINTER(ctypes.c_double)]
    lib.phc_fp64_peak.restype = ctypes.c_int
    lib.phc_profile_enable.argtypes = [P, ctypes.c_int]
    lib.phc_profile_enable.restype = ctypes.c_int
    lib.phc_profile_read.argtypes = [P, P, P, ctypes.c_int]
    lib.phc_profile_read.restype = ctypes.c_int
    lib.phc_last_error.argtypes = []
    lib.phc_last_error.restype = ctypes.c_char_p
    lib.phc_version.argtypes = []
    lib.phc_version.restype = ctypes.c_char_p
    return lib


lib = _load()


def check(rc):
    if rc != PHC_OK:
        raise PhcError(rc, lib.phc_last_error().decode())
    return rc


# --- thin same-name wrappers (raw pointers / ints) -------------------------------------------

def phc_system_create(n_eq, n_var, limbs, n_terms, poly_ptr, term_ptr, var_idx, exponent, coeff, device):
    h = ctypes.c_void_p()
    check(lib.phc_system_create(ctypes.byref(h), n_eq, n_var, limbs, n_terms, poly_ptr, term_ptr, var_idx,
                                exponent, coeff, device))
    return h


def phc_system_destroy(h):
    lib.phc_system_destroy(h)


def phc_eval_jacobian(h, x, f, jac, stream):
    return check(lib.phc_eval_jacobian(h, x, f, jac, stream))


def phc_eval_jacobian_batch(h, n_points, x, f, jac, devices, n_devices, stream):
    return check(lib.phc_eval_jacobian_batch(h, n_points, x, f, jac, devices, n_devices, stream))


def phc_eval_jacobian_batch_host(h, n_points, x, f, jac, devices, n_devices):
    return check(lib.phc_eval_jacobian_batch_host(h, n_points, x, f, jac, devices, n_devices))


def phc_eval_jacobian_batch_range(h, n_points, p_begin, p_end, x, f, jac, stream):
    return check(lib.phc_eval_jacobian_batch_range(h, n_points, p_begin, p_end, x, f, jac, stream))


PHC_IPC_HANDLE_BYTES = 64


def phc_ipc_get_handle(dev_ptr):
    """-> (handle bytes, offset of dev_ptr inside its allocation)"""
    buf = ctypes.create_string_buffer(PHC_IPC_HANDLE_BYTES)
    off = ctypes.c_int64()
    check(lib.phc_ipc_get_handle(dev_ptr, buf, ctypes.byref(off)))
    return buf.raw, off.value


def phc_ipc_open(handle, device):
    """-> base device pointer (int) of the exported allocation, mapped on `device`"""
    if len(handle) != PHC_IPC_HANDLE_BYTES:
        raise ValueError(f"IPC handle must be {PHC_IPC_HANDLE_BYTES} bytes")
    base = ctypes.c_void_p()
    check(lib.phc_ipc_open(ctypes.create_string_buffer(bytes(handle), PHC_IPC_HANDLE_BYTES), device,
                           ctypes.byref(base)))
    return base.value


def phc_ipc_close(base, device):
    return check(lib.phc_ipc_close(base, device))


def phc_newton_step_batch(h, n_points, x, x_new, residual, status, stream):
    return check(lib.phc_newton_step_batch(h, n_points, x, x_new, residual, status, stream))


def phc_system_create_common(n_eq, n_var, limbs, n_mono, mono_ptr, var_idx, exponent, coeff, device):
    h = ctypes.c_void_p()
    check(lib.phc_system_create_common(ctypes.byref(h), n_eq, n_var, limbs, n_mono, mono_ptr, var_idx, exponent,
                                       coeff, device))
    return h


def phc_arith_test(op, limbs, n, a, b, out, stream):
    return check(lib.phc_arith_test(op, limbs, n, a, b, out, stream))


def phc_predict_batch(limbs, n_var, n_paths, order, n_hist, t_hist, x_hist, t_new, x_out, stream):
    return check(lib.phc_predict_batch(limbs, n_var, n_paths, order, n_hist, t_hist, x_hist, t_new, x_out, stream))


def phc_track_paths(h, n_paths, x, params, status, path_stats, t_end, stream):
    return check(lib.phc_track_paths(h, n_paths, x, ctypes.byref(params), status, path_stats, t_end, stream))


def phc_system_set_target(h, coeff_target):
    return check(lib.phc_system_set_target(h, coeff_target))


def phc_eval_homotopy_batch(h, n_points, x, t, f, jac, devices, n_devices, stream):
    return check(lib.phc_eval_homotopy_batch(h, n_points, x, t, f, jac, devices, n_devices, stream))


def phc_newton_step_homotopy_batch(h, n_points, x, t, x_new, residual, status, stream):
    return check(lib.phc_newton_step_homotopy_batch(h, n_points, x, t, x_new, residual, status, stream))


def phc_newton_solve_batch(h, n_points, x, t, tol, max_it, x_out, residual, iterations, status, stream):
    return check(lib.phc_newton_solve_batch(h, n_points, x, t, tol, max_it, x_out, residual, iterations, status, stream))


def phc_homotopy_old_create(n_eq, n_var, limbs, n_terms, poly_ptr, term_ptr, var_idx, exponent, coeff_start,
                            coeff_target, device):
    h = ctypes.c_void_p()
    check(lib.phc_homotopy_old_create(ctypes.byref(h), n_eq, n_var, limbs, n_terms, poly_ptr, term_ptr, var_idx,
                                      exponent, coeff_start, coeff_target, device))
    return h


def phc_system_stats(h):
    out = (ctypes.c_int64 * 18)()
    check(lib.phc_system_stats(h, out))
    return list(out)


def phc_fp64_peak(device=0, ms_target=200.0):
    v = ctypes.c_double()
    check(lib.phc_fp64_peak(device, ms_target, ctypes.byref(v)))
    return v.value


def phc_profile_enable(h, enable=True):
    return check(lib.phc_profile_enable(h, 1 if enable else 0))


def phc_profile_read(h, reset=True):
    ms = (ctypes.c_double * 4)()
    n = (ctypes.c_int64 * 4)()
    check(lib.phc_profile_read(h, ms, n, 1 if reset else 0))
    return list(ms), list(n)


def phc_last_error():
    return lib.phc_last_error().decode()


def phc_version():
    return lib.phc_version().decode()
