"""phc-b200: evaluate a sparse polynomial system and its Jacobian on a B200 in complex
double-double / quad-double arithmetic (Verschelde & Yoffe 2011, arXiv 1109.0545, §6).

The C ABI (include/phc.h) is the boundary; this package only marshals arguments.
"""
from ._lib import (  # noqa: F401
    PHC_EINVAL,
    PHC_ECUDA,
    PHC_ENOMEM,
    PHC_EUNSUPPORTED,
    PHC_OK,
    PhcError,
    phc_eval_jacobian,
    phc_eval_jacobian_batch,
    phc_eval_jacobian_batch_host,
    phc_eval_jacobian_batch_range,
    phc_ipc_get_handle,
    phc_ipc_open,
    phc_ipc_close,
    phc_fp64_peak,
    phc_last_error,
    phc_newton_step_batch,
    phc_newton_step_homotopy_batch,
    phc_newton_solve_batch,
    phc_eval_homotopy_batch,
    phc_system_set_target,
    phc_system_create_common,
    phc_predict_batch,
    phc_arith_test,
    phc_track_paths,
    TrackParams,
    phc_homotopy_old_create,
    phc_profile_enable,
    phc_profile_read,
    phc_system_create,
    phc_system_destroy,
    phc_system_stats,
    phc_version,
)
from .system import System, predict_batch  # noqa: F401
