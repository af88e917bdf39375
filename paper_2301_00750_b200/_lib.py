"""ctypes binding of lib/libstreamstab_b200.so (include/streamstab_b200.h).

The product path has no CPU fallback: if the library is missing this module
raises at import, and every op requires a CUDA device.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

_PKG = os.path.dirname(os.path.abspath(__file__))
# SS_LIB_PATH: an alternative build of the same library (diagnostics)
LIB_PATH = os.environ.get("SS_LIB_PATH") or os.path.join(_PKG, "lib", "libstreamstab_b200.so")
CSRC = os.path.join(_PKG, "csrc")

SS_OK = 0
SS_RESOLUTION_MISMATCH = 1
SS_VALUE_ERROR = 2
SS_SOLVER_DIVERGENCE = 3
SS_STATE_POSITION, SS_STATE_OUTPUT, SS_STATE_CLEAR = 0, 1, 2
SS_CUDA_ERROR = 4
SS_NO_MEMORY = 5
SS_HOST = 0
SS_DEVICE = 1
SS_F32 = 0
SS_U8 = 1

# every symbol include/streamstab_b200.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "ss_abi_version", "ss_kernel_launches", "ss_status_string", "ss_last_error", "ss_init", "ss_params_validate",
    "ss_backward_warp", "ss_occlusion_mask", "ss_warp_weight", "ss_local_blend",
    "ss_adaptive_blend", "ss_consistency_weight", "ss_laplacian", "ss_solve_screened_poisson",
    "ss_session_create", "ss_session_destroy", "ss_session_reset", "ss_push_pair", "ss_stage_pair",
    "ss_solved_through", "ss_session_set_state", "ss_pending", "ss_set_flow", "ss_set_constant_flow", "ss_check_step",
    "ss_step", "ss_output", "ss_output_async", "ss_output_wait", "ss_output_device", "ss_last_timing", "ss_flows",
    "ss_session_stream", "ss_session_join", "ss_flownet_num_params", "ss_flownet_create", "ss_flownet_set_downscale", "ss_flownet_destroy",
    "ss_flownet_flow", "ss_session_attach_flownet", "ss_session_compute_flow",
    "ss_warping_error_sums", "ss_ssim", "ss_session_time_conv", "ss_dis_flow",
    "ss_session_compute_dis_flow", "ss_session_wait_stream", "ss_session_signal_stream",
)
SS_FLOW_FP32 = 0
SS_FLOW_BF16 = 1


class SSParams(ctypes.Structure):
    _fields_ = [
        ("k1", ctypes.c_float), ("k2", ctypes.c_float), ("alpha", ctypes.c_float),
        ("lam", ctypes.c_float), ("eta", ctypes.c_float), ("kappa", ctypes.c_float),
        ("iterations", ctypes.c_int32), ("flow_downscale", ctypes.c_int32),
    ]


class SSTiming(ctypes.Structure):
    _fields_ = [("flow_ms", ctypes.c_float), ("warp_blend_ms", ctypes.c_float),
                ("solve_ms", ctypes.c_float)]


def build(force: bool = False) -> str:
    """Compile the CUDA library for sm_100a in-tree (nvcc; no GPU needed)."""
    if force or not os.path.exists(LIB_PATH):
        subprocess.run(["make", "-s", "-C", CSRC], check=True)
    return LIB_PATH


def _declare(L):
    vp, i32, i64, f32 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_float
    P = ctypes.POINTER
    sig = {
        "ss_abi_version": (i32, []),
        "ss_kernel_launches": (ctypes.c_longlong, []),
        "ss_status_string": (ctypes.c_char_p, [i32]),
        "ss_last_error": (ctypes.c_char_p, []),
        "ss_init": (i32, [i32]),
        "ss_params_validate": (i32, [P(SSParams)]),
        "ss_backward_warp": (i32, [vp, i32, i32, i32, vp, vp, vp, vp, vp]),
        "ss_occlusion_mask": (i32, [vp, vp, vp, vp, i32, i32, vp, vp]),
        "ss_warp_weight": (i32, [vp, vp, i32, i32, i32, f32, f32, vp, vp, vp]),
        "ss_local_blend": (i32, [vp, vp, vp, vp, vp, i32, i32, i32, vp, vp]),
        "ss_adaptive_blend": (i32, [vp, vp, vp, i32, i32, i32, vp, vp]),
        "ss_consistency_weight": (i32, [vp, vp, i32, i32, i32, f32, f32, vp, vp]),
        "ss_laplacian": (i32, [vp, i32, i32, i32, vp, vp]),
        "ss_solve_screened_poisson": (i32, [vp, vp, vp, i32, i32, i32, P(SSParams), vp, vp,
                                            P(i32), vp]),
        "ss_session_create": (i32, [i32, i32, i32, i32, vp, P(vp)]),
        "ss_session_destroy": (i32, [vp]),
        "ss_session_reset": (i32, [vp]),
        "ss_push_pair": (i32, [vp, i64, vp, vp, i32, i32]),
        "ss_stage_pair": (i32, [vp, i64, vp, vp, i32, i32]),
        "ss_solved_through": (i64, [vp]),
        "ss_session_set_state": (i32, [vp, i32, i64, vp, i32, i32]),
        "ss_pending": (i32, [vp, P(i64), P(i32), P(i32)]),
        "ss_set_flow": (i32, [vp, i32, vp, vp, i32]),
        "ss_set_constant_flow": (i32, [vp, i32, ctypes.c_double, ctypes.c_double, i32]),
        "ss_check_step": (i32, [vp, i32, P(i64)]),
        "ss_step": (i32, [vp, i32, P(SSParams), P(i32)]),
        "ss_output": (i32, [vp, vp, i32, i32]),
        "ss_output_async": (i32, [vp, vp, i32, i32]),
        "ss_output_wait": (i32, [vp]),
        "ss_output_device": (vp, [vp]),
        "ss_last_timing": (i32, [vp, P(SSTiming)]),
        "ss_flows": (i32, [vp, i32, vp, vp, i32]),
        "ss_session_stream": (vp, [vp]),
        "ss_session_join": (i32, [vp]),
        "ss_flownet_num_params": (i64, []),
        "ss_flownet_create": (i32, [vp, i64, i32, P(vp)]),
        "ss_flownet_set_downscale": (i32, [vp, i32]),
        "ss_flownet_destroy": (i32, [vp]),
        "ss_flownet_flow": (i32, [vp, vp, vp, i32, i32, i32, vp, vp, vp]),
        "ss_session_attach_flownet": (i32, [vp, vp]),
        "ss_session_compute_flow": (i32, [vp, i32]),
        "ss_warping_error_sums": (i32, [vp, vp, i32, i32, i32, vp, vp, vp, vp,
                                        P(ctypes.c_double), vp]),
        "ss_ssim": (i32, [vp, vp, i32, i32, i32, P(ctypes.c_double), vp]),
        "ss_session_time_conv": (i32, [vp, i32, i32, P(f32), P(ctypes.c_double)]),
        "ss_dis_flow": (i32, [vp, vp, i32, i32, i32, i32, i32, i32, i32, vp, vp, vp]),
        "ss_session_compute_dis_flow": (i32, [vp, i32, i32, i32, i32, i32]),
        "ss_session_wait_stream": (i32, [vp, vp]),
        "ss_session_signal_stream": (i32, [vp, vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args


_lib = None


def lib():
    """Load the CUDA library; raises if it is missing (no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the B200 path has no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        _declare(L)
        _lib = L
    return _lib


def last_error() -> str:
    return lib().ss_last_error().decode()


class CudaError(RuntimeError):
    pass
