"""ctypes declarations of the C ABI in include/fftconv.h (argument marshalling
only -- every step of the convolution runs inside libfftconv.so).

Loading fails loudly if the library has not been built: there is no
fallback path."""
from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FFTCONV_LIB", os.path.join(HERE, "libfftconv.so"))  # override: experiments only

FFTCONV_F16, FFTCONV_BF16, FFTCONV_F32 = 0, 1, 2
STATUS = {
    0: "FFTCONV_OK",
    1: "FFTCONV_ERR_INVALID_ARG",
    2: "FFTCONV_ERR_NOT_POW2",
    3: "FFTCONV_ERR_KERNEL_TOO_LONG",
    4: "FFTCONV_ERR_BAD_SPARSITY",
    5: "FFTCONV_ERR_UNSUPPORTED",
    6: "FFTCONV_ERR_MISALIGNED",
    7: "FFTCONV_ERR_CUDA",
}

# every symbol include/fftconv.h declares (tests check the exports)
ABI_SYMBOLS = [
    "fftconv_plan", "fftconv_plan_info", "fftconv_plan_upload", "fftconv_precompute_kf",
    "fftconv_fwd", "fftconv_gated_fwd", "fftconv_bwd", "fftconv_plan_destroy",
    "fftconv_last_error", "fftconv_launch_count_reset", "fftconv_workspace_size",
    "fftconv_fwd_host", "fftconv_host_stage_size", "fftconv_fwd_stream", "fftconv_stream_stage_size",
    "fftconv_cost_eq2", "fftconv_select_order", "fftconv_factorize", "fftconv_cost_features",
    "fftconv_cost_predict", "fftconv_precompute_kf_bidir", "fftconv_bwd_bidir",
]


class FFTConvError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{STATUS.get(status, status)}: {message}")
        self.status = status


class Sparsity(ctypes.Structure):
    _fields_ = [("ndims", ctypes.c_int32), ("dims", ctypes.c_int32 * 4),
                ("keep", ctypes.POINTER(ctypes.c_uint8) * 4)]


class PlanInfo(ctypes.Structure):
    _fields_ = [
        ("N", ctypes.c_int64), ("fft_size", ctypes.c_int64), ("causal", ctypes.c_int32),
        ("dtype", ctypes.c_int32), ("regime", ctypes.c_int32), ("order", ctypes.c_int32),
        ("factors", ctypes.c_int32 * 6), ("rows_per_tile", ctypes.c_int32),
        ("max_kernel_len", ctypes.c_int64), ("table_bytes", ctypes.c_size_t),
        ("kf_bytes_per_head", ctypes.c_size_t), ("workspace_bytes_per_head", ctypes.c_size_t),
        ("mask_fraction", ctypes.c_double), ("skip_fraction", ctypes.c_double),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_2311_05908_b200.build` "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.c_void_p
        i64, i32 = ctypes.c_int64, ctypes.c_int32
        L.fftconv_plan.argtypes = [ctypes.POINTER(P), i64, i64, ctypes.c_int, ctypes.c_int,
                                   ctypes.POINTER(Sparsity)]
        L.fftconv_plan_info.argtypes = [P, ctypes.POINTER(PlanInfo)]
        L.fftconv_plan_upload.argtypes = [P, P, P]
        L.fftconv_precompute_kf.argtypes = [P, P, i64, i64, P, P]
        L.fftconv_fwd.argtypes = [P, P, P, P, i64, i64, P, P]
        L.fftconv_gated_fwd.argtypes = [P, P, P, P, P, P, i64, i64, P, P]
        L.fftconv_bwd.argtypes = [P, P, P, P, P, P, P, P, P, P, i64, i64, i64, P, P]
        L.fftconv_precompute_kf_bidir.argtypes = [P, P, P, i64, i64, P, P]
        L.fftconv_bwd_bidir.argtypes = [P, P, P, P, P, P, P, P, P, P, P, i64, i64, i64, P, P]
        L.fftconv_workspace_size.argtypes = [P, i64, i64, ctypes.c_int, ctypes.POINTER(ctypes.c_size_t)]
        L.fftconv_fwd_host.argtypes = [P, P, P, P, P, P, i64, i64, i64, P, ctypes.c_size_t, P]
        L.fftconv_fwd_host.restype = ctypes.c_int
        L.fftconv_host_stage_size.argtypes = [P, i64, i64, ctypes.c_int, ctypes.POINTER(ctypes.c_size_t)]
        L.fftconv_host_stage_size.restype = ctypes.c_int
        L.fftconv_fwd_stream.argtypes = [P, P, P, P, P, P, i64, i64, i64, P, ctypes.c_size_t, P]
        L.fftconv_fwd_stream.restype = ctypes.c_int
        L.fftconv_stream_stage_size.argtypes = [P, i64, i64, ctypes.c_int, ctypes.POINTER(ctypes.c_size_t)]
        L.fftconv_stream_stage_size.restype = ctypes.c_int
        L.fftconv_workspace_size.restype = ctypes.c_int
        for f in ("fftconv_plan", "fftconv_plan_info", "fftconv_plan_upload", "fftconv_precompute_kf",
                  "fftconv_fwd", "fftconv_gated_fwd", "fftconv_bwd", "fftconv_precompute_kf_bidir",
                  "fftconv_bwd_bidir"):
            getattr(L, f).restype = ctypes.c_int
        L.fftconv_plan_destroy.argtypes = [P]
        L.fftconv_plan_destroy.restype = None
        L.fftconv_last_error.restype = ctypes.c_char_p
        L.fftconv_launch_count_reset.restype = i64
        L.fftconv_cost_eq2.argtypes = [i64, i32] + [ctypes.c_double] * 6
        L.fftconv_cost_eq2.restype = ctypes.c_double
        L.fftconv_select_order.argtypes = [i64] + [ctypes.c_double] * 6
        L.fftconv_select_order.restype = i32
        D = ctypes.POINTER(ctypes.c_double)
        L.fftconv_cost_features.argtypes = [P, i64, i64, ctypes.c_int, ctypes.c_int, D]
        L.fftconv_cost_features.restype = ctypes.c_int
        L.fftconv_cost_predict.argtypes = [P, i64, i64, ctypes.c_int, ctypes.c_int, D, D]
        L.fftconv_cost_predict.restype = ctypes.c_int
        L.fftconv_factorize.argtypes = [i64, i32, ctypes.POINTER(i64)]
        L.fftconv_factorize.restype = i32
        _lib = L
    return _lib


def check(status: int) -> None:
    if status != 0:
        msg = lib().fftconv_last_error().decode()
        raise FFTConvError(status, msg)
