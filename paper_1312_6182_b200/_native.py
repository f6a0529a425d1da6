"""ctypes binding of libgpspca_b200.so (include/gpspca_b200.h).

There is no fallback: if the library is missing or no sm_100 device is
visible, every numeric entry point raises.  Importing this module does not
touch the GPU; the first call that needs a context does.
"""

import ctypes as C
import os
import threading

import numpy as np

# Load every kernel when the CUDA context is created instead of on first
# launch: a solve should not pay module-loading latency the first time it
# reaches a code path (only effective if nothing initialised CUDA earlier in
# the process; set CUDA_MODULE_LOADING yourself to override).
os.environ.setdefault("CUDA_MODULE_LOADING", "EAGER")

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GPSPCA_LIB", os.path.join(_PKG, "libgpspca_b200.so"))

GPS_OK, GPS_E_ARG, GPS_E_RANK, GPS_E_OOM, GPS_E_CUDA, GPS_E_UNSUPPORTED = range(6)
F32, F64 = 0, 1
PENALTY_CODE = {"l1": 0, "l0": 1}

_dp = C.POINTER(C.c_double)
_vp = C.c_void_p
_i64 = C.c_int64
_i64p = C.POINTER(C.c_int64)
_ip = C.POINTER(C.c_int)

# name -> (restype, argtypes); the exported surface of include/gpspca_b200.h
SIGNATURES = {
    "gps_version": (C.c_int, []),
    "gps_last_error": (C.c_char_p, []),
    "gps_device_count": (C.c_int, [_ip]),
    "gps_device_free_bytes": (C.c_int, [_vp, C.POINTER(C.c_size_t)]),
    "gps_ctx_create": (C.c_int, [C.c_int, C.POINTER(_vp)]),
    "gps_ctx_destroy": (C.c_int, [_vp]),
    "gps_ctx_set_stream": (C.c_int, [_vp, _vp]),
    "gps_ctx_sync": (C.c_int, [_vp]),
    "gps_ctx_launch_count": (_i64, [_vp]),
    "gps_matrix_create": (C.c_int, [_vp, _vp, _i64, _i64, _i64, C.c_int, C.POINTER(_vp)]),
    "gps_matrix_create_device": (C.c_int, [_vp, _vp, _i64, _i64, _i64, C.c_int, C.POINTER(_vp)]),
    "gps_matrix_wrap_device": (C.c_int, [_vp, _vp, _i64, _i64, _i64, C.c_int, C.POINTER(_vp)]),
    "gps_matrix_create_rowmajor": (C.c_int, [_vp, _vp, _i64, _i64, C.c_int, C.POINTER(_vp)]),
    "gps_matrix_destroy": (C.c_int, [_vp]),
    "gps_matrix_info": (C.c_int, [_vp, _i64p, _i64p, _i64p, _ip]),
    "gps_matrix_download": (C.c_int, [_vp, _vp]),
    "gps_matrix_column": (C.c_int, [_vp, _i64, _dp]),
    "gps_matrix_device_ptr": (_vp, [_vp]),
    "gps_column_norms": (C.c_int, [_vp, _dp, _ip]),
    "gps_matrix_deflate": (C.c_int, [_vp, _dp, C.POINTER(_vp)]),
    "gps_matrix_gather": (C.c_int, [_vp, _i64p, _i64, C.POINTER(_vp)]),
    "gps_bench_read_stream": (C.c_int, [_vp, C.c_int, _dp]),
    "gps_matvec_t": (C.c_int, [_vp, _dp, _dp]),
    "gps_gram_apply": (C.c_int, [_vp, _dp, _dp]),
    "gps_threshold_accumulate": (C.c_int, [_vp, _dp, C.c_double, C.c_int, _dp]),
    "gps_su_sweep": (C.c_int, [_vp, _dp, C.c_double, C.c_int, _dp, _dp, _dp, _dp, _i64p]),
    "gps_su_create": (C.c_int, [_vp, C.c_int, C.c_double, C.c_double, C.c_int, C.POINTER(_vp)]),
    "gps_su_destroy": (C.c_int, [_vp]),
    "gps_su_start": (C.c_int, [_vp, _dp]),
    "gps_su_run": (C.c_int, [_vp, C.c_int]),
    "gps_su_set_deflation": (C.c_int, [_vp, _dp, C.c_int]),
    "gps_su_enqueue_sweep": (C.c_int, [_vp]),
    "gps_su_exchange": (C.c_int, [_vp, C.POINTER(_vp), _i64p]),
    "gps_su_set_exchange": (C.c_int, [_vp, _vp]),
    "gps_su_enqueue_step": (C.c_int, [_vp]),
    "gps_su_enqueue": (C.c_int, [_vp, C.c_int]),
    "gps_su_poll": (C.c_int, [_vp, _ip, _ip, _ip]),
    "gps_su_result": (C.c_int, [_vp, _dp, _dp, _ip, _ip, _dp, _dp]),
    "gps_su_launches_per_iter": (C.c_int, [_vp]),
    "gps_su_band": (C.c_int, [_vp, _i64p, C.c_int, _ip]),
    "gps_bk_diagnostics": (C.c_int, [_vp, _dp, _ip, _ip]),
    "gps_bk_band": (C.c_int, [_vp, _i64p, C.c_int, _ip]),
    "gps_bk_last_sweep": (C.c_int, [_vp, _dp, _dp]),
    "gps_bk_create": (C.c_int, [_vp, C.c_int, C.c_int, _dp, _dp, C.c_double, C.c_int, C.POINTER(_vp)]),
    "gps_bk_destroy": (C.c_int, [_vp]),
    "gps_bk_start": (C.c_int, [_vp, _dp]),
    "gps_bk_start_qr": (C.c_int, [_vp, _dp]),
    "gps_bk_start_columns": (C.c_int, [_vp, _i64p]),
    "gps_bk_run": (C.c_int, [_vp, C.c_int]),
    "gps_bk_enqueue_sweep": (C.c_int, [_vp]),
    "gps_bk_exchange": (C.c_int, [_vp, C.POINTER(_vp), _i64p]),
    "gps_bk_set_exchange": (C.c_int, [_vp, _vp]),
    "gps_bk_enqueue_step": (C.c_int, [_vp]),
    "gps_bk_poll": (C.c_int, [_vp, _ip, _ip, _ip]),
    "gps_bk_result": (C.c_int, [_vp, _dp, _dp, _ip, _ip, _dp, _ip, _ip]),
    "gps_bk_sweep": (C.c_int, [_vp, _dp, C.c_int, _dp, _dp, C.c_int, _dp, _dp, _dp]),
    "gps_polar": (C.c_int, [_vp, _dp, _i64, C.c_int, _dp, _ip]),
    "gps_polar_cholqr2": (C.c_int, [_vp, _dp, _i64, C.c_int, _dp, _ip, _dp, _ip]),
    "gps_orthonormalize": (C.c_int, [_vp, _dp, _i64, C.c_int, _dp]),
    "gps_gram_apply_block": (C.c_int, [_vp, _dp, C.c_int, _dp]),
    "gps_matrix_center": (C.c_int, [_vp, _dp, C.POINTER(_vp)]),
    "gps_row_sqnorms": (C.c_int, [_vp, _vp, _i64, C.c_int, _vp]),
    "gps_knn_distances": (C.c_int, [_vp, _vp, _i64, _vp, _i64, C.c_int, _vp, _vp, _vp]),
    "gps_knn_topk": (C.c_int, [_vp, _vp, _i64, _i64, C.c_int, _vp]),
    "gps_matrix_svd": (C.c_int, [_vp, _dp, _dp, _ip]),
    "gps_px_create": (C.c_int, [_vp, C.c_int, C.c_int, _i64, C.POINTER(_vp)]),
    "gps_px_handle_size": (C.c_int, []),
    "gps_px_ipc_handle": (C.c_int, [_vp, _vp]),
    "gps_px_open": (C.c_int, [_vp, C.c_int, _vp]),
    "gps_px_allreduce": (C.c_int, [_vp, _vp]),
    "gps_px_allreduce_phase": (C.c_int, [_vp, _vp, C.c_int]),
    "gps_px_reduce_phase": (C.c_int, [_vp, _vp, _vp, C.c_int, C.c_int, C.c_int, _vp, C.c_int]),
    "gps_px_destroy": (C.c_int, [_vp]),
    "gps_px_set_timeout": (C.c_int, [_vp, C.c_double]),
    "gps_px_error": (C.c_int, [_vp, _ip]),
    "gps_px_emulate_timeout": (C.c_int, [_vp, C.c_int, _i64, C.c_double, _ip]),
    "gps_px_emulate": (C.c_int, [_vp, C.c_int, _i64, C.c_int, _dp, _dp]),
    "gps_su_attach_px": (C.c_int, [_vp, _vp]),
    "gps_bk_attach_px": (C.c_int, [_vp, _vp]),
    "gps_bk_exchange_stride": (C.c_int, [_vp, _i64p]),
    "gps_px_emulate_reduce": (C.c_int, [_vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _dp, _dp, _dp]),
}


class NativeError(RuntimeError):
    """A CUDA-side failure inside libgpspca_b200 (GPS_E_CUDA)."""


_lib = None
_lib_lock = threading.Lock()


def lib():
    """Load the shared library (once).  Raises if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lib_lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(
                    f"{LIB_PATH} is missing: build it with `python -m paper_1312_6182_b200._build` "
                    "(there is no CPU fallback)")
            handle = C.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def last_error():
    msg = lib().gps_last_error()
    return msg.decode() if msg else ""


def check(rc, what=""):
    """Map a gps_status to the reference's exception types."""
    if rc == GPS_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if rc == GPS_E_ARG:
        raise ValueError(msg)
    if rc == GPS_E_OOM:
        raise MemoryError(msg)
    if rc == GPS_E_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise NativeError(msg)


def dptr(a):
    """Pointer to a C-contiguous float64 numpy array."""
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


class Context:
    """One device + one CUDA stream (gps_ctx)."""

    def __init__(self, device):
        self.device = int(device)
        h = _vp()
        check(lib().gps_ctx_create(self.device, C.byref(h)), "gps_ctx_create")
        self.handle = h

    def sync(self):
        check(lib().gps_ctx_sync(self.handle))

    def set_stream(self, stream_ptr):
        """Adopt a caller CUDA stream (None: back to a library-owned stream)."""
        check(lib().gps_ctx_set_stream(self.handle, None if stream_ptr is None else _vp(stream_ptr)))

    @property
    def launch_count(self):
        return int(lib().gps_ctx_launch_count(self.handle))


_contexts = {}
_ctx_lock = threading.Lock()


def default_device():
    for var in ("GPSPCA_DEVICE", "LOCAL_RANK"):
        if var in os.environ:
            return int(os.environ[var])
    return 0


def context(device=None):
    device = default_device() if device is None else int(device)
    with _ctx_lock:
        ctx = _contexts.get(device)
        if ctx is None:
            ctx = Context(device)
            _contexts[device] = ctx
        return ctx


def device_count():
    n = C.c_int(0)
    check(lib().gps_device_count(C.byref(n)))
    return n.value
