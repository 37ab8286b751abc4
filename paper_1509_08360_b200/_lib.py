"""ctypes binding of the C ABI in include/csemb_cuda.h (libcsemb_cuda.so).

The shared library is built in-tree (``python -m paper_1509_08360_b200.build``
or ``__graft_entry__.build()``).  There is no CPU fallback: if the library or
a GPU is missing, every device entry point raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from .errors import CudaUnavailableError, DivergenceError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CSEMB_LIB_PATH") or os.path.join(_HERE, "libcsemb_cuda.so")

OK, ERR_INVALID, ERR_CUDA, ERR_NOMEM, ERR_DIVERGED, ERR_UNSUPPORTED = range(6)
F64, F32 = 0, 1
OMEGA_GIVEN, OMEGA_SPLITMIX, OMEGA_PHILOX = 0, 1, 2
OPT_EXACT_PEAKS, OPT_REVERSE_SWEEP, OPT_SPLIT_THRESHOLD, OPT_ROW_ORDER, OPT_E_FOLD, OPT_GRAPH = 1, 2, 3, 4, 5, 6
OPT_VALUE_FREE = 7

DIVERGENCE_MESSAGE = (
    "iteration r={r} produced non-finite values; the matrix likely has "
    "spectral norm > 1 - rescale it (estimate_spectral_norm) and retry"
)  # engine.py:222-224

_p = C.c_void_p
_i64 = C.c_int64
_u64 = C.c_uint64
_int = C.c_int
_dbl = C.c_double
_pp = C.POINTER(C.c_void_p)
_pi = C.POINTER(C.c_int)
_pi64 = C.POINTER(C.c_int64)
_pf = C.POINTER(C.c_float)
_pd = C.POINTER(C.c_double)

# name -> (restype, argtypes); mirrors include/csemb_cuda.h
SIGNATURES = {
    "csemb_last_error": (C.c_char_p, []),
    "csemb_abi_version": (_int, []),
    "csemb_device_count": (_int, [_pi]),
    "csemb_ctx_create": (_int, [_int, _pp]),
    "csemb_ctx_destroy": (_int, [_p]),
    "csemb_ctx_stream": (_p, [_p]),
    "csemb_ctx_sync": (_int, [_p]),
    "csemb_ctx_sm_count": (_int, [_p, _pi]),
    "csemb_matrix_upload": (_int, [_p, _i64, _i64, _i64, _p, _p, _p, _int, _pp]),
    "csemb_matrix_upload_device": (_int, [_p, _i64, _i64, _i64, _p, _p, _int, _p, _int, _pp]),
    "csemb_matrix_destroy": (_int, [_p]),
    "csemb_matrix_info": (_int, [_p, _pi64, _pi64, _pi64, _pi]),
    "csemb_matrix_scale": (_int, [_p, _dbl]),
    "csemb_matrix_value_free": (_int, [_p, _pi]),
    "csemb_matrix_download_values": (_int, [_p, _p]),
    "csemb_matrix_convert": (_int, [_p, _int, _pp]),
    "csemb_matrix_device_arrays": (_int, [_p, _pp, _pp, _pp]),
    "csemb_build_normalized_adjacency": (_int, [_p, _i64, _i64, _p, _int, _int, _pp]),
    "csemb_build_dilation": (_int, [_p, _pp]),
    "csemb_diag_bandwidth": (_int, [_p, _int, _i64, _i64, _int, _pd]),
    "csemb_diag_gather_csr": (_int, [_p, _i64, _int, _pd, _pd]),
    "csemb_plan_create": (_int, [_p, _i64, _pp]),
    "csemb_plan_destroy": (_int, [_p]),
    "csemb_plan_set_option": (_int, [_p, _int, _i64]),
    "csemb_plan_run": (_int, [_p, _p, _int, _int, _p, _int, _u64, _i64, _i64, _int]),
    "csemb_plan_download": (_int, [_p, _p, _int]),
    "csemb_plan_output": (_int, [_p, _pp, _pi64, _pi]),
    "csemb_plan_copy_output": (_int, [_p, _p, _i64]),
    "csemb_plan_diagnostics": (_int, [_p, _p, _pi, _pi]),
    "csemb_plan_timing": (_int, [_p, _pf, _pf, _pi]),
    "csemb_apply_expansion": (
        _int, [_p, _p, _int, _int, _p, _int, _u64, _i64, _i64, _int, _p, _p, _pi, _pi]),
    "csemb_plan_partition": (_int, [_p, _i64, _i64, _p, _p, _p]),
    "csemb_plan_partition_peers": (_int, [_p, _i64, _i64, _p, _p, _int, _p, _p]),
    "csemb_plan_partition_multicast": (_int, [_p, _i64, _i64, _p, _p, _p, _p]),
    "csemb_plan_partition_split": (_int, [_p, _i64, _i64, _p, _p, _p]),
    "csemb_plan_step_local": (_int, [_p, _int]),
    "csemb_plan_begin": (_int, [_p, _p, _int, _p, _int, _u64, _i64, _i64]),
    "csemb_plan_step": (_int, [_p, _int]),
    "csemb_plan_end": (_int, [_p, _int]),
    "csemb_sample_projection": (_int, [_p, _i64, _i64, _u64, _i64, _i64, _int, _p]),
    "csemb_rownorm": (_int, [_p, _p, _i64, _i64, _i64, _int]),
    "csemb_spectral_norm": (_int, [_p, _int, _i64, _p, _u64, _dbl, _pd]),
    # downstream consumers (cluster.py, oracle.py:88-119)
    "csemb_pair_cosines": (_int, [_p, _p, _int, _int, _i64, _i64, _i64, _p, _i64, _p, _p]),
    "csemb_kmeans_create": (_int, [_p, _p, _int, _int, _i64, _i64, _i64, _int, _pp]),
    "csemb_kmeans_destroy": (_int, [_p]),
    "csemb_kmeans_seed": (_int, [_p, _int, _i64, _pd]),
    "csemb_kmeans_pick": (_int, [_p, _dbl, _pi64]),
    "csemb_kmeans_assign": (_int, [_p, _pd, _pi64, _p]),
    "csemb_kmeans_reseed": (_int, [_p, _int, _pi64]),
    "csemb_kmeans_commit": (_int, [_p, _int]),
    "csemb_kmeans_download": (_int, [_p, _p, _p]),
    "csemb_kmeans_set_centroids": (_int, [_p, _p]),
    "csemb_kmeans_reset": (_int, [_p]),
    "csemb_kmeans_labels": (_p, [_p]),
    "csemb_modularity_counts": (_int, [_p, _p, _int, _i64, _p, _p]),
}

_lock = threading.Lock()
_lib = None


def load():
    """Load libcsemb_cuda.so (raises CudaUnavailableError if it is not built)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise CudaUnavailableError(
                    f"{LIB_PATH} is not built; run __graft_entry__.build() "
                    "(there is no CPU fallback)"
                )
            lib = C.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            if lib.csemb_abi_version() != 1:
                raise CudaUnavailableError("libcsemb_cuda.so ABI version mismatch")
            _lib = lib
    return _lib


def last_error() -> str:
    return (load().csemb_last_error() or b"").decode(errors="replace")


def check(rc: int, what: str = "") -> None:
    """Map a C status code to the reference's exception types."""
    if rc == OK:
        return
    msg = last_error()
    if what:
        msg = f"{what}: {msg}"
    if rc == ERR_INVALID:
        raise ValueError(msg)
    if rc == ERR_DIVERGED:
        raise DivergenceError(msg)
    if rc == ERR_NOMEM:
        raise MemoryError(msg)
    if rc == ERR_UNSUPPORTED:
        raise NotImplementedError(msg)
    raise CudaUnavailableError(msg)


def device_count() -> int:
    try:
        lib = load()
    except CudaUnavailableError:
        return 0
    n = C.c_int(0)
    lib.csemb_device_count(C.byref(n))
    return int(n.value)


def host_empty(shape, dtype=np.float64) -> np.ndarray:
    """An uninitialised host array for a device -> host result, backed by
    torch's caching pinned-host allocator when torch is present: a fresh
    np.empty of config 2's 640 MB E costs ~100 ms of first-touch page faults
    plus a pageable (staged) copy, while a cached pinned block is reused
    across calls and filled by DMA at full link speed.  The returned ndarray
    owns the block through its base (freed back to the cache with it)."""
    nbytes = int(np.prod(shape)) * np.dtype(dtype).itemsize
    if (1 << 20) <= nbytes <= (16 << 30) and _pinning_available():
        try:
            import torch

            t = torch.empty(int(np.prod(shape)), dtype=getattr(torch, np.dtype(dtype).name), pin_memory=True)
            return t.numpy().reshape(shape)
        except Exception:  # no pinned memory available: plain pageable array
            pass
    return np.empty(shape, dtype=dtype)


_PINNING = None


def _pinning_available() -> bool:
    global _PINNING
    if _PINNING is None:
        try:
            import torch

            _PINNING = bool(torch.cuda.is_available())
        except Exception:
            _PINNING = False
    return _PINNING


def ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class Context:
    """One CUDA device + stream (csemb_ctx)."""

    def __init__(self, device: int = 0):
        self.lib = load()
        h = C.c_void_p()
        check(self.lib.csemb_ctx_create(int(device), C.byref(h)), "csemb_ctx_create")
        self.handle = h
        self.device = int(device)
        sm = C.c_int(0)
        check(self.lib.csemb_ctx_sm_count(h, C.byref(sm)))
        self.sm_count = int(sm.value)

    @property
    def stream(self) -> int:
        return int(self.lib.csemb_ctx_stream(self.handle) or 0)

    def sync(self) -> None:
        check(self.lib.csemb_ctx_sync(self.handle), "csemb_ctx_sync")

    def torch_stream(self):
        """The context stream as a torch ExternalStream.  The library stream is
        created non-blocking, so torch / NCCL work is NOT ordered with it
        implicitly: run torch ops that touch library buffers under
        `torch.cuda.stream(ctx.torch_stream())` (device-side ordering, no host
        sync), or call `after_torch()` first."""
        import torch

        return torch.cuda.ExternalStream(self.stream, device=torch.device("cuda", self.device))

    def after_torch(self) -> None:
        """Order the context stream after everything queued so far on torch's
        current stream of this device (device-side wait, the host does not block)."""
        import torch

        self.torch_stream().wait_stream(torch.cuda.current_stream(torch.device("cuda", self.device)))

    def close(self) -> None:
        if self.handle:
            self.lib.csemb_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass


_contexts: dict[int, Context] = {}


def context(device: int = 0) -> Context:
    with _lock:
        ctx = _contexts.get(device)
    if ctx is None:
        ctx = Context(device)
        with _lock:
            _contexts.setdefault(device, ctx)
            ctx = _contexts[device]
    return ctx
