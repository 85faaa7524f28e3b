"""ctypes binding of ``libspa2.so`` (the C ABI declared in ``include/spa2.h``).

The library is built in-tree by ``__graft_entry__.build()`` (``make -C csrc``) and loaded
from this directory (always this file: no environment variable can swap the product
library).  There is no fallback: if the library or a CUDA device is missing, every
operator raises.  ``load_diag()`` loads ``libspa2_diag.so`` (``include/spa2_diag.h``:
micro-benchmarks and probes for tests/ and tools/ only).  Status codes map to the exceptions the reference raises
(``ValueError`` / ``FloatingPointError``, numerics.py:17-32) or ``RuntimeError`` for CUDA
failures.
"""

from __future__ import annotations

import ctypes
import os
import re
import threading

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libspa2.so")
DIAG_LIB_PATH = os.path.join(_HERE, "libspa2_diag.so")
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "spa2.h")
DIAG_HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "spa2_diag.h")

SPA2_OK = 0
SPA2_ERR_VALUE = -1
SPA2_ERR_NONFINITE = -2
SPA2_ERR_UNSUPPORTED = -3
SPA2_ERR_CUDA = -4

DTYPE_CODES = {torch.bfloat16: 0, torch.float16: 1, torch.float32: 2, torch.float64: 3}


class View(ctypes.Structure):
    """``spa2_view``: base pointer + element strides of the B, H, N axes."""

    _fields_ = [("ptr", ctypes.c_void_p), ("sb", ctypes.c_int64), ("sh", ctypes.c_int64), ("sn", ctypes.c_int64)]


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int
_F32 = ctypes.c_float
_F64 = ctypes.c_double

SIGNATURES = {
    "spa2_version": ([], ctypes.c_char_p),
    "spa2_last_error": ([], ctypes.c_char_p),
    "spa2_device_supported": ([_I32], _I32),
    "spa2_pooled_map": ([View, View, _I32, _I64, _I64, _I64, _I64, _I64, _I64, _P, _P, _P, _P], _I32),
    "spa2_select": ([_P, _I64, _I64, _I64, _F64, _P, _P, _P], _I32),
    "spa2_check_finite": ([View, _I32, _I64, _I64, _I64, _I64, _P, _P], _I32),
    "spa2_pooled_scores": ([View, View, _I32, _I64, _I64, _I64, _I64, _I64, _I64, _P, _P, _P, _P], _I32),
    "spa2_block_mean_pool": ([View, View, _I32, _I64, _I64, _I64, _I64, _I64, _I64, _P, _P, _P, _P], _I32),
    "spa2_select_scores": ([_P, _I64, _I64, _I64, _F64, _P, _P, _P], _I32),
    "spa2_build_lists": ([_P, _I64, _I64, _I64, _P, _P, _P, _P, _P, _P, _P, _P], _I32),
    "spa2_fwd": ([View, View, View, View, _P, _I32, _I64, _I64, _I64, _I64, _I64, _I64, _P, _P, _P, _F32, _P, _P],
                 _I32),
    "spa2_bwd": ([View, View, View, View, View, _P, _P, View, View, View, _I32, _I64, _I64, _I64, _I64, _I64, _I64,
                  _P, _P, _P, _P, _P, _P, _F32, _P], _I32),
    "spa2_bwd_delta": ([View, View, _P, _I32, _I64, _I64, _I64, _I64, _P], _I32),
    "spa2_bwd_dq": ([View, View, View, View, _P, _P, View, _I32, _I64, _I64, _I64, _I64, _I64, _I64, _P, _P, _P, _F32,
                     _P], _I32),
    "spa2_bwd_dkdv": ([View, View, View, View, _P, _P, View, View, _I32, _I64, _I64, _I64, _I64, _I64, _I64, _P, _P,
                       _P, _F32, _P], _I32),
    "spa2_bwd_dq_delta": ([View, View, View, View, View, _P, _P, View, _I32, _I64, _I64, _I64, _I64, _I64, _I64, _P, _P,
                           _P, _F32, _P], _I32),
}

DIAG_SIGNATURES = {
    "spa2_last_error": ([], ctypes.c_char_p),
    "spa2_probe_gemm": ([_P, _P, _P, _I32, _I32, _I32, _I32, _I32, _I32, _P], _I32),
    "spa2_probe_mma_rate": ([_I32, _I32, _I32, _I32, _I32, _I32, _I32, _I32, _P, _P], _I32),
    "spa2_probe_tma_rate": ([_P, ctypes.c_longlong, _I32, _I32, _I32, _I32, _P, _P], _I32),
    "spa2_probe_mma_mix": ([_I32, _I32, _I32, _P, _P, _P], _I32),
    "spa2_probe_mbar_latency": ([_I32, _I32, _I32, _P, _P], _I32),
    "spa2_probe_tmem_rate": ([_I32, _I32, _I32, _I32, _P, _P], _I32),
    "spa2_probe_tma_rate2": ([_P, ctypes.c_longlong, _I32, _I32, _I32, _I32, _I32, _I32, _I32, _P, _P], _I32),
    "spa2_probe_red_rate": ([_P, _I32, _I32, _I32, _I32, _P], _I32),
    "spa2_probe_clock": ([_I32, _I32, _P, _P], _I32),
    "spa2_probe_smem_contend": ([_I32, _I32, _I32, _P, _P, _P], _I32),
    "spa2_probe_dkdv_mix": ([_I32, _I32, _I32, _P, _P], _I32),
    "spa2_probe_cp_rate": ([_I32, _I32, _I32, _P, _P], _I32),
}

# Kernels each entry point launches (for the bench's gpu_launches accounting).
KERNELS_PER_CALL = {"spa2_check_finite": 1, "spa2_block_mean_pool": 1, "spa2_pooled_map": 3, "spa2_select": 1, "spa2_pooled_scores": 2, "spa2_select_scores": 1, "spa2_build_lists": 3, "spa2_fwd": 1,
                    "spa2_bwd_delta": 1, "spa2_bwd_dq": 1, "spa2_bwd_dkdv": 1, "spa2_bwd": 2,
                    "spa2_bwd_dq_delta": 1}


class LaunchStats:
    """Counts kernels launched through the hot-path entry points, and optionally times
    chosen entry points with CUDA events on the launching stream."""

    def __init__(self):
        self.launches = 0
        self.timing = None  # dict name -> list[(start_event, end_event)] while enabled

    def begin(self, name: str, stream):
        self.launches += KERNELS_PER_CALL.get(name, 0)
        if self.timing is not None and name in self.timing:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(stream)
            return ev
        return None

    def end(self, name: str, start, stream):
        if start is not None:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(stream)
            self.timing[name].append((start, ev))


STATS = LaunchStats()


def call(name: str, *args, stream_obj=None):
    """Invoke entry point ``name`` (its last argument is the stream handle)."""
    start = STATS.begin(name, stream_obj) if stream_obj is not None else None
    if stream_obj is None:
        STATS.launches += KERNELS_PER_CALL.get(name, 0)
    fn = getattr(load(), name)
    if stream_obj is not None:
        # the C entry points launch on the calling thread's current device: make it the
        # device of the stream (and of the tensors) even if the caller's current device differs
        with torch.cuda.device(stream_obj.device):
            rc = fn(*args)
    else:
        rc = fn(*args)
    if start is not None:
        STATS.end(name, start, stream_obj)
    check(rc, name)
    if _SYNC_CALLS:  # diagnostic: attribute an asynchronous fault to the call that caused it
        try:
            torch.cuda.synchronize()
        except Exception as e:  # noqa: BLE001
            raise RuntimeError(f"{name}: asynchronous failure: {e}") from e


_SYNC_CALLS = os.environ.get("SPA2_SYNC_CALLS", "0") == "1"

_lock = threading.Lock()
_lib = None
_checked_devices: set[int] = set()


def header_symbols(path: str = HEADER_PATH) -> list[str]:
    """Every function a public header declares."""
    with open(path) as f:
        text = f.read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w[\w\s\*]*?\b(spa2_\w+)\s*\(", text, flags=re.M)))


def _open(path: str, signatures: dict) -> ctypes.CDLL:
    if not os.path.exists(path):
        raise RuntimeError(
            f"{os.path.basename(path)} not found at {path}; build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` (there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (args, res) in signatures.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


def load() -> ctypes.CDLL:
    """Load (once) and type the product library.  Raises if it has not been built."""
    global _lib
    with _lock:
        if _lib is None:
            _lib = _open(LIB_PATH, SIGNATURES)
    return _lib


_diag = None


def load_diag() -> ctypes.CDLL:
    """Load (once) the diagnostics library (tests/ and tools/ only)."""
    global _diag
    with _lock:
        if _diag is None:
            _diag = _open(DIAG_LIB_PATH, DIAG_SIGNATURES)
    return _diag


def use_library(path: str) -> None:
    """Load the product library from ``path`` instead of the in-tree build (A/B timing of an
    alternative build by tools; an explicit call, never an environment variable).  Must run
    before the first operator call."""
    global LIB_PATH
    with _lock:
        if _lib is not None and os.path.abspath(path) != os.path.abspath(LIB_PATH):
            raise RuntimeError("libspa2.so is already loaded; use_library() must come first")
        LIB_PATH = os.path.abspath(path)


def last_error() -> str:
    return load().spa2_last_error().decode(errors="replace")


def check(rc: int, what: str, _err=None) -> None:
    if rc == SPA2_OK:
        return
    msg = f"{what}: {(_err or last_error)()}"
    if rc in (SPA2_ERR_VALUE, SPA2_ERR_UNSUPPORTED):
        raise ValueError(msg)
    if rc == SPA2_ERR_NONFINITE:
        raise FloatingPointError(msg)
    raise RuntimeError(msg)


def check_diag(rc: int, what: str) -> None:
    """``check`` for libspa2_diag.so calls (its error message lives in that library)."""
    check(rc, what, lambda: load_diag().spa2_last_error().decode(errors="replace"))


def require_device(device: torch.device) -> None:
    """Fail loudly unless ``device`` is a CUDA sm_100 GPU (no CPU fallback exists)."""
    if device.type != "cuda":
        raise RuntimeError("paper_2602_13515_b200 runs on CUDA (B200, sm_100a) only; got device " + str(device))
    idx = device.index if device.index is not None else torch.cuda.current_device()
    if idx not in _checked_devices:
        check(load().spa2_device_supported(idx), "device check")
        _checked_devices.add(idx)


def stream_of(t: torch.Tensor) -> int:
    return torch.cuda.current_stream(t.device).cuda_stream


def ptr(t: torch.Tensor | None):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def view4(t: torch.Tensor) -> View:
    """``spa2_view`` of a [B, H, N, d] tensor whose last axis is contiguous."""
    if t.dim() != 4 or (t.stride(3) != 1 and t.shape[3] > 1):
        raise ValueError(f"expected a [B,H,N,d] tensor with contiguous last axis, got {tuple(t.shape)} "
                         f"strides {t.stride()}")
    return View(t.data_ptr(), t.stride(0), t.stride(1), t.stride(2))
