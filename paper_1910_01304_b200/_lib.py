"""ctypes binding of lib/libhrpp_b200.so (the C ABI in include/hrpp_b200.h).

There is no fallback: if the shared library is missing the import of the
package fails with instructions to build it, and every compute call goes
through the CUDA kernels (a call without a CUDA device raises).
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from .errors import CapacityExceeded, NonFiniteInput

import os

LIB_PATH = Path(os.environ.get("HRPP_LIB") or
                Path(__file__).resolve().parent / "lib" / "libhrpp_b200.so")

OK, NONFINITE, CAPACITY, INVALID_ARG, CUDA_ERR = 0, 1, 2, 3, 4
HIT_ANY, CLOSEST_HIT = 0, 1
MODE_BASELINE, MODE_LIMIT, MODE_LIVE, MODE_FAST = 0, 1, 2, 3
STATS_LEN = 11

P = C.c_void_p
I64 = C.c_int64
I32 = C.c_int32


class WaveOut(C.Structure):
    _fields_ = [("found", P), ("t", P), ("slot", P), ("leaf", P), ("u", P), ("v", P),
                ("box", P), ("tri", P), ("visited", P), ("keys", P)]


class OutcomeLogC(C.Structure):
    _fields_ = [("cls", P), ("eval_box", P), ("pred_t", P), ("pred_slot", P)]


def _load():
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build the sm_100a library first with "
            "`python -m paper_1910_01304_b200.build` (no CPU fallback exists)")
    L = C.CDLL(str(LIB_PATH))
    L.hrpp_last_error.restype = C.c_char_p
    L.hrpp_version.restype = C.c_int
    L.hrpp_launch_count.restype = I64
    L.hrpp_device_count.argtypes = [P]
    L.hrpp_set_live_rounds.argtypes = [C.c_int]
    L.hrpp_set_fast_rounds.argtypes = [C.c_int, C.c_int]
    L.hrpp_set_consult_short.argtypes = [C.c_int]
    L.hrpp_gen_primary.argtypes = [P, P, C.c_double, C.c_double, I64, I64, I64, I64, I64,
                                   C.c_uint64, C.c_int, P, P, P]
    L.hrpp_spawn.argtypes = [P, P, P, P, P, P, I64, C.c_int, P, C.c_double, C.c_int, C.c_uint64,
                             P, P, P, P, P, P, P, P, P, P]
    L.hrpp_profile_enable.argtypes = [C.c_int]
    L.hrpp_profile_stages.argtypes = [C.c_uint]
    L.hrpp_profile_read.argtypes = [P, P, C.c_int, C.c_int]
    L.hrpp_hash_rays.argtypes = [P, P, I64, C.c_int, P, P]
    L.hrpp_hash_floats.argtypes = [P, I64, C.c_int, P, P]
    L.hrpp_coarsen_keys.argtypes = [P, I64, C.c_int, P, P]
    L.hrpp_bvh_create.argtypes = [P] * 13 + [I64, I64, C.c_int, P]
    L.hrpp_bvh_destroy.argtypes = [P]
    L.hrpp_bvh_ancestor_lut.argtypes = [P, C.c_int, P]
    L.hrpp_build_bvh.argtypes = [P, P, P, P, I64, C.c_int, C.c_int] + [P] * 16
    L.hrpp_trace_batch.argtypes = [P, C.c_int, P, P, P, P, I32, I64, C.POINTER(WaveOut), P]
    L.hrpp_table_create.argtypes = [C.c_int, C.c_int, C.c_int, I64, C.c_int, P]
    L.hrpp_table_destroy.argtypes = [P]
    L.hrpp_table_clear.argtypes = [P]
    L.hrpp_table_clear_async.argtypes = [P, P]
    L.hrpp_table_info.argtypes = [P, P, P, P]
    L.hrpp_table_record.argtypes = [P, P, P, I64, P, P]
    L.hrpp_table_lookup.argtypes = [P, C.c_uint64, P, I64, P]
    L.hrpp_table_export.argtypes = [P, P, P, P]
    L.hrpp_table_set_deferred.argtypes = [P, C.c_int]
    L.hrpp_table_pending.argtypes = [P, P, P, P, I64, P]
    L.hrpp_partition_by_owner.argtypes = [P, I64, C.c_int, P, P, P]
    L.hrpp_pack_rays.argtypes = [P, I64, P, P, P, P, P, P]
    L.hrpp_unpack_rays.argtypes = [P, I64, P, P, P, P, P]
    L.hrpp_pack_hits.argtypes = [I64, P, P, P, P, P, P]
    L.hrpp_unpack_hits.argtypes = [P, P, I64, P, P, P, P, P]
    L.hrpp_predict_batch.argtypes = [P, P, P, P, P, P, P, I64] + [P] * 10 + [P]
    L.hrpp_trace_wave.argtypes = [P, P, C.c_int, C.c_int, P, P, P, P, I64, C.POINTER(WaveOut),
                                  C.POINTER(OutcomeLogC), P, P]
    for name in ("hrpp_device_count", "hrpp_set_live_rounds", "hrpp_set_fast_rounds",
                 "hrpp_hash_rays",
                 "hrpp_hash_floats", "hrpp_coarsen_keys", "hrpp_bvh_create", "hrpp_bvh_destroy",
                 "hrpp_bvh_ancestor_lut", "hrpp_build_bvh", "hrpp_trace_batch",
                 "hrpp_table_create", "hrpp_table_destroy", "hrpp_table_clear",
                 "hrpp_table_clear_async", "hrpp_table_info", "hrpp_table_record", "hrpp_table_lookup",
                 "hrpp_table_export", "hrpp_predict_batch", "hrpp_trace_wave",
                 "hrpp_profile_enable", "hrpp_profile_read", "hrpp_table_set_deferred",
                 "hrpp_table_pending", "hrpp_set_consult_short",
                 "hrpp_gen_primary", "hrpp_spawn", "hrpp_partition_by_owner",
                 "hrpp_profile_stages", "hrpp_pack_rays", "hrpp_unpack_rays",
                 "hrpp_pack_hits", "hrpp_unpack_hits"):
        getattr(L, name).restype = C.c_int
    return L


class _LazyLib:
    """Loads the shared library on first use, so that importing the package
    (e.g. to run the build) works before the library exists.  Any compute
    call without the library raises ImportError: there is no fallback."""

    _real = None

    def __getattr__(self, name):
        if _LazyLib._real is None:
            _LazyLib._real = _load()
        return getattr(_LazyLib._real, name)


lib = _LazyLib()

EXPORTED = ("hrpp_last_error", "hrpp_version", "hrpp_launch_count", "hrpp_device_count",
            "hrpp_hash_rays", "hrpp_hash_floats", "hrpp_coarsen_keys", "hrpp_bvh_create", "hrpp_bvh_destroy",
            "hrpp_bvh_ancestor_lut", "hrpp_build_bvh", "hrpp_trace_batch", "hrpp_table_create",
            "hrpp_table_destroy", "hrpp_table_clear", "hrpp_table_clear_async", "hrpp_table_info",
            "hrpp_table_record",
            "hrpp_table_lookup", "hrpp_table_export", "hrpp_predict_batch", "hrpp_trace_wave",
            "hrpp_set_live_rounds", "hrpp_set_fast_rounds", "hrpp_profile_enable",
            "hrpp_profile_read",
            "hrpp_table_set_deferred", "hrpp_table_pending", "hrpp_set_consult_short",
            "hrpp_gen_primary", "hrpp_spawn", "hrpp_partition_by_owner",
            "hrpp_profile_stages", "hrpp_pack_rays", "hrpp_unpack_rays", "hrpp_pack_hits",
            "hrpp_unpack_hits")

PROFILE_STAGES = ("hash", "trace", "trace_queue", "group", "consult", "commit", "other")


def profile_enable(on: bool = True, stages=None):
    """Enable the per-stage event profiler (all stages, or only the named
    ones: fewer events disturb the timed path less)."""
    if stages is None:
        lib.hrpp_profile_enable(int(bool(on)))
    else:
        mask = 0
        for k in stages:
            mask |= 1 << PROFILE_STAGES.index(k)
        lib.hrpp_profile_stages(mask if on else 0)


def profile_read(reset: bool = True) -> dict:
    """{stage: (milliseconds, launches)} accumulated since the last reset."""
    ms = np.zeros(len(PROFILE_STAGES), np.float64)
    cnt = np.zeros(len(PROFILE_STAGES), np.int64)
    lib.hrpp_profile_read(ms.ctypes.data_as(C.c_void_p), cnt.ctypes.data_as(C.c_void_p),
                          len(PROFILE_STAGES), int(bool(reset)))
    return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(PROFILE_STAGES)}


def last_error() -> str:
    return (lib.hrpp_last_error() or b"").decode("utf-8", "replace")


def check(rc: int, what: str = ""):
    """Map C-ABI status codes to the reference's exceptions (hrpp/errors.py)."""
    if rc == OK:
        return
    msg = last_error() or what
    if rc == NONFINITE:
        raise NonFiniteInput(msg)
    if rc == CAPACITY:
        raise CapacityExceeded(msg + " (override with HRPP_MAX_TABLE_ENTRIES)")
    if rc == INVALID_ARG:
        raise ValueError(msg)
    raise RuntimeError(f"CUDA error in {what}: {msg}")


def launch_count() -> int:
    return int(lib.hrpp_launch_count())


# ---------------------------------------------------------------------------
# array plumbing: numpy (host, staged by the library) or torch CUDA tensors
# (device, zero-copy)
# ---------------------------------------------------------------------------

def is_torch(a) -> bool:
    return type(a).__module__.startswith("torch")


def ptr(a):
    if a is None:
        return None
    if is_torch(a):
        return C.c_void_p(a.data_ptr())
    return a.ctypes.data_as(C.c_void_p)


_TORCH_DT = {np.float32: "float32", np.float64: "float64", np.int32: "int32",
             np.int64: "int64", np.uint8: "uint8", np.int8: "int8", np.uint64: "uint64",
             np.bool_: "bool"}


def as_array(a, dtype, like=None, shape=None):
    """Contiguous array of `dtype`, on the device if `a` is a CUDA tensor."""
    if is_torch(a):
        import torch
        tdt = getattr(torch, _TORCH_DT[dtype])
        t = a if a.dtype == tdt else a.to(dtype=tdt)
        if not t.is_contiguous():
            t = t.contiguous()
        if shape is None:
            return t
        if len(shape) == 2 and t.dim() == 2 and t.shape[1] == shape[1]:
            return t  # already (n, k): no view object per call (wave hot path)
        return t.reshape(shape)
    out = np.ascontiguousarray(a, dtype=dtype)
    return out.reshape(shape) if shape is not None else out


def empty(n, dtype, like=None, fill=None):
    if like is not None and is_torch(like):
        import torch
        tdt = getattr(torch, _TORCH_DT[dtype])
        if fill is None:
            return torch.empty(n, dtype=tdt, device=like.device)
        return torch.full((n,), fill, dtype=tdt, device=like.device)
    if fill is None:
        return np.empty(n, dtype=dtype)
    return np.full(n, fill, dtype=dtype)


def stream_of(like):
    if like is not None and is_torch(like) and like.is_cuda:
        import torch
        return C.c_void_p(torch.cuda.current_stream(like.device).cuda_stream)
    return None


def current_stream_handle(device=None):
    """torch's current CUDA stream (raw handle) if torch with CUDA is in use,
    else None (the legacy default stream)."""
    import sys
    torch = sys.modules.get("torch")
    try:
        if torch is not None and torch.cuda.is_available() and torch.cuda.is_initialized():
            return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)
    except Exception:
        pass
    return None


def device_index(like=None) -> int:
    if like is not None and is_torch(like) and like.is_cuda:
        return like.device.index or 0
    try:
        import torch
        if torch.cuda.is_available():
            return torch.cuda.current_device()
    except Exception:
        pass
    return 0
