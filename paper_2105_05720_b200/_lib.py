"""ctypes binding of libcoconet_cuda.so (include/coconet_cuda.h).

The product path has no CPU fallback: if the shared library is missing, or
was built without the CUDA entry points, importing the ops fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

PKG = Path(__file__).resolve().parent
LIB_PATH = PKG / "libcoconet_cuda.so"

F32, F16, BF16 = 0, 1, 2
SUM, MAX, MIN = 0, 1, 2
MATH_EXACT, MATH_FAST = 0, 1
ALGO_AUTO, ALGO_TWO_SHOT, ALGO_ONE_SHOT, ALGO_NVLS = 0, 1, 2, 3
HEAP_DEFAULT, HEAP_CUDAMALLOC, HEAP_CUMEM, HEAP_CUMEM_NVLS = 0, 1, 2, 3
HEAP_KINDS = {"default": HEAP_DEFAULT, "cudamalloc": HEAP_CUDAMALLOC, "cumem": HEAP_CUMEM, "nvls": HEAP_CUMEM_NVLS}
LAMB_AUTO, LAMB_GRID, LAMB_STREAMED, LAMB_TMA, LAMB_WINDOWED, LAMB_ONCHIP, LAMB_NVLS = 0, 1, 2, 3, 4, 5, 6
MODE_VIRTUAL, MODE_DISTRIBUTED = 0, 1
MAX_RANKS = 8

# status -> ccopt::ErrCode name (types.hpp:102-124); 1..20 are ErrCode+1
ERRCODE_NAMES = [
    "LayoutMismatch", "ShapeMismatch", "InvalidInput", "NotAllReduce", "NotSliceable",
    "NotAConsumer", "DependencyViolation", "NotComputation", "ChainBroken", "NotConsumer",
    "NotProducerConsumerChain", "ConsumerNotSliced", "StillLive", "NoSuchRank",
    "OperandLayoutMismatch", "DivisibilityError", "ReplicationViolation", "CandidateFailed",
    "UnknownId", "ParseError",
]


class CoconetError(RuntimeError):
    """Raised for a non-zero status; `.code` is the C status, `.name` the
    ccopt::ErrCode name where the status mirrors one."""

    def __init__(self, status: int, msg: str):
        self.code = status
        if 1 <= status <= len(ERRCODE_NAMES):
            self.name = ERRCODE_NAMES[status - 1]
        else:
            self.name = {100: "CudaError", 101: "Timeout", 102: "Unsupported", 103: "OutOfHeap"}.get(
                status, f"status{status}")
        super().__init__(f"{self.name}: {msg}")


class AdamParams(C.Structure):
    _fields_ = [("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float), ("t", C.c_float),
                ("eps", C.c_float), ("cv_beta1", C.c_int), ("math", C.c_int), ("algo", C.c_int)]


class LambParams(C.Structure):
    _fields_ = [("lr", C.c_float), ("beta1", C.c_float), ("beta2", C.c_float), ("t", C.c_float),
                ("eps", C.c_float), ("wd", C.c_float), ("math", C.c_int), ("sched", C.c_int),
                ("lag_elems", C.c_int64), ("trust_guard", C.c_int), ("pad_", C.c_int)]


class BdrParams(C.Structure):
    _fields_ = [("rate", C.c_double), ("seed", C.c_uint64), ("key", C.c_uint64), ("math", C.c_int)]


_P = C.c_void_p
_I = C.c_int
_I64 = C.c_int64
_U64 = C.c_uint64
_SZ = C.c_size_t
_PP = C.POINTER(C.c_void_p)
_PI64 = C.POINTER(C.c_int64)

_SIGNATURES = {
    "coconet_last_error": (C.c_char_p, []),
    "coconet_status_name": (C.c_char_p, [_I]),
    "coconet_init": (_I, [C.POINTER(_P), _I, _I, _I, _I, _SZ]),
    "coconet_init_ex": (_I, [C.POINTER(_P), _I, _I, _I, _I, _SZ, _I]),
    "coconet_heap_kind": (_I, [_P]),
    "coconet_nvls_supported": (_I, [_I, _I, C.c_char_p, _SZ]),
    "coconet_nvls_setup": (_I, [_P, _I]),
    "coconet_nvls_mapped": (_I, [_P]),
    "coconet_finalize": (_I, [_P]),
    "coconet_world": (_I, [_P, C.POINTER(_I), C.POINTER(_I), C.POINTER(_I)]),
    "coconet_heap_handle": (_I, [_P, _P, C.POINTER(_SZ)]),
    "coconet_open_peers": (_I, [_P, _P, _SZ]),
    "coconet_symm_alloc": (_I, [_P, _SZ, C.POINTER(_SZ)]),
    "coconet_symm_free": (_I, [_P, _SZ]),
    "coconet_symm_reset": (_I, [_P]),
    "coconet_symm_high_water": (_SZ, [_P]),
    "coconet_symm_ptr": (_P, [_P, _I, _SZ]),
    "coconet_heap_bytes": (_SZ, [_P]),
    "coconet_group_create": (_I, [_P, _I, _I, C.POINTER(_I)]),
    "coconet_check": (_I, [_P, _P]),
    "coconet_set_timeout_ms": (_I, [_P, C.c_uint32]),
    "coconet_launch_count": (_U64, [_P]),
    "coconet_gen_values": (_I, [_P, _P, _I, _U64, _U64, _I, _I, _I, _PI64, _I, _I, _P]),
    "coconet_tlist_create": (_I, [_P, _I, _I, _PI64, _I64, C.POINTER(_P)]),
    "coconet_tlist_plan": (_I, [_I, _I, _PI64, _I64, C.POINTER(_P)]),
    "coconet_tlist_destroy": (_I, [_P]),
    "coconet_tlist_shard_elems": (_I64, [_P]),
    "coconet_tlist_total": (_I64, [_P]),
    "coconet_tlist_state_elems": (_I64, [_P]),
    "coconet_tlist_buckets": (_I64, [_P]),
    "coconet_tlist_metadata_bytes": (_I64, [_P]),
    "coconet_tlist_chunk": (_I, [_P, _I, _PI64, _PI64]),
    "coconet_tlist_shard_index": (_I64, [_P, _I64]),
    "coconet_tlist_segments": (_I64, [_P, _I, _PI64, _PI64, _PI64, _PI64, _I64]),
    "coconet_tlist_stream_items": (_I64, [_P, _I64, _I, _PI64, _PI64, _PI64, _PI64, _I64]),
    "coconet_tlist_onchip_spilled": (_I64, [_P]),
    "coconet_fused_rs_adam_ag": (_I, [_P, _P, _PP, _I, _PP, _P, _P, C.POINTER(AdamParams), _P]),
    "coconet_send": (_I, [_P, _I, _I, _P, _P, _I, _I64, _P]),
    "coconet_convert": (_I, [_P, _P, _I, _P, _I, _I64, _P]),
    "coconet_unfused_lamb": (_I, [_P, _P, _PP, _I, _PP, _P, _P, _P, _P, C.POINTER(LambParams), _P]),
    "coconet_fused_rs_lamb_ag": (_I, [_P, _P, _PP, _I, _PP, _P, _P, C.POINTER(LambParams), _P]),
    "coconet_allreduce": (_I, [_P, _P, _PP, _PP, _I, _I, _I, _P]),
    "coconet_reduce_scatter": (_I, [_P, _I, _P, _P, _I, _I, _I, _PI64, _I, _P]),
    "coconet_all_gather": (_I, [_P, _I, _P, _P, _I, _I, _PI64, _I, _P]),
    "coconet_reduce": (_I, [_P, _I, _P, _P, _I, _I, _I64, _I, _P]),
    "coconet_broadcast": (_I, [_P, _I, _P, _P, _I, _I64, _I, _P]),
    "coconet_fused_rs_bdr_ag": (_I, [_P, _I, _P, _P, _P, _P, _I, _I64, _I64, C.POINTER(BdrParams), _P]),
    "coconet_rs_fused_send_ag": (_I, [_P, _I, _I, _P, _P, _P, _P, _I, _I64, C.POINTER(BdrParams), _P]),
    "coconet_matmul": (_I, [_P, _I, _P, _P, _P, _I, _I, _I64, _I64, _I64, _I, _P]),
    "coconet_mm_overlap_fused_ar": (_I, [_P, _I, _P, _P, _P, _P, _P, _P, _I, _I64, _I64, _I64,
                                         C.POINTER(BdrParams), _P]),
    # generic expression programs (driven by GpuEngine; opaque here)
    "coconet_pointwise": (_I, [_P, _I, _P, C.POINTER(C.c_double), C.POINTER(C.c_double), _P]),
    "coconet_pointwise_reduce": (_I, [_P, _I, _P, _I, _I, C.POINTER(C.c_double),
                                      C.POINTER(C.c_double), _P]),
}

_lib = None


def load(path: os.PathLike | None = None):
    """Loads the shared library (once). Raises if it is missing: there is no
    fallback implementation."""
    global _lib
    if _lib is not None:
        return _lib
    # COCONET_LIB: an alternative build of the same library (kernel variants in probes)
    p = Path(path) if path else Path(os.environ.get("COCONET_LIB", str(LIB_PATH)))
    if not p.exists():
        raise ImportError(
            f"{p} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(the CUDA path has no CPU fallback)")
    lib = C.CDLL(str(p))
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def exported_symbols() -> list[str]:
    return list(_SIGNATURES)


def last_error() -> str:
    """Thread-local message of the last failed call (coconet_last_error)."""
    return load().coconet_last_error().decode(errors="replace")


def check(status: int) -> None:
    if status != 0:
        msg = load().coconet_last_error().decode(errors="replace")
        raise CoconetError(status, msg)


def ptr_array(ptrs) -> C.Array:
    return (C.c_void_p * len(ptrs))(*ptrs)


def i64_array(vals) -> C.Array:
    arr = (C.c_int64 * len(vals))()
    for i, v in enumerate(vals):
        arr[i] = int(v)
    return arr
