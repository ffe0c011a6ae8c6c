"""ctypes binding of the C ABI in include/decplane_b200.h.

The shared library is built in-tree by `build.py` (nvcc, sm_100a).  There is
no fallback: if the library or a CUDA device is missing, every entry point
raises `NativeUnavailable`.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DP_LIB") or os.path.join(_HERE, "_lib", "libdecplane_b200.so")   # DP_LIB: tools / A-B variants

DP_OK, DP_ERR_ARG, DP_ERR_CUDA, DP_ERR_UNSUPPORTED, DP_ERR_CAPACITY = 0, -1, -2, -3, -4
DP_F32, DP_BF16 = 0, 1
FLAG_EOS = 0x01
FLAG_ACCEPTED_HOT = 0x02
FLAG_NEAR_BOUNDARY = 0x04
FLAG_REJECTED = 0x08
FLAG_PEN_OVERFLOW = 0x40
FLAG_DEGENERATE = 0x80
PLAN_FORCE_RESUM = 0x1
PLAN_NO_PERSIST = 0x2
PLAN_FORCE_PERSIST = 0x4
PLAN_HOT_SORT = 0x8
PLAN_HOT_SORT_ALL = 0x10

EXPORTS = [
    "dp_version", "dp_device_check", "dp_last_error", "dp_uniforms", "dp_sample_full",
    "dp_row_summary", "dp_sample_shvs", "dp_penalty_update", "dp_penalty_reset",
    "dp_ready_rows", "dp_synth_logits", "dp_hot_mass_curve", "dp_row_summary_raw", "dp_sample_shvs_split",
    "dp_stage_hot", "dp_sample_full_sharded", "dp_workspace_len", "dp_encode_decisions",
    "dp_nccl_available", "dp_nccl_unique_id", "dp_nccl_comm_init", "dp_nccl_comm_destroy", "dp_allgather_tokens",
]


class NativeUnavailable(RuntimeError):
    """The sm_100a library (or a CUDA device) is not available."""


class NativeError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        super().__init__(f"{where} failed with status {status}: {detail}")
        self.status = status


class Params(C.Structure):
    """dp_params_t == core.SamplingParams (core.py:23-34)."""

    _fields_ = [
        ("temperature", C.c_double), ("top_k", C.c_int32), ("reserved", C.c_int32),
        ("top_p", C.c_double), ("min_p", C.c_double), ("rep_penalty", C.c_double),
        ("presence_penalty", C.c_double), ("frequency_penalty", C.c_double), ("seed", C.c_uint64),
    ]


class Penalty(C.Structure):
    """dp_penalty_t: the sparse device SequenceState table (core.py:100-169)."""

    _fields_ = [
        ("ids", C.c_void_p), ("out_count", C.c_void_p), ("len", C.c_void_p),
        ("prompt_len", C.c_void_p), ("cap", C.c_int32), ("vocab_size", C.c_int32),
        ("max_len", C.c_int32), ("reserved", C.c_int32),
    ]


class Debug(C.Structure):
    _fields_ = [
        ("topk_ids", C.c_void_p), ("topk_ready", C.c_void_p), ("topk_stride", C.c_int32),
        ("reserved", C.c_int32), ("margin", C.c_void_p), ("kept", C.c_void_p),
        ("alpha", C.c_void_p), ("bytes_touched", C.c_void_p), ("stats", C.c_void_p),
    ]


class Plan(C.Structure):
    _fields_ = [("max_top_k", C.c_int32), ("split", C.c_int32), ("threads", C.c_int32),
                ("summary_raw", C.c_int32), ("min_top_k", C.c_int32), ("kernel", C.c_int32),
                ("fuse_update", C.c_int32), ("flags", C.c_int32),
                ("workspace", C.c_void_p), ("workspace_len", C.c_int64)]


assert C.sizeof(Params) == 64
assert C.sizeof(Penalty) == 48
assert C.sizeof(Plan) == 48

_P, _I64, _U64, _I32, _D = C.c_void_p, C.c_int64, C.c_uint64, C.c_int32, C.c_double
_SIGS = {
    "dp_version": ([], C.c_int),
    "dp_device_check": ([C.c_int], C.c_int),
    "dp_last_error": ([], C.c_char_p),
    "dp_workspace_len": ([_I64], C.c_int64),
    "dp_encode_decisions": ([_P, _P, _P, _P, _I64, _P, _P], C.c_int),
    "dp_uniforms": ([_P, _P, _I64, _U64, _P, _P], C.c_int),
    "dp_sample_full": ([_P, C.c_int, _I64, _I64, _I64, _P, C.POINTER(Penalty), _P, _P, _U64,
                        _P, _P, _P, C.POINTER(Debug), C.POINTER(Plan), _P], C.c_int),
    "dp_row_summary": ([_P, C.c_int, _I64, _I64, _I64, _P, C.POINTER(Penalty), _P, _P, _P, _P], C.c_int),
    "dp_row_summary_raw": ([_P, C.c_int, _I64, _I64, _I64, _P, _P, _P, _P], C.c_int),
    "dp_sample_shvs": ([_P, C.c_int, _I64, _I64, _I64, _I64, _P, _P, _P, _P, _P, C.POINTER(Penalty),
                        _P, _P, _U64, _P, _P, _P, C.POINTER(Debug), C.POINTER(Plan), _P, _P], C.c_int),
    "dp_sample_shvs_split": ([_P, _I64, _P, _I64, C.c_int, _I64, _I64, _I64, _P, _P, _P, _P, _P, C.POINTER(Penalty),
                              _P, _P, _U64, _P, _P, _P, C.POINTER(Debug), C.POINTER(Plan), _P, _P], C.c_int),
    "dp_sample_full_sharded": ([C.POINTER(C.c_void_p), C.c_int32, C.c_int, _I64, _I64, _I64, _P,
                                C.POINTER(Penalty), _P, _P, _U64, _P, _P, _P, C.POINTER(Debug), C.POINTER(Plan),
                                _P], C.c_int),
    "dp_stage_hot": ([_P, _I64, C.c_int, _I64, _I64, _P, _I64, _P], C.c_int),
    "dp_penalty_update": ([C.POINTER(Penalty), _P, _I64, _P, _P], C.c_int),
    "dp_penalty_reset": ([C.POINTER(Penalty), _I64, _P], C.c_int),
    "dp_ready_rows": ([_P, C.c_int, _I64, _I64, _I64, _P, C.POINTER(Penalty), _P, _P], C.c_int),
    "dp_synth_logits": ([_P, _D, _U64, _U64, _P, _I64, _I64, _I64, _P, C.c_int, _P, _P, _P, _P, _P], C.c_int),
    "dp_nccl_available": ([], C.c_int),
    "dp_nccl_unique_id": ([_P], C.c_int),
    "dp_nccl_comm_init": ([C.POINTER(C.c_void_p), _I32, _P, _I32], C.c_int),
    "dp_nccl_comm_destroy": ([_P], C.c_int),
    "dp_allgather_tokens": ([_P, _P, _I64, _P, _P], C.c_int),
    "dp_hot_mass_curve": ([_P, C.c_int, _I64, _I64, _I64, _P, _P, _P, C.POINTER(Penalty), _P, _P, _P, _I32,
                           _P, _P], C.c_int),
}

_lock = threading.Lock()
_lib = None


def load(path: str = LIB_PATH) -> C.CDLL:
    """Load the library (no device needed).  Raises NativeUnavailable if absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise NativeUnavailable(
                f"{path} is missing: build it with `python build.py` (nvcc, sm_100a). "
                "There is no CPU fallback for the decision plane.")
        # torch first: its libnccl.so.2 (DT_NEEDED of libtorch_cuda) must be the
        # process's copy before the library resolves NCCL (collective.cu reuses
        # an already-loaded libnccl.so.2; loading the system one first would
        # break a later `import torch` with a different NCCL version)
        import torch  # noqa: F401

        lib = C.CDLL(path)
        for name, (args, res) in _SIGS.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
        return lib


def check(status: int, where: str) -> None:
    if status != DP_OK:
        raise NativeError(status, where, load().dp_last_error().decode(errors="replace"))


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)


def require_device(device) -> None:
    """Fail loudly unless `device` is a CUDA sm_100 device."""
    import torch

    if not torch.cuda.is_available():
        raise NativeUnavailable("no CUDA device: the decision plane runs only on B200 (sm_100a)")
    idx = torch.device(device).index
    check(load().dp_device_check(torch.cuda.current_device() if idx is None else idx), "dp_device_check")
