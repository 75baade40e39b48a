"""ctypes binding of libldpc_b200.so (include/ldpc_b200.h).

There is no fallback: if the shared library is missing, or no CUDA device is
present, every decoder entry point raises RuntimeError.  Build the library
with ``python -m paper_1609_01567_b200.build`` (or __graft_entry__.build()).
"""

from __future__ import annotations

import ctypes
import os
import pathlib
import threading

_HERE = pathlib.Path(__file__).resolve().parent
# LDPC_LIB selects an alternative build of the same library (A/B layout experiments)
LIB_PATH = pathlib.Path(os.environ["LDPC_LIB"]) if os.environ.get("LDPC_LIB") else _HERE / "_native" / "libldpc_b200.so"

LDPC_OK = 0
LDPC_EINVAL = -1
LDPC_ECUDA = -2
LDPC_ENOMEM = -3
LDPC_ECLOSED = -4

FLAG_EARLY_STOP = 0
FLAG_FIXED_ITERS = 1
FLAG_FP32 = 2
FLAG_STREAMING = 4
FLAG_ONCHIP = 8
FLAG_GRID = 16

VARIABLE = 0
CHECK = 1

KCLASS = ("check", "variable", "estimate", "syndrome", "layout")

_lock = threading.Lock()
_lib = None

vp = ctypes.c_void_p
i32 = ctypes.c_int32
i64 = ctypes.c_int64
u32 = ctypes.c_uint32
sz = ctypes.c_size_t
P_i32 = ctypes.POINTER(ctypes.c_int32)
P_i64 = ctypes.POINTER(ctypes.c_int64)


class Profile(ctypes.Structure):
    """ldpc_profile: per-kernel-class event-timed ms, launches, algorithmic bytes."""

    _fields_ = [("ms", ctypes.c_double * 5), ("launches", ctypes.c_int64 * 5), ("bytes", ctypes.c_int64 * 5)]

    def as_dict(self) -> dict:
        return {k: {"ms": self.ms[i], "launches": int(self.launches[i]), "bytes": int(self.bytes[i])}
                for i, k in enumerate(KCLASS)}


def _declare(L):
    L.ldpc_last_error.restype = ctypes.c_char_p
    L.ldpc_abi_version.restype = ctypes.c_int
    L.ldpc_kernel_launches.restype = ctypes.c_int64
    L.ldpc_graph_create.argtypes = [i32, i32, i64, P_i32, P_i32, vp, ctypes.POINTER(vp)]
    L.ldpc_graph_destroy.argtypes = [vp]
    L.ldpc_graph_destroy.restype = None
    L.ldpc_graph_info.argtypes = [vp, P_i64]
    L.ldpc_graph_get_tables.argtypes = [vp, ctypes.c_int] + [P_i64] * 6
    L.ldpc_graph_get_var_groups.argtypes = [vp, P_i64, P_i64]
    L.ldpc_graph_get_buckets.argtypes = [vp, ctypes.c_int, P_i32, P_i32, i32]
    L.ldpc_workspace_bytes.argtypes = [vp, i32]
    L.ldpc_workspace_bytes.restype = sz
    L.ldpc_decode.argtypes = [vp, vp, i32, i32, u32, vp, vp, vp, vp, vp, sz, vp, ctypes.POINTER(Profile)]
    L.ldpc_count_errors.argtypes = [vp, vp, vp, vp, i32, vp, vp]
    L.ldpc_phase_to_check.argtypes = [vp, vp, vp, vp, i32, vp, sz, vp]
    L.ldpc_phase_to_variable.argtypes = [vp, vp, vp, i32, vp, sz, vp]
    L.ldpc_phase_estimate.argtypes = [vp, vp, vp, vp, i32, vp, sz, vp]
    L.ldpc_phase_syndrome.argtypes = [vp, vp, vp, i32, vp, sz, vp]
    L.ldpc_decoder_create.argtypes = [vp, i32, i32, ctypes.POINTER(vp)]
    L.ldpc_decoder_decode_host.argtypes = [vp, vp, i32, i32, u32, vp, vp, vp, vp]
    L.ldpc_decoder_submit.argtypes = [vp, vp, i32, i32, u32, vp, vp, vp, vp, P_i64]
    L.ldpc_decoder_wait.argtypes = [vp, i64]
    L.ldpc_decode_awgn.argtypes = [vp, vp, vp, i32, i32, u32, vp, vp, vp, vp, vp, sz, vp, ctypes.POINTER(Profile)]
    L.ldpc_priors_awgn.argtypes = [vp, vp, i32, i32, vp, vp]
    L.ldpc_npexp.argtypes = [vp, i64, vp, vp]
    L.ldpc_decoder_decode_awgn_host.argtypes = [vp, vp, vp, i32, i32, u32, vp, vp, vp, vp]
    L.ldpc_decoder_submit_awgn.argtypes = [vp, vp, vp, i32, i32, u32, vp, vp, vp, vp, P_i64]
    L.ldpc_decoder_destroy.argtypes = [vp]
    L.ldpc_decoder_destroy.restype = None
    u64 = ctypes.c_uint64
    L.ldpc_channel_awgn.argtypes = [u64, u64, u64, i32, i32, ctypes.c_double, vp, vp]
    L.ldpc_channel_awgn.restype = ctypes.c_int
    L.ldpc_channel_awgn_host.argtypes = [u64, u64, u64, i32, i32, ctypes.c_double, vp, i32]
    L.ldpc_channel_awgn_host.restype = ctypes.c_int
    L.ldpc_decode_channel.argtypes = [vp, u64, u64, u64, i32, ctypes.c_double, i32, u32, vp, vp, vp, vp, vp, sz, vp]
    L.ldpc_decode_channel.restype = ctypes.c_int
    L.ldpc_phase_f32.argtypes = [vp, ctypes.c_int, vp, vp, vp, i32, vp, sz, vp]
    L.ldpc_phase_f32.restype = ctypes.c_int
    L.ldpc_comm_unique_id.argtypes = [vp]
    L.ldpc_comm_create.argtypes = [i32, i32, vp, ctypes.POINTER(vp)]
    L.ldpc_allreduce_counts_i64.argtypes = [vp, vp, i32, vp]
    L.ldpc_comm_destroy.argtypes = [vp]
    L.ldpc_comm_destroy.restype = None
    L.ldpc_selftest_division.argtypes = [ctypes.c_uint64, i64, P_i64]
    L.ldpc_selftest_division.restype = ctypes.c_int
    for name in ("ldpc_graph_create", "ldpc_graph_info", "ldpc_graph_get_tables", "ldpc_graph_get_var_groups",
                 "ldpc_graph_get_buckets", "ldpc_decode", "ldpc_count_errors", "ldpc_phase_to_check",
                 "ldpc_phase_to_variable", "ldpc_phase_estimate", "ldpc_phase_syndrome", "ldpc_decoder_create",
                 "ldpc_decoder_decode_host", "ldpc_decoder_submit", "ldpc_decoder_wait", "ldpc_comm_unique_id",
                 "ldpc_comm_create", "ldpc_allreduce_counts_i64", "ldpc_decode_awgn", "ldpc_priors_awgn",
                 "ldpc_npexp", "ldpc_decoder_decode_awgn_host", "ldpc_decoder_submit_awgn"):
        getattr(L, name).restype = ctypes.c_int
    return L


def load_library():
    """Load the shared library without touching the GPU (symbols only)."""
    global _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise RuntimeError(f"CUDA extension missing: {LIB_PATH} (run python -m paper_1609_01567_b200.build)")
            _lib = _declare(ctypes.CDLL(str(LIB_PATH)))
    return _lib


def lib():
    """The library, after checking that a CUDA device is usable."""
    L = load_library()
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device: the B200 decoder has no CPU fallback")
    return L


def last_error() -> str:
    return (load_library().ldpc_last_error() or b"").decode(errors="replace")


def check(rc: int, what: str = "ldpc") -> None:
    if rc == LDPC_OK:
        return
    msg = f"{what}: {last_error()}"
    if rc == LDPC_EINVAL:
        raise ValueError(msg)
    raise RuntimeError(msg)


def current_stream_handle(device=None):
    """torch's current stream on `device` (a graph's device index or torch device; default: current)."""
    import torch

    if device is None:
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(device, int):
        device = torch.device("cuda", device)
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)
