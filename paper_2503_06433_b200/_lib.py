"""ctypes binding of libseesaw_b200.so (the C ABI in include/seesaw_b200.h).

The product path has no fallback: if the library is missing or a call fails,
:class:`SeesawKernelError` is raised with the library's own error text.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

# SSB_LIB: an A/B build of the same library (tools/build_ab_lib.py)
LIB_PATH = Path(os.environ.get("SSB_LIB") or Path(__file__).resolve().parent / "libseesaw_b200.so").resolve()

SSB_EPI_NONE = 0
SSB_EPI_RESIDUAL = 1
SSB_EPI_SILU_MUL = 2
SSB_EPI_F32 = 3
SSB_EPI_ROPE_KV = 4
SSB_GEMM_MC1 = 1 << 16
SSB_GEMM_MC2 = 1 << 17
SSB_GEMM_2SM = 1 << 18
SSB_GEMM_SPLIT_SHIFT = 20
SSB_GEMM_TAIL = 1 << 28
SSB_GEMM_STREAMK = 1 << 29
SSB_MAX_PEERS = 64


class SeesawKernelError(RuntimeError):
    """A libseesaw_b200 call returned a non-zero status."""


class KVGeometry(ctypes.Structure):
    _fields_ = [
        ("n_layers", ctypes.c_int),
        ("n_heads", ctypes.c_int),
        ("block_size", ctypes.c_int),
        ("head_dim", ctypes.c_int),
    ]


class CopyDesc(ctypes.Structure):
    _fields_ = [
        ("src_off", ctypes.c_int64),
        ("dst_off", ctypes.c_int64),
        ("src_stride", ctypes.c_int64),
        ("dst_stride", ctypes.c_int64),
        ("cum_bytes", ctypes.c_int64),
        ("rows", ctypes.c_int32),
        ("row_bytes", ctypes.c_int32),
    ]


class RowNorm(ctypes.Structure):
    """ssb_rownorm (include/seesaw_b200.h): RMSNorm folded into the GEMMs."""

    _fields_ = [
        ("ss_out", ctypes.c_void_p),
        ("ss_in", ctypes.c_void_p),
        ("ss_in_parts", ctypes.c_int),
        ("hidden", ctypes.c_int),
        ("eps", ctypes.c_float),
        ("ss_parts", ctypes.c_int),
    ]


_P = ctypes.c_void_p
_PRN = ctypes.POINTER(RowNorm)
_I = ctypes.c_int
_I64 = ctypes.c_int64
_F = ctypes.c_float
_PI32 = ctypes.POINTER(ctypes.c_int32)
_PI64 = ctypes.POINTER(ctypes.c_int64)
_PU64 = ctypes.POINTER(ctypes.c_uint64)

# name -> argtypes (restype is int for all compute entry points)
SIGNATURES: dict[str, list] = {
    "ssb_gemm_bf16": [_P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _I, _I, _I, _P],
    "ssb_gemm_bf16_ws": [_P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _I, _I, _I, _P, _I64, _P],
    "ssb_gemm_bf16_rn": [_P, _P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _I, _I, _I, _P, _I64, _PRN, _P],
    "ssb_gemm_qkv_rope_kv": [_P, _P, _P, _I, _I, _I, _I, _I, _I, _I, _I, _P, _P, _P, _I, _P, KVGeometry, _I, _P,
                             _I, _I, _P, _I64, _PRN, _P],
    "ssb_gemm_lm_head_argmax": [_P, _P, _I, _I, _I, _I, _I, _I, _P, _I, _I, _P, _I64, _PRN, _P],
    "ssb_argmax_keys_decode": [_P, _I, _P, _P, _P],
    "ssb_kv_reshard_pack": [_P, KVGeometry, _P, _I, _I, _PI32, _PI32, _PI32, _PI32, _PI64, _P, _P],
    "ssb_kv_reshard_pack_p2p": [_P, KVGeometry, _P, _I, _I, _PI32, _PI32, _PI32, _PI32, _PI64, _P],
    "ssb_kv_reshard_unpack": [_P, KVGeometry, _P, _I, _I, _PI32, _PI32, _PI32, _PI32, _PI64, _P, _P],
    "ssb_copy2d_batched": [_P, _P, _P, _I, _I64, _P],
    "ssb_init_weights": [_P, _P, _I, _I64, ctypes.c_uint64, _P],
    "ssb_kv_hnd_copy": [_I, _P, KVGeometry, _P, _I, _I, _I, _I, _I, _I, _P, _P],
    "ssb_memcpy2d_async": [_P, _I64, _P, _I64, _I64, _I64, _P],
    "ssb_rmsnorm": [_P, _I, _P, _P, _P, _I, _I, _I, _F, _P],
    "ssb_decode_positions": [_P, _P, _I, _I, _P, _P, _I, _P],
    "ssb_rope_kv_append": [_P, _I, _I, _I, _I, _P, _P, _P, _I, _P, KVGeometry, _I, _P, _P],
    "ssb_embedding": [_P, _I, _P, _I, _I, _I, _P, _I, _P],
    "ssb_argmax_rows": [_P, _I, _I, _I, _I, _P, _P, _P],
    "ssb_argmax_combine": [_P, _P, _I, _I, _P, _P],
    "ssb_prefill_attention": [_P, _I, _I, _I, _I, _I, _P, _I, _I, _P, _I, _F, _I, _P],
    "ssb_decode_attention": [_P, _I, _I, _I, _P, KVGeometry, _I, _I, _P, _I, _P, _I, _P, _I, _F, _P],
    "ssb_tp_allreduce_rmsnorm": [_PU64, _PU64, _PU64, _PU64, _I, _I, _I, _I, _I, _P, _F, ctypes.c_uint32, _I, _P,
                                 _P],
    "ssb_tp_allreduce_rowss": [_PU64, _PU64, _PU64, _PU64, _I, _I, _I, _I, _I, ctypes.c_uint32, _I, _P, _P],
    "ssb_debug_read_stream": [_P, _I64, _I, _I, _I, _P],
    "ssb_tp_argmax_keys": [_PU64, _PU64, _I, _I, _I, _P, ctypes.c_uint32, _I, _P, _P],
}

_lock = threading.Lock()
_lib: ctypes.CDLL | None = None


def load() -> ctypes.CDLL:
    """Load the library once; raise if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise SeesawKernelError(
                    f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)"
                )
            lib = ctypes.CDLL(str(LIB_PATH))
            lib.ssb_last_error.restype = ctypes.c_char_p
            lib.ssb_last_error.argtypes = []
            lib.ssb_version.restype = ctypes.c_int
            lib.ssb_device_sm_count.restype = ctypes.c_int
            lib.ssb_set_pdl.restype = ctypes.c_int
            lib.ssb_set_pdl.argtypes = [_I]
            if hasattr(lib, "ssb_debug_attn_trace"):  # absent from older A/B builds (SSB_LIB)
                lib.ssb_debug_attn_trace.restype = ctypes.c_int
                lib.ssb_debug_attn_trace.argtypes = [_P]
            lib.ssb_ipc_export.restype = ctypes.c_int
            lib.ssb_ipc_export.argtypes = [_P, _P, ctypes.POINTER(ctypes.c_int64)]
            lib.ssb_ipc_open.restype = ctypes.c_int
            lib.ssb_ipc_open.argtypes = [_P, _I, ctypes.POINTER(ctypes.c_void_p)]
            lib.ssb_ipc_close.restype = ctypes.c_int
            lib.ssb_ipc_close.argtypes = [_P, _I]
            lib.ssb_gemm_plan.restype = ctypes.c_int64
            lib.ssb_gemm_plan.argtypes = [_I, _I, _I, _I, _I, _I64, _PI32]
            lib.ssb_tp_signal_bytes.restype = ctypes.c_size_t
            lib.ssb_tp_signal_bytes.argtypes = []
            for name, args in SIGNATURES.items():
                if name.startswith("ssb_debug_") and not hasattr(lib, name):
                    continue  # older A/B builds (SSB_LIB) lack the debug entry points
                fn = getattr(lib, name)
                fn.argtypes = args
                fn.restype = ctypes.c_int
            _lib = lib
    return _lib


class LaunchStats:
    """Counts library launches; optionally brackets each with CUDA events
    (bench.py's per-kernel timing inside the timed region)."""

    def __init__(self) -> None:
        self.count = 0
        self.timing = False
        self.records: list = []   # (tag, start_event, end_event, flops, bytes)
        self.tagger = None        # fn(name, args) -> (tag, flops, bytes)


STATS = LaunchStats()


def call(name: str, *args) -> None:
    lib = load()
    st = STATS
    st.count += 1
    if st.timing:
        import torch

        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        rc = getattr(lib, name)(*args)
        e.record()
        tag = st.tagger(name, args) if st.tagger else (name, 0, 0)
        st.records.append((tag[0], s, e, tag[1], tag[2]))
    else:
        rc = getattr(lib, name)(*args)
    if rc != 0:
        msg = lib.ssb_last_error().decode(errors="replace")
        raise SeesawKernelError(f"{name} failed ({rc}): {msg}")


def int32_array(values) -> ctypes.Array:
    vals = list(values)
    return (ctypes.c_int32 * max(len(vals), 1))(*vals)


def int64_array(values) -> ctypes.Array:
    vals = list(values)
    return (ctypes.c_int64 * max(len(vals), 1))(*vals)


def uint64_array(values) -> ctypes.Array:
    vals = [int(v) for v in values]
    return (ctypes.c_uint64 * max(len(vals), 1))(*vals)
