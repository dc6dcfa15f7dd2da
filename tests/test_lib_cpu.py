"""The C-ABI library loads without a GPU and exports every symbol the public
header declares; argument errors come back as negative codes with a message
(no GPU work is issued by these calls)."""

from __future__ import annotations

import ctypes
import re
from pathlib import Path

import pytest

from paper_2503_06433_b200 import _lib

HEADER = Path(__file__).resolve().parent.parent / "include" / "seesaw_b200.h"


def declared_functions() -> list[str]:
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ssb_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    names = declared_functions()
    assert "ssb_gemm_bf16" in names and "ssb_kv_reshard_pack" in names and len(names) >= 15


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, f"missing exports: {missing}"
    assert lib.ssb_version() == 1


def test_ctypes_signatures_cover_header():
    declared = set(declared_functions())
    bound = set(_lib.SIGNATURES) | {"ssb_last_error", "ssb_version", "ssb_device_sm_count", "ssb_gemm_plan",
                                    "ssb_tp_signal_bytes", "ssb_set_pdl", "ssb_ipc_export", "ssb_ipc_open", "ssb_debug_attn_trace",
                                    "ssb_ipc_close"}
    assert declared == bound


def test_ipc_entry_points_reject_null_arguments():
    """The CUDA IPC mapping calls (comm.TorchComm.peer_addresses) report a
    null argument as an error code, without touching a device."""
    lib = _lib.load()
    out = ctypes.c_void_p(0)
    assert lib.ssb_ipc_open(None, 0, ctypes.byref(out)) < 0
    assert b"null" in lib.ssb_last_error()
    off = ctypes.c_int64(0)
    assert lib.ssb_ipc_export(None, None, ctypes.byref(off)) < 0


def test_argument_errors_are_reported_not_raised():
    lib = _lib.load()
    rc = lib.ssb_gemm_bf16(None, None, None, None, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, None)
    assert rc < 0
    assert b"empty problem" in lib.ssb_last_error()
    with pytest.raises(_lib.SeesawKernelError, match="n_peers"):
        geo = _lib.KVGeometry(1, 1, 64, 128)
        arr = _lib.int32_array([0])
        p32 = ctypes.cast(arr, ctypes.POINTER(ctypes.c_int32))
        p64 = ctypes.cast(_lib.int64_array([0]), ctypes.POINTER(ctypes.c_int64))
        _lib.call("ssb_kv_reshard_pack", None, geo, None, 1, 0, p32, p32, p32, p32, p64, None, None)


def test_struct_layouts_match_header():
    """ctypes mirrors of the header's structs: sizes and field offsets as a
    C compiler lays them out (x86-64 / aarch64 LP64)."""
    import ctypes

    assert ctypes.sizeof(_lib.RowNorm) == 32
    assert _lib.RowNorm.ss_in.offset == 8 and _lib.RowNorm.ss_in_parts.offset == 16
    assert _lib.RowNorm.eps.offset == 24 and _lib.RowNorm.ss_parts.offset == 28
    assert ctypes.sizeof(_lib.CopyDesc) == 48


def test_rownorm_and_tp_combine_argument_errors():
    lib = _lib.load()
    rn = _lib.RowNorm(None, 1, 0, 0, 0.0, 0)  # ss_in without parts
    import ctypes

    rc = lib.ssb_gemm_bf16_rn(16, 16, 16, None, 128, 128, 64, 64, 64, 128, 0, 0, 0, 0, None, 0, ctypes.byref(rn),
                              None)
    assert rc < 0 and b"ss_in" in lib.ssb_last_error()
    # two barrier phases x 512 CTAs x 8 ranks, then 512 per-CTA epoch counters
    assert lib.ssb_tp_signal_bytes() == (2 * 512 * 8 + 512) * 4
    addrs = _lib.uint64_array([16, 32])
    rc = lib.ssb_tp_allreduce_rmsnorm(addrs, addrs, None, addrs, 9, 0, 4, 256, 256, None, 1e-5, 1, 4, None, None)
    assert rc < 0 and b"nranks" in lib.ssb_last_error()
    rc = lib.ssb_tp_allreduce_rmsnorm(addrs, addrs, None, addrs, 2, 0, 4, 250, 256, None, 1e-5, 0, 4, None, None)
    assert rc < 0 and b"hidden" in lib.ssb_last_error()
    rc = lib.ssb_tp_argmax_keys(addrs, addrs, 2, 3, 4, None, 0, 4, None, None)
    assert rc < 0 and b"rank" in lib.ssb_last_error()
    rc = lib.ssb_tp_argmax_keys(addrs, addrs, 2, 0, 4, None, 0, 4, None, None)
    assert rc < 0 and b"null" in lib.ssb_last_error()


def test_tp_arena_cache_grows_collectively(monkeypatch):
    """tpcombine.get_arena: one arena per (TP group, hidden), rebuilt only to
    grow (power-of-two rows, never below 256), and an arena whose self-test
    failed is remembered as unusable (every later call falls back)."""
    from paper_2503_06433_b200 import tpcombine

    built = []

    class FakeArena:
        def __init__(self, comm, device, hidden, rows, max_blocks):
            self.rows, self.usable = rows, comm != "bad"
            built.append(rows)

    monkeypatch.setattr(tpcombine, "PeerArena", FakeArena)
    cache: dict = {}
    a = tpcombine.get_arena(cache, "grp", None, 4096, 100, 16)
    assert a.rows == 256 and built == [256]
    assert tpcombine.get_arena(cache, "grp", None, 4096, 256, 16) is a
    b = tpcombine.get_arena(cache, "grp", None, 4096, 300, 16)
    assert b.rows == 512 and built == [256, 512]
    assert tpcombine.get_arena(cache, "grp", None, 4096, 17, 16) is b
    assert tpcombine.get_arena(cache, "bad", None, 4096, 10, 16) is None
    assert tpcombine.get_arena(cache, "bad", None, 4096, 10, 16) is None and built == [256, 512, 256]
