"""The debug entry points behind the round-2 measurements keep working:
ssb_debug_attn_trace records CTA 0's timeline of the prefill attention pair
kernel (tools/attn_trace.py) without changing its output, and
ssb_debug_read_stream (tools/read_bw.py) streams a buffer and reports
argument errors."""

from __future__ import annotations

import ctypes

import numpy as np
import pytest
import torch

from paper_2503_06433_b200 import _lib, ops

pytestmark = pytest.mark.gpu


def test_attention_trace_records_every_role_and_keeps_the_output(cuda):
    lens, nq, nk, d = [256, 128], 8, 2, 128
    T = sum(lens)
    g = torch.Generator(device=cuda).manual_seed(5)
    qkv = torch.randn(T, (nq + 2 * nk) * d, device=cuda, generator=g).to(torch.bfloat16)
    cu = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int32, device=cuda)
    ref = torch.empty(T, nq * d, dtype=torch.bfloat16, device=cuda)
    ops.prefill_attention(qkv, nq, nk, d, cu, max(lens), ref, d ** -0.5)
    buf = torch.zeros(5 * 4096, dtype=torch.int64, device=cuda)
    lib = _lib.load()
    assert lib.ssb_debug_attn_trace(ctypes.c_void_p(buf.data_ptr())) == 0
    try:
        out = torch.empty_like(ref)
        ops.prefill_attention(qkv, nq, nk, d, cu, max(lens), out, d ** -0.5)
        torch.cuda.synchronize()
    finally:
        lib.ssb_debug_attn_trace(None)
    assert torch.equal(out, ref)
    raw = buf.cpu().numpy().astype(np.uint64).reshape(5, 4096)
    for role in range(5):  # producer K, producer V, MMA issuer, softmax A, softmax B
        entries = raw[role][raw[role] != 0]
        assert entries.size > 0, role
        t = entries >> np.uint64(24)
        assert np.all(np.diff(t.astype(np.int64)) >= 0), role  # one thread per role: time-ordered


def test_read_stream_runs_and_rejects_bad_arguments(cuda):
    lib = _lib.load()
    x = torch.zeros(1 << 24, dtype=torch.uint8, device=cuda)
    stream = torch.cuda.current_stream().cuda_stream
    assert lib.ssb_debug_read_stream(x.data_ptr(), x.numel(), 2, 32768, 3, stream) == 0
    torch.cuda.synchronize()
    assert lib.ssb_debug_read_stream(x.data_ptr(), x.numel(), 2, 100, 3, stream) < 0  # chunk % 16
    assert b"bad arguments" in lib.ssb_last_error()
