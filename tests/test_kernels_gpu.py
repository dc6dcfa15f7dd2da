"""Per-kernel numerics on the B200: each sm_100a kernel against a plain
PyTorch fp32 reference (floating point) or the CPU oracle (bit-exact init,
copies, index work)."""

from __future__ import annotations

import math

import numpy as np
import pytest
import torch

from oracle import llama as lo
from paper_2503_06433_b200 import PRESETS, ops
from paper_2503_06433_b200.layout import weight_layout
from paper_2503_06433_b200.runtime import _copy_desc_rows, init_segment_table, rope_tables

pytestmark = pytest.mark.gpu


def test_init_weights_bit_exact_vs_oracle(cuda):
    arch = PRESETS["tiny"]
    wl = weight_layout(arch, 2, 1, 1)  # TP rank 1: sliced + interleaved segments
    table, total = init_segment_table(wl)
    arena = torch.zeros(wl.arena_elems, dtype=torch.bfloat16, device=cuda)
    ops.init_weights(arena, torch.from_numpy(table).to(cuda), total, 0)
    got = arena.float().cpu().numpy()
    oa = lo.Arch(arch.num_layers, arch.hidden, arch.num_query_heads, arch.num_kv_heads, arch.head_dim, arch.ffn,
                 arch.vocab, arch.rope_theta)
    specs = lo.tensor_specs(oa)
    for t in wl.tensors.values():
        loc = got[t.offset : t.offset + t.numel].reshape(t.rows, t.cols)
        for s in t.segments:
            full = lo.init_tensor(0, specs[s.logical])
            np.testing.assert_array_equal(loc[s.dst_row : s.dst_row + s.rows, s.dst_col : s.dst_col + s.cols],
                                          full[s.row0 : s.row0 + s.rows, s.col0 : s.col0 + s.cols])


def test_copy2d_batched(cuda):
    src = torch.arange(4096, dtype=torch.int16, device=cuda)
    dst = torch.zeros(4096, dtype=torch.int16, device=cuda)
    # (src_off, dst_off, src_stride, dst_stride, rows, row_bytes) in bytes
    entries = [(0, 1024, 256, 64, 4, 64), (2048, 0, 32, 32, 16, 32), (4096, 4096, 128, 256, 3, 128)]
    d, tot = _copy_desc_rows(entries)
    ops.copy2d_batched(src, dst, torch.from_numpy(d).to(cuda), tot)
    s = src.cpu().numpy().view(np.uint8)
    exp = np.zeros(8192, np.uint8)
    for so, do, ss, ds, rows, rb in entries:
        for r in range(rows):
            exp[do + r * ds : do + r * ds + rb] = s[so + r * ss : so + r * ss + rb]
    np.testing.assert_array_equal(dst.cpu().numpy().view(np.uint8), exp)


def test_rmsnorm_and_gather(cuda):
    x = torch.randn(37, 4096, device=cuda).to(torch.bfloat16)
    w = (1 + 0.1 * torch.randn(4096, device=cuda)).to(torch.bfloat16)
    out = ops.rmsnorm(x, w, 1e-5)
    xf = x.float()
    ref = xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + 1e-5) * w.float()
    assert (out.float() - ref).abs().max().item() < 0.02
    idx = torch.tensor([36, 0, 5], dtype=torch.int32, device=cuda)
    g = ops.rmsnorm(x, w, 1e-5, row_idx=idx)
    assert torch.equal(g, out[idx.long()])


def test_rope_and_paged_append(cuda):
    arch = PRESETS["llama3-8b"]
    nq, nk, d, T = 8, 2, 128, 70
    cos, sin = rope_tables(arch, 256)
    tc, ts = torch.from_numpy(cos).to(cuda), torch.from_numpy(sin).to(cuda)
    qkv = torch.randn(T, (nq + 2 * nk) * d, device=cuda).to(torch.bfloat16)
    orig = qkv.clone()
    pos = torch.arange(T, dtype=torch.int32, device=cuda) + 5
    L, NB, BS = 3, 6, 64
    pool = torch.zeros(NB * L * 2 * nk * BS * d, dtype=torch.bfloat16, device=cuda)
    blocks = [4, 1]
    slots = torch.tensor([blocks[t // BS] * BS + t % BS for t in range(T)], dtype=torch.int64, device=cuda)
    ops.rope_kv_append(qkv, nq, nk, pos, tc, ts, pool, (L, nk, BS, d), 2, slots)
    # reference rotate-half
    x = orig.float().view(T, nq + 2 * nk, d)
    c = tc[pos.long()][:, None, :]
    s = ts[pos.long()][:, None, :]
    x1, x2 = x[..., : d // 2], x[..., d // 2 :]
    rot = torch.cat([x1 * c - x2 * s, x2 * c + x1 * s], -1)
    got = qkv.float().view(T, nq + 2 * nk, d)
    assert (got[:, : nq + nk] - rot[:, : nq + nk]).abs().max().item() < 0.05
    assert torch.equal(got[:, nq + nk :], x[:, nq + nk :])
    P = pool.view(NB, L, 2, nk, BS, d)
    for t in range(T):
        b, o = blocks[t // BS], t % BS
        assert torch.equal(P[b, 2, 0, :, o], qkv.view(T, -1, d)[t, nq : nq + nk])
        assert torch.equal(P[b, 2, 1, :, o], qkv.view(T, -1, d)[t, nq + nk :])


@pytest.mark.parametrize("flag", ["auto", "b128", "b256_2sm", "split3", "split3_2sm", "sk128", "sk256_2sm"])
@pytest.mark.parametrize("M,nq,nk,K,neg", [(300, 8, 2, 512, False), (512, 32, 8, 4096, False),
                                           (129, 4, 1, 1024, True), (64, 32, 8, 256, True)])
def test_qkv_gemm_rope_kv_fused_bit_exact(cuda, M, nq, nk, K, neg, flag):
    """The QKV GEMM with RoPE + paged K/V append in its epilogue equals the
    unfused gemm -> rope_kv_append pair bit for bit (qkv buffer and pool),
    for every tile/cluster/split configuration."""
    from paper_2503_06433_b200._lib import SSB_GEMM_2SM, SSB_GEMM_SPLIT_SHIFT, SSB_GEMM_STREAMK as SK

    bn = {"auto": 0, "b128": 128, "b256_2sm": 256 | SSB_GEMM_2SM, "split3": 128 | (3 << SSB_GEMM_SPLIT_SHIFT),
          "split3_2sm": 256 | SSB_GEMM_2SM | (3 << SSB_GEMM_SPLIT_SHIFT), "sk128": 128 | SK,
          "sk256_2sm": 256 | SSB_GEMM_2SM | SK}[flag]
    arch = PRESETS["llama3-8b"]
    d = 128
    cos, sin = rope_tables(arch, 2048)
    tc, ts = torch.from_numpy(cos).to(cuda), torch.from_numpy(sin).to(cuda)
    g = torch.Generator(device="cuda").manual_seed(M + K)
    a = torch.randn(M, K, device=cuda, generator=g).to(torch.bfloat16)
    w = (torch.randn((nq + 2 * nk) * d, K, device=cuda, generator=g) / K**0.5).to(torch.bfloat16)
    pos = torch.randint(0, 2000, (M,), dtype=torch.int32, device=cuda, generator=g)
    L, BS = 3, 64
    NB = -(-M // BS) + 3
    perm = torch.randperm(NB * BS, device=cuda, generator=g)[:M]
    slots = perm.to(torch.int64)
    if neg:
        slots[::7] = -1
    geo = (L, nk, BS, d)
    ws = torch.zeros(64 << 20, dtype=torch.uint8, device=cuda)
    pool_a = torch.zeros(NB * L * 2 * nk * BS * d, dtype=torch.bfloat16, device=cuda)
    pool_b = torch.zeros_like(pool_a)
    if flag == "auto":  # the unfused reference runs the plan the fused launch picks (same fp32 sums)
        from paper_2503_06433_b200._lib import SSB_EPI_ROPE_KV

        from paper_2503_06433_b200._lib import SSB_GEMM_STREAMK, SSB_GEMM_TAIL

        (mode, pbn, sp), _ = ops.gemm_plan(M, w.shape[0], K, SSB_EPI_ROPE_KV, 0, ws.numel())
        ref_bn = pbn | (SSB_GEMM_2SM if mode == 2 else 0) | (abs(sp) << SSB_GEMM_SPLIT_SHIFT if abs(sp) > 1 else 0)
        ref_bn |= SSB_GEMM_TAIL if sp < 0 else 0
        ref_bn |= SSB_GEMM_STREAMK if sp == 0 else 0
    else:
        ref_bn = bn
    ref = ops.gemm(a, w, workspace=ws, block_n=ref_bn)
    ops.rope_kv_append(ref, nq, nk, pos, tc, ts, pool_a, geo, 1, slots)
    got = torch.empty_like(ref)
    ops.gemm_qkv_rope_kv(a, w, got, nq, nk, pos, tc, ts, pool_b, geo, 1, slots, block_n=bn, workspace=ws)
    torch.cuda.synchronize()
    assert torch.equal(got, ref)
    assert torch.equal(pool_a, pool_b)


@pytest.mark.parametrize("M,N,K", [(512, 16032, 4096), (7, 1000, 256), (300, 128256, 512), (129, 4000, 1024)])
def test_lm_head_argmax_fused(cuda, M, N, K):
    """LM head with the argmax in the GEMM epilogue == fp32 logits + argmax_rows
    (same values, smallest index on ties; duplicated weight rows force ties)."""
    g = torch.Generator(device="cuda").manual_seed(M * N)
    h = torch.randn(M, K, device=cuda, generator=g).to(torch.bfloat16)
    w = (torch.randn(N, K, device=cuda, generator=g) / K**0.5).to(torch.bfloat16)
    w[N // 2] = w[N // 3]  # exact ties between two columns
    w[N - 1] = w[5]
    h[0] = 0  # an all-zero row: every logit ties at 0 -> index 0
    ws = torch.zeros(64 << 20, dtype=torch.uint8, device=cuda)
    base = 1000
    logits = ops.gemm(h, w, out_f32=True, workspace=ws)
    v_ref = torch.empty(M, dtype=torch.float32, device=cuda)
    i_ref = torch.empty(M, dtype=torch.int32, device=cuda)
    ops.argmax_rows(logits, base, v_ref, i_ref)
    v = torch.empty_like(v_ref)
    i = torch.empty_like(i_ref)
    ops.lm_head_argmax(h, w, base, v, i, workspace=ws)
    torch.cuda.synchronize()
    assert torch.equal(i, i_ref)
    assert torch.equal(v, v_ref)
    assert int(i[0]) == base


def test_embedding_vocab_parallel(cuda):
    table = torch.randn(100, 256, device=cuda).to(torch.bfloat16)
    ids = torch.tensor([5, 150, 100, 199, 120], dtype=torch.int32, device=cuda)
    out = torch.empty(5, 256, dtype=torch.bfloat16, device=cuda)
    ops.embedding(ids, table, 100, out)
    assert torch.equal(out[1], table[50]) and torch.equal(out[3], table[99])
    assert out[0].abs().sum() == 0 and torch.equal(out[2], table[0])


def test_argmax_rows_and_combine(cuda):
    logits = torch.randn(9, 1000, device=cuda)
    logits[3, 10] = logits[3, 500] = 100.0  # tie -> smallest index
    v = torch.empty(9, device=cuda)
    i = torch.empty(9, dtype=torch.int32, device=cuda)
    ops.argmax_rows(logits, 2000, v, i)
    assert i[3].item() == 2010
    ref = logits.argmax(-1).int() + 2000
    ref[3] = 2010
    assert torch.equal(i, ref)
    vals = torch.tensor([[1.0, 5.0], [3.0, 5.0]], device=cuda)
    idxs = torch.tensor([[7, 9], [2, 4]], dtype=torch.int32, device=cuda)
    o = torch.empty(2, dtype=torch.int32, device=cuda)
    ops.argmax_combine(vals, idxs, o)
    assert o.tolist() == [2, 4]


def _attn_ref(q, k, v, causal_offset=None):
    # q [Tq, H, d], k/v [Tk, Hk, d] fp32
    g = q.shape[1] // k.shape[1]
    k = k.repeat_interleave(g, 1)
    v = v.repeat_interleave(g, 1)
    s = torch.einsum("qhd,khd->hqk", q, k) / math.sqrt(q.shape[-1])
    if causal_offset is not None:
        Tq, Tk = q.shape[0], k.shape[0]
        mask = torch.arange(Tk, device=q.device)[None, :] > (torch.arange(Tq, device=q.device)[:, None] + causal_offset)
        s = s.masked_fill(mask[None], float("-inf"))
    return torch.einsum("hqk,khd->qhd", s.softmax(-1), v)


@pytest.mark.parametrize("variant", [0, 1, 2])
@pytest.mark.parametrize("d,nq,nk,lens", [(128, 8, 2, [1024, 77, 130]), (64, 4, 4, [64, 1, 200]),
                                          (128, 32, 8, [300]), (128, 4, 4, [128, 129, 1, 255, 256]),
                                          (128, 32, 8, [1024] * 6 + [77, 700])])
def test_prefill_attention(cuda, d, nq, nk, lens, variant):
    T = sum(lens)
    qkv = torch.randn(T, (nq + 2 * nk) * d, device=cuda).to(torch.bfloat16)
    cu = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int32, device=cuda)
    out = torch.empty(T, nq * d, dtype=torch.bfloat16, device=cuda)
    ops.prefill_attention(qkv, nq, nk, d, cu, max(lens), out, 1 / math.sqrt(d), variant=variant)
    x = qkv.float().view(T, nq + 2 * nk, d)
    start = 0
    for L in lens:
        q, k, v = x[start : start + L, :nq], x[start : start + L, nq : nq + nk], x[start : start + L, nq + nk :]
        ref = _attn_ref(q, k, v, causal_offset=0).reshape(L, nq * d)
        err = (out[start : start + L].float() - ref).abs().max().item()
        assert err < 0.03, f"len {L}: {err}"
        start += L


@pytest.mark.parametrize("d,nq,nk,ctxs", [(128, 32, 8, [1, 64, 65, 1000, 1280]), (64, 4, 4, [96, 7, 128]),
                                          (128, 4, 1, [500, 33]),
                                          # more (sequence, KV head) items than resident CTAs: the
                                          # persistent kernel's ring carries blocks across items
                                          (128, 32, 8, list(np.random.default_rng(3).integers(1, 400, 90))),
                                          (128, 8, 1, [1] * 700 + [65, 130])])
def test_decode_attention_paged(cuda, d, nq, nk, ctxs):
    B, L, BS = len(ctxs), 2, 64
    nblk = [-(-c // BS) for c in ctxs]
    NB = sum(nblk) + 3
    pool = torch.randn(NB * L * 2 * nk * BS * d, device=cuda).to(torch.bfloat16)
    perm = np.random.default_rng(0).permutation(NB)
    maxb = max(nblk)
    tables = np.zeros((B, maxb), dtype=np.int32)
    pos = 0
    for b, n in enumerate(nblk):
        tables[b, :n] = perm[pos : pos + n]
        pos += n
    qkv = torch.randn(B, (nq + 2 * nk) * d, device=cuda).to(torch.bfloat16)
    out = torch.empty(B, nq * d, dtype=torch.bfloat16, device=cuda)
    layer = 1
    ops.decode_attention(qkv, nq, nk, pool, (L, nk, BS, d), NB, layer, torch.from_numpy(tables).to(cuda),
                         torch.tensor(ctxs, dtype=torch.int32, device=cuda), out, 1 / math.sqrt(d))
    P = pool.view(NB, L, 2, nk, BS, d).float()
    for b, c in enumerate(ctxs):
        ids = torch.from_numpy(tables[b, : nblk[b]]).long().to(cuda)
        K = P[ids, layer, 0].permute(0, 2, 1, 3).reshape(-1, nk, d)[:c]
        V = P[ids, layer, 1].permute(0, 2, 1, 3).reshape(-1, nk, d)[:c]
        q = qkv[b, : nq * d].float().view(1, nq, d)
        ref = _attn_ref(q, K, V).reshape(nq * d)
        err = (out[b].float() - ref).abs().max().item()
        assert err < 0.03, f"ctx {c}: {err}"
