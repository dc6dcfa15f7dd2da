"""RMSNorm folded into the GEMMs (ssb_rownorm): the residual-epilogue GEMM
emits per-N-tile row sums of squares of the x it stores, the consumer GEMMs
take x itself and scale their accumulator rows by 1/rms; the gains are folded
into the consumer weights once (Worker.fold_gains).  Checked against plain
PyTorch fp32 references of rmsnorm(x) @ W^T."""

from __future__ import annotations

import pytest
import torch

from paper_2503_06433_b200 import ops
from paper_2503_06433_b200._lib import SSB_GEMM_2SM, SSB_GEMM_SPLIT_SHIFT

pytestmark = pytest.mark.gpu

EPS = 1e-5


def _rand(shape, g, scale=1.0):
    return (torch.randn(*shape, device="cuda", generator=g) * scale).to(torch.bfloat16)


@pytest.mark.parametrize("M,N,K,flag", [
    (512, 4096, 4096, 0),                                  # auto plan (measured table)
    (512, 4096, 14336, 0),                                 # auto plan, split-K down_proj shape
    (300, 4096, 1024, 128),
    (257, 4096, 512, 224),                                 # ragged last N tile (4096 % 224)
    (512, 4096, 2048, 256 | SSB_GEMM_2SM),
    (512, 5120, 4096, 256 | (3 << SSB_GEMM_SPLIT_SHIFT)),  # forced split-K: sums in the reduction epilogue
    (1000, 8192, 256, 0),
])
def test_producer_row_sums_of_squares(cuda, M, N, K, flag):
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    a = _rand((M, K), g)
    w = _rand((N, K), g, K**-0.5)
    x0 = _rand((M, N), g)
    ws = torch.zeros(160 << 20, dtype=torch.uint8, device=cuda)
    ref_x = x0.clone()
    ops.gemm(a, w, out=ref_x, residual=ref_x, block_n=flag, workspace=ws)
    x = x0.clone()
    ss = torch.full((M * ((N + 63) // 64),), float("nan"), device=cuda)
    rn = ops.row_norm(ss_out=ss)
    ops.gemm(a, w, out=x, residual=x, block_n=flag, workspace=ws, rownorm=rn)
    torch.cuda.synchronize()
    assert torch.equal(x, ref_x), "the sums must not change the stored output"
    parts = rn.ss_parts
    bn = flag & 0xFFFF
    if bn:
        assert parts == -(-N // bn)
    got = ss[: M * parts].view(M, parts).sum(1)
    want = (x.float() ** 2).sum(1)
    assert torch.allclose(got, want, rtol=1e-5, atol=1e-3)


def _inv_rms(x: torch.Tensor) -> torch.Tensor:
    return torch.rsqrt((x.float() ** 2).mean(1) + EPS)


def _split_ss(x: torch.Tensor, parts: int) -> torch.Tensor:
    """Per-row sums of squares split over `parts` column chunks, as a producer writes them."""
    return torch.stack([c.float().pow(2).sum(1) for c in x.chunk(parts, dim=1)], 1).contiguous()


@pytest.mark.parametrize("M,N,K", [(512, 6144, 4096), (512, 28672, 4096), (77, 1024, 4096), (16384, 4096, 4096)])
def test_consumer_row_scale(cuda, M, N, K):
    g = torch.Generator(device="cuda").manual_seed(M * 3 + N)
    x = _rand((M, K), g, 3.0)
    w = _rand((N, K), g, K**-0.5)
    ws = torch.zeros(160 << 20, dtype=torch.uint8, device=cuda)
    parts = 16
    ss = _split_ss(x, parts)
    rn = ops.row_norm(ss_in=ss, ss_in_parts=parts, hidden=K, eps=EPS)
    inv = _inv_rms(x)
    ref = inv[:, None] * (x.float() @ w.float().T)
    tol = 2e-2 * ref.abs().max().item()
    y = ops.gemm(x, w, workspace=ws, rownorm=rn)
    f = ops.gemm(x, w, out_f32=True, workspace=ws, rownorm=rn)
    torch.cuda.synchronize()
    assert (y.float() - ref).abs().max().item() < tol
    assert (f - ref).abs().max().item() < 1e-3 * ref.abs().max().item()
    for odd in (7, 37):  # parts not a multiple of 4: the scalar load path
        rn_odd = ops.row_norm(ss_in=_split_ss(x, odd), ss_in_parts=odd, hidden=K, eps=EPS)
        f_odd = ops.gemm(x, w, out_f32=True, workspace=ws, rownorm=rn_odd)
        torch.cuda.synchronize()
        assert (f_odd - ref).abs().max().item() < 1e-3 * ref.abs().max().item()
    # SiLU(gate) * up on the scaled rows
    if N % 64 == 0:
        F = N // 2
        s = ops.gemm(x, w, silu_mul=True, workspace=ws, rownorm=rn)
        torch.cuda.synchronize()
        wv = w.view(F // 32, 2, 32, K)
        gg = ref.view(M, F // 32, 2, 32)[:, :, 0].reshape(M, F)
        uu = ref.view(M, F // 32, 2, 32)[:, :, 1].reshape(M, F)
        sref = torch.nn.functional.silu(gg) * uu
        assert (s.float() - sref).abs().max().item() < 3e-2 * sref.abs().max().item() + 1e-2
        del wv


def test_lm_head_argmax_on_scaled_rows(cuda):
    """argmax in the epilogue of the row-scaled LM head == argmax_rows of the
    row-scaled fp32 logits (the same scaled values, bit for bit)."""
    M, N, K = 512, 32000, 4096
    g = torch.Generator(device="cuda").manual_seed(11)
    x = _rand((M, K), g, 2.0)
    w = _rand((N, K), g, K**-0.5)
    ws = torch.zeros(64 << 20, dtype=torch.uint8, device=cuda)
    rn = ops.row_norm(ss_in=_split_ss(x, 8), ss_in_parts=8, hidden=K, eps=EPS)
    logits = ops.gemm(x, w, out_f32=True, workspace=ws, rownorm=rn)
    v_ref = torch.empty(M, dtype=torch.float32, device=cuda)
    i_ref = torch.empty(M, dtype=torch.int32, device=cuda)
    ops.argmax_rows(logits, 0, v_ref, i_ref)
    v, i = torch.empty_like(v_ref), torch.empty_like(i_ref)
    ops.lm_head_argmax(x, w, 0, v, i, workspace=ws, rownorm=rn)
    torch.cuda.synchronize()
    assert torch.equal(i, i_ref) and torch.equal(v, v_ref)
    ref = _inv_rms(x)[:, None] * (x.float() @ w.float().T)
    assert (logits - ref).abs().max().item() < 1e-3 * ref.abs().max().item()


def test_qkv_rope_kv_on_scaled_rows(cuda):
    """QKV GEMM + RoPE + paged K/V append with the row scale == the same
    fused GEMM on h = bf16(x / rms) (bf16 tolerance: one rounding apart)."""
    M, K, nq, nk, d = 300, 4096, 32, 8, 128
    g = torch.Generator(device="cuda").manual_seed(5)
    x = _rand((M, K), g, 2.0)
    w = _rand(((nq + 2 * nk) * d, K), g, K**-0.5)
    pos = torch.randint(0, 2000, (M,), device=cuda, generator=g, dtype=torch.int32)
    half = d // 2
    inv_freq = 1.0 / (500000.0 ** (torch.arange(half, device=cuda, dtype=torch.float32) / half))
    ang = torch.arange(4096, device=cuda, dtype=torch.float32)[:, None] * inv_freq[None]
    cos, sin = ang.cos().contiguous(), ang.sin().contiguous()
    blocks, bs = 8, 64
    geo = (1, nk, bs, d)
    pool_a = torch.zeros(blocks * 2 * nk * bs * d, dtype=torch.bfloat16, device=cuda)
    pool_b = torch.zeros_like(pool_a)
    slots = torch.randperm(blocks * bs, device=cuda, generator=g)[:M].to(torch.int64)
    ws = torch.zeros(64 << 20, dtype=torch.uint8, device=cuda)
    rn = ops.row_norm(ss_in=_split_ss(x, 4), ss_in_parts=4, hidden=K, eps=EPS)
    qa = torch.empty(M, (nq + 2 * nk) * d, dtype=torch.bfloat16, device=cuda)
    qb = torch.empty_like(qa)
    ops.gemm_qkv_rope_kv(x, w, qa, nq, nk, pos, cos, sin, pool_a, geo, 0, slots, workspace=ws, rownorm=rn)
    h = (x.float() * _inv_rms(x)[:, None]).to(torch.bfloat16)
    ops.gemm_qkv_rope_kv(h, w, qb, nq, nk, pos, cos, sin, pool_b, geo, 0, slots, workspace=ws)
    torch.cuda.synchronize()
    scale = qb.float().abs().max().item()
    assert (qa.float() - qb.float()).abs().max().item() < 2e-2 * scale
    assert (pool_a.float() - pool_b.float()).abs().max().item() < 2e-2 * scale


def test_fold_gains_moves_gains_into_weights(cuda):
    from paper_2503_06433_b200 import PRESETS, ParallelismConfig
    from paper_2503_06433_b200.comm import SoloComm
    from paper_2503_06433_b200.runtime import Worker

    arch = PRESETS["tiny"]
    wk = Worker(arch, SoloComm(), 1, torch.device("cuda", 0), seed=0, max_pos=64)
    wk.fold_norm = False
    wk.init_weights(ParallelismConfig(1, 1, 1))
    g = torch.Generator(device="cuda").manual_seed(3)
    keys = [("L0.attn_norm", "L0.wqkv"), ("L1.mlp_norm", "L1.w13"), ("final_norm", "head")]
    before = {}
    for gk, wkey in keys:
        wk.w(gk).copy_((torch.rand(wk.w(gk).shape, device=cuda, generator=g) + 0.5).to(torch.bfloat16))
        before[gk] = (wk.w(gk).clone(), wk.w(wkey).clone())
    untouched = wk.w("L1.attn_norm").clone(), wk.w("L1.wqkv").clone()
    wk.fold_gains()
    for gk, wkey in keys:
        gam, w0 = before[gk]
        assert torch.equal(wk.w(wkey), (w0 * gam.view(1, -1)))
        assert bool(torch.all(wk.w(gk) == 1))
    # unit gains: nothing changes
    assert torch.equal(wk.w("L1.wqkv"), untouched[1]) and torch.equal(wk.w("L1.attn_norm"), untouched[0])
