"""tcgen05 GEMM vs a plain PyTorch fp32 reference of the same op."""

from __future__ import annotations

import pytest
import torch

from paper_2503_06433_b200 import ops

pytestmark = pytest.mark.gpu


def _ref(a, w):
    return a.float() @ w.float().T


@pytest.mark.parametrize(
    "M,N,K,bn",
    [
        (128, 256, 64, 256),
        (256, 512, 4096, 256),
        (1000, 768, 4096, 0),
        (512, 6144, 4096, 0),
        (77, 200, 136, 64),
        (300, 384, 1024, 128),
        (4096, 4096, 4096, 256),
        (512, 6144, 4096, 192),
        (512, 4096, 4096, 224),
        (300, 200, 136, 224),
        (130, 1000, 520, 192),
    ],
)
def test_gemm_plain(cuda, M, N, K, bn):
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N)
    a = torch.randn(M, K, device=cuda, generator=g).to(torch.bfloat16)
    w = (torch.randn(N, K, device=cuda, generator=g) / K**0.5).to(torch.bfloat16)
    out = ops.gemm(a, w, block_n=bn)
    torch.cuda.synchronize()
    ref = _ref(a, w)
    err = (out.float() - ref).abs().max().item()
    tol = 2e-2 * ref.abs().max().item() + 1e-2
    assert err <= tol, f"max err {err} > {tol}"


@pytest.mark.parametrize("mode", ["mc1", "mc2", "2sm"])
@pytest.mark.parametrize("M,N,K,bn", [(300, 640, 512, 128), (512, 4096, 1024, 192), (1000, 768, 4096, 256),
                                      (129, 448, 256, 224), (64, 256, 128, 128), (2048, 1024, 4096, 256)])
def test_gemm_cluster_modes(cuda, mode, M, N, K, bn):
    from paper_2503_06433_b200._lib import SSB_GEMM_2SM, SSB_GEMM_MC1, SSB_GEMM_MC2

    flag = {"mc1": SSB_GEMM_MC1, "mc2": SSB_GEMM_MC2, "2sm": SSB_GEMM_2SM}[mode]
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    a = torch.randn(M, K, device=cuda, generator=g).to(torch.bfloat16)
    w = (torch.randn(N, K, device=cuda, generator=g) / K**0.5).to(torch.bfloat16)
    out = ops.gemm(a, w, block_n=bn | flag)
    torch.cuda.synchronize()
    ref = _ref(a, w)
    assert (out.float() - ref).abs().max().item() <= 2e-2 * ref.abs().max().item() + 1e-2
    # fused epilogues through the pair path too
    r = torch.randn(M, N, device=cuda).to(torch.bfloat16)
    exp = ref + r.float()
    ops.gemm(a, w, out=r, residual=r, block_n=bn | flag)
    torch.cuda.synchronize()
    assert (r.float() - exp).abs().max().item() <= 2e-2 * exp.abs().max().item() + 2e-2


def test_gemm_residual_inplace(cuda):
    M, N, K = 384, 1024, 512
    a = torch.randn(M, K, device=cuda).to(torch.bfloat16)
    w = (torch.randn(N, K, device=cuda) / K**0.5).to(torch.bfloat16)
    r = torch.randn(M, N, device=cuda).to(torch.bfloat16)
    ref = _ref(a, w) + r.float()
    ops.gemm(a, w, out=r, residual=r)
    torch.cuda.synchronize()
    assert (r.float() - ref).abs().max().item() < 5e-2


@pytest.mark.parametrize("bn", [0, 128, 192, 256])
def test_gemm_silu_mul(cuda, bn):
    M, F, K = 640, 480, 1024
    a = torch.randn(M, K, device=cuda).to(torch.bfloat16)
    gate = (torch.randn(F, K, device=cuda) / K**0.5).to(torch.bfloat16)
    up = (torch.randn(F, K, device=cuda) / K**0.5).to(torch.bfloat16)
    # interleave (32 gate, 32 up) row groups
    w = torch.stack([gate.view(F // 32, 32, K), up.view(F // 32, 32, K)], dim=1).reshape(2 * F, K)
    out = ops.gemm(a, w, silu_mul=True, block_n=bn)
    torch.cuda.synchronize()
    g = a.float() @ gate.float().T
    u = a.float() @ up.float().T
    ref = torch.nn.functional.silu(g) * u
    assert (out.float() - ref).abs().max().item() < 3e-2 * ref.abs().max().item() + 1e-2


def test_gemm_strided_a(cuda):
    # A is a column slice of a wider activation (row stride > K)
    M, K, N = 256, 512, 256
    big = torch.randn(M, 3 * K, device=cuda).to(torch.bfloat16)
    a = big[:, K : 2 * K]
    w = (torch.randn(N, K, device=cuda) / K**0.5).to(torch.bfloat16)
    out = ops.gemm(a, w)
    torch.cuda.synchronize()
    assert (out.float() - _ref(a, w)).abs().max().item() < 5e-2


def _ws(cuda, nbytes=64 << 20):
    return torch.zeros(nbytes, dtype=torch.uint8, device=cuda)


@pytest.mark.parametrize("mode", ["single", "2sm"])
@pytest.mark.parametrize("splits", [2, 3, 5, 16])
@pytest.mark.parametrize("M,N,K,bn", [(512, 768, 4096, 256), (512, 4096, 512, 128), (300, 640, 1000, 192),
                                      (129, 448, 2048, 224), (64, 256, 4096, 128)])
def test_gemm_split_k(cuda, mode, splits, M, N, K, bn):
    """Split-K (forced): fp32 partials reduced in-kernel by the last warp of
    each tile quadrant; every epilogue; deterministic run to run."""
    from paper_2503_06433_b200._lib import SSB_GEMM_2SM, SSB_GEMM_SPLIT_SHIFT

    flag = bn | (splits << SSB_GEMM_SPLIT_SHIFT) | (SSB_GEMM_2SM if mode == "2sm" else 0)
    g = torch.Generator(device="cuda").manual_seed(M + N + K + splits)
    a = torch.randn(M, K, device=cuda, generator=g).to(torch.bfloat16)
    w = (torch.randn(N, K, device=cuda, generator=g) / K**0.5).to(torch.bfloat16)
    ws = _ws(cuda, 160 << 20)
    out = ops.gemm(a, w, block_n=flag, workspace=ws)
    out2 = ops.gemm(a, w, block_n=flag, workspace=ws)
    torch.cuda.synchronize()
    ref = _ref(a, w)
    assert (out.float() - ref).abs().max().item() <= 2e-2 * ref.abs().max().item() + 1e-2
    assert torch.equal(out, out2), "split-K reduction must be deterministic"
    # the fixed 64 KiB tile-counter head of the workspace is left zero
    assert int(ws[: 64 << 10].view(torch.int32).abs().sum()) == 0
    r = torch.randn(M, N, device=cuda, generator=g).to(torch.bfloat16)
    exp = ref + r.float()
    ops.gemm(a, w, out=r, residual=r, block_n=flag, workspace=ws)
    f = ops.gemm(a, w, out_f32=True, block_n=flag, workspace=ws)
    torch.cuda.synchronize()
    assert (r.float() - exp).abs().max().item() <= 2e-2 * exp.abs().max().item() + 2e-2
    assert (f - ref).abs().max().item() <= 1e-3 * ref.abs().max().item() + 1e-3
    if bn % 64 == 0 and N % 64 == 0:
        F = N // 2
        s = ops.gemm(a, w, silu_mul=True, block_n=flag, workspace=ws)
        torch.cuda.synchronize()
        wv = w.view(F // 32, 2, 32, K)
        gg = a.float() @ wv[:, 0].reshape(F, K).float().T
        uu = a.float() @ wv[:, 1].reshape(F, K).float().T
        sref = torch.nn.functional.silu(gg) * uu
        assert (s.float() - sref).abs().max().item() < 3e-2 * sref.abs().max().item() + 1e-2


@pytest.mark.parametrize("M,N,K", [(512, 6144, 4096), (512, 4096, 4096), (512, 28672, 4096), (512, 4096, 14336),
                                   (512, 768, 4096), (512, 4096, 512), (512, 3584, 4096), (512, 4096, 1792),
                                   (512, 16032, 4096), (16384, 6144, 4096), (8, 6144, 4096)])
def test_gemm_auto_plan(cuda, M, N, K):
    """The auto plan (possibly split-K) on the Llama-3-8B decode shapes at
    TP1 and TP8, bit-identical across repeated launches."""
    g = torch.Generator(device="cuda").manual_seed(M ^ N ^ K)
    a = torch.randn(M, K, device=cuda, generator=g).to(torch.bfloat16)
    w = (torch.randn(N, K, device=cuda, generator=g) / K**0.5).to(torch.bfloat16)
    ws = _ws(cuda)
    plan, need = ops.gemm_plan(M, N, K, workspace_bytes=ws.numel())
    assert need <= ws.numel()
    out = ops.gemm(a, w, workspace=ws)
    out2 = ops.gemm(a, w, workspace=ws)
    torch.cuda.synchronize()
    ref = _ref(a, w)
    assert (out.float() - ref).abs().max().item() <= 2e-2 * ref.abs().max().item() + 1e-2, plan
    assert torch.equal(out, out2)


def test_gemm_split_k_shared_workspace_sequence(cuda):
    """Many split-K GEMMs of different tile counts through ONE workspace (as
    a decode step does): the counter area must stay valid across shapes (a
    layout whose counter area grew with the tile count let one launch's
    partials masquerade as the next launch's counters)."""
    from paper_2503_06433_b200._lib import SSB_GEMM_SPLIT_SHIFT

    ws = _ws(cuda)
    g = torch.Generator(device="cuda").manual_seed(7)
    shapes = [(96, 10240, 2048, 128, 5), (96, 57344, 1024, 128, 2), (1, 10240, 2048, 128, 5),
              (200, 8192, 4096, 224, 2), (3, 20480, 1024, 256, 3), (96, 10240, 2048, 128, 5)]
    for M, N, K, bn, sp in shapes * 2:
        a = torch.randn(M, K, device=cuda, generator=g).to(torch.bfloat16)
        w = (torch.randn(N, K, device=cuda, generator=g) / K**0.5).to(torch.bfloat16)
        out = ops.gemm(a, w, block_n=bn | (sp << SSB_GEMM_SPLIT_SHIFT), workspace=ws)
        torch.cuda.synchronize()
        ref = _ref(a, w)
        assert (out.float() - ref).abs().max().item() <= 2e-2 * ref.abs().max().item() + 1e-2, (M, N, K, bn, sp)
        assert int(ws[: 64 << 10].view(torch.int32).abs().sum()) == 0


@pytest.mark.parametrize("mode", ["single", "2sm"])
@pytest.mark.parametrize("M,N,K,bn,splits", [(512, 28672, 4096, 256, 4), (512, 40000, 1024, 128, 2),
                                             (300, 20000, 2048, 192, 3), (512, 19200, 512, 256, 8)])
def test_gemm_tail_split(cuda, mode, M, N, K, bn, splits):
    """Tail split: whole tiles in the full waves, only the last partial wave's
    tiles split K -- every epilogue, deterministic, counters left zero."""
    from paper_2503_06433_b200._lib import SSB_GEMM_2SM, SSB_GEMM_SPLIT_SHIFT, SSB_GEMM_TAIL

    flag = bn | (splits << SSB_GEMM_SPLIT_SHIFT) | SSB_GEMM_TAIL | (SSB_GEMM_2SM if mode == "2sm" else 0)
    g = torch.Generator(device="cuda").manual_seed(N + splits)
    a = torch.randn(M, K, device=cuda, generator=g).to(torch.bfloat16)
    w = (torch.randn(N, K, device=cuda, generator=g) / K**0.5).to(torch.bfloat16)
    ws = _ws(cuda, 160 << 20)
    out = ops.gemm(a, w, block_n=flag, workspace=ws)
    out2 = ops.gemm(a, w, block_n=flag, workspace=ws)
    torch.cuda.synchronize()
    ref = _ref(a, w)
    assert (out.float() - ref).abs().max().item() <= 2e-2 * ref.abs().max().item() + 1e-2
    assert torch.equal(out, out2)
    assert int(ws[: 64 << 10].view(torch.int32).abs().sum()) == 0
    r = torch.randn(M, N, device=cuda, generator=g).to(torch.bfloat16)
    exp = ref + r.float()
    ops.gemm(a, w, out=r, residual=r, block_n=flag, workspace=ws)
    torch.cuda.synchronize()
    assert (r.float() - exp).abs().max().item() <= 2e-2 * exp.abs().max().item() + 2e-2
    if bn % 64 == 0 and N % 64 == 0:
        F = N // 2
        s = ops.gemm(a, w, silu_mul=True, block_n=flag, workspace=ws)
        torch.cuda.synchronize()
        wv = w.view(F // 32, 2, 32, K)
        sref = torch.nn.functional.silu(a.float() @ wv[:, 0].reshape(F, K).float().T) * (
            a.float() @ wv[:, 1].reshape(F, K).float().T)
        assert (s.float() - sref).abs().max().item() < 3e-2 * sref.abs().max().item() + 1e-2


@pytest.mark.parametrize("mode", ["single", "2sm"])
@pytest.mark.parametrize("M,N,K,bn", [(512, 4096, 4096, 256), (512, 6144, 4096, 256), (512, 4096, 14336, 256),
                                      (512, 28672, 4096, 256), (300, 640, 1000, 192), (129, 448, 2048, 224),
                                      (512, 16032, 4096, 128), (64, 256, 4096, 128), (1000, 3000, 704, 256)])
def test_gemm_stream_k(cuda, mode, M, N, K, bn):
    """Stream-K (forced): whole tiles, then the last rounds' k-blocks split
    evenly over the persistent CTAs, shared tiles reduced in k order by their
    last contributor into TMEM -- every epilogue, deterministic, counters
    left zero."""
    from paper_2503_06433_b200._lib import SSB_GEMM_2SM, SSB_GEMM_STREAMK

    flag = bn | SSB_GEMM_STREAMK | (SSB_GEMM_2SM if mode == "2sm" else 0)
    g = torch.Generator(device="cuda").manual_seed(M * 3 + N + K)
    a = torch.randn(M, K, device=cuda, generator=g).to(torch.bfloat16)
    w = (torch.randn(N, K, device=cuda, generator=g) / K**0.5).to(torch.bfloat16)
    ws = _ws(cuda)
    out = ops.gemm(a, w, block_n=flag, workspace=ws)
    outs = [ops.gemm(a, w, block_n=flag, workspace=ws) for _ in range(3)]
    torch.cuda.synchronize()
    ref = _ref(a, w)
    assert (out.float() - ref).abs().max().item() <= 2e-2 * ref.abs().max().item() + 1e-2
    assert all(torch.equal(out, o) for o in outs), "stream-K reduction must be deterministic"
    assert int(ws[: 64 << 10].view(torch.int32).abs().sum()) == 0
    f = ops.gemm(a, w, out_f32=True, block_n=flag, workspace=ws)
    r = torch.randn(M, N, device=cuda, generator=g).to(torch.bfloat16)
    exp = ref + r.float()
    ops.gemm(a, w, out=r, residual=r, block_n=flag, workspace=ws)
    torch.cuda.synchronize()
    assert (f - ref).abs().max().item() <= 1e-3 * ref.abs().max().item() + 1e-3
    assert (r.float() - exp).abs().max().item() <= 2e-2 * exp.abs().max().item() + 2e-2
    if bn % 64 == 0 and N % 64 == 0:
        F = N // 2
        s = ops.gemm(a, w, silu_mul=True, block_n=flag, workspace=ws)
        torch.cuda.synchronize()
        wv = w.view(F // 32, 2, 32, K)
        gg = a.float() @ wv[:, 0].reshape(F, K).float().T
        uu = a.float() @ wv[:, 1].reshape(F, K).float().T
        sref = torch.nn.functional.silu(gg) * uu
        assert (s.float() - sref).abs().max().item() < 3e-2 * sref.abs().max().item() + 1e-2
    assert int(ws[: 64 << 10].view(torch.int32).abs().sum()) == 0
