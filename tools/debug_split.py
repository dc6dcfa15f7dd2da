"""Auto-plan (split-K capable) GEMMs vs fp32 torch on given shapes."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2503_06433_b200 import ops  # noqa: E402
from paper_2503_06433_b200._lib import SSB_EPI_NONE, SSB_EPI_RESIDUAL, SSB_EPI_SILU_MUL  # noqa: E402

ws = torch.zeros(64 << 20, dtype=torch.uint8, device="cuda")
for M in (96, 1, 3, 200):
    for (N, K, epi) in [(10240, 8192, SSB_EPI_NONE), (8192, 8192, SSB_EPI_RESIDUAL), (57344, 8192, SSB_EPI_SILU_MUL),
                        (8192, 28672, SSB_EPI_RESIDUAL), (28672, 8192, SSB_EPI_SILU_MUL), (8192, 14336, SSB_EPI_RESIDUAL)]:
        a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        w = (torch.randn(N, K, device="cuda") / K**0.5).to(torch.bfloat16)
        plan, need = ops.gemm_plan(M, N, K, epi, 0, ws.numel())
        ref = a.float() @ w.float().T
        if epi == SSB_EPI_SILU_MUL:
            F = N // 2
            wv = w.view(F // 32, 2, 32, K)
            g = a.float() @ wv[:, 0].reshape(F, K).float().T
            u = a.float() @ wv[:, 1].reshape(F, K).float().T
            ref = torch.nn.functional.silu(g) * u
            out = ops.gemm(a, w, silu_mul=True, workspace=ws)
        elif epi == SSB_EPI_RESIDUAL:
            r = torch.randn(M, N, device="cuda").to(torch.bfloat16)
            ref = ref + r.float()
            out = ops.gemm(a, w, out=r, residual=r, workspace=ws)
        else:
            out = ops.gemm(a, w, workspace=ws)
        torch.cuda.synchronize()
        err = (out.float() - ref).abs().max().item()
        cnt = int(ws[:65536].view(torch.int32).abs().sum())
        print(f"M={M} N={N} K={K} epi={epi} plan={plan} need={need} err={err:.4f} ref_max={ref.abs().max().item():.3f} "
              f"zero_rows={int((out.float().abs().sum(1) == 0).sum())} counters_after={cnt}", flush=True)
