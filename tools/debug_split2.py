import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2503_06433_b200 import ops  # noqa: E402
from paper_2503_06433_b200._lib import SSB_GEMM_SPLIT_SHIFT  # noqa: E402


def run(M, N, K, bn, sp, silu, fresh=True):
    ws = torch.zeros(128 << 20, dtype=torch.uint8, device="cuda")
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    w = (torch.randn(N, K, device="cuda") / K**0.5).to(torch.bfloat16)
    flag = bn | (sp << SSB_GEMM_SPLIT_SHIFT)
    if silu:
        F = N // 2
        wv = w.view(F // 32, 2, 32, K)
        g = a.float() @ wv[:, 0].reshape(F, K).float().T
        u = a.float() @ wv[:, 1].reshape(F, K).float().T
        ref = torch.nn.functional.silu(g) * u
        out = ops.gemm(a, w, silu_mul=True, workspace=ws, block_n=flag)
    else:
        ref = a.float() @ w.float().T
        out = ops.gemm(a, w, workspace=ws, block_n=flag)
    torch.cuda.synchronize()
    tiles = -(-M // 128) * -(-N // bn)
    cnt = ws[: tiles * 16].view(torch.int32)
    bad_rows = (out.float() - ref).abs().amax(1) > 0.1
    bad_cols = ((out.float() - ref).abs() > 0.1).any(0).nonzero().flatten()
    print(f"M={M} N={N} K={K} bn={bn} sp={sp} silu={silu} err={(out.float()-ref).abs().max().item():.4f} "
          f"nonzero_counters={int((cnt != 0).sum())} first_bad_tile={int(cnt.view(-1,4).abs().sum(1).nonzero()[0]) if (cnt!=0).any() else -1} "
          f"bad_cols={bad_cols.numel()} first_bad_col={int(bad_cols[0]) if bad_cols.numel() else -1}", flush=True)


for args in [(96, 57344, 8192, 128, 2, True), (96, 57344, 8192, 128, 2, False), (96, 28672, 8192, 128, 2, True),
             (96, 16384, 8192, 128, 2, False), (96, 8192, 4096, 128, 2, False), (96, 19200, 1024, 128, 2, False),
             (96, 38400, 1024, 128, 2, False), (96, 57344, 1024, 128, 2, False), (300, 57344, 1024, 128, 2, False),
             (96, 57344, 1024, 128, 1, False), (96, 57344, 1024, 256, 2, False)]:
    run(*args)
