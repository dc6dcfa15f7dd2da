"""Launch one GEMM shape a few times (ncu target)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2503_06433_b200 import ops  # noqa: E402

M, N, K = (int(x) for x in sys.argv[1:4])
bn = int(sys.argv[4]) if len(sys.argv) > 4 else 0
a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
w = (torch.randn(N, K, device="cuda") / K**0.5).to(torch.bfloat16)
for _ in range(3):
    ops.gemm(a, w, block_n=bn)
torch.cuda.synchronize()
