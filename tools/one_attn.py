"""Launch the prefill attention a few times at the bench shape (ncu target)."""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2503_06433_b200 import ops  # noqa: E402

lens = [1024] * 16
nq, nk, d = 32, 8, 128
T = sum(lens)
qkv = torch.randn(T, (nq + 2 * nk) * d, device="cuda").to(torch.bfloat16)
cu = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int32, device="cuda")
out = torch.empty(T, nq * d, dtype=torch.bfloat16, device="cuda")
for _ in range(3):
    ops.prefill_attention(qkv, nq, nk, d, cu, max(lens), out, d ** -0.5)
torch.cuda.synchronize()
