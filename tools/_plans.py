import sys
sys.path.insert(0, "/root/repo")
from paper_2503_06433_b200 import ops
from paper_2503_06433_b200._lib import SSB_EPI_NONE, SSB_EPI_RESIDUAL, SSB_EPI_SILU_MUL, SSB_EPI_ROPE_KV
for (N, K, e) in [(6144, 4096, SSB_EPI_ROPE_KV), (4096, 4096, SSB_EPI_RESIDUAL), (28672, 4096, SSB_EPI_SILU_MUL), (4096, 14336, SSB_EPI_RESIDUAL), (128256, 4096, 5)]:
    print(N, K, e, ops.gemm_plan(512, N, K, e, 0, 64 << 20))
