import torch
from paper_2503_06433_b200 import ops
dev = torch.device("cuda", 0)
g = torch.Generator(device="cuda").manual_seed(0)
for M in (17, 130, 200, 475):
    for (N, K) in ((256, 256), (256, 768)):
        a = torch.randn(M, K, device=dev, generator=g).to(torch.bfloat16)
        w = (torch.randn(N, K, device=dev, generator=g) / K**0.5).to(torch.bfloat16)
        x = torch.randn(M, N, device=dev, generator=g).to(torch.bfloat16)
        ss = torch.full((M * 4,), float("nan"), device=dev)
        rn = ops.row_norm(ss_out=ss)
        ref_x = x.clone(); ops.gemm(a, w, out=ref_x, residual=ref_x)
        ops.gemm(a, w, out=x, residual=x, rownorm=rn)
        torch.cuda.synchronize()
        p = rn.ss_parts
        got = ss[: M * p].view(M, p).sum(1); want = (x.float() ** 2).sum(1)
        print("producer", M, N, K, "parts", p, "x equal", torch.equal(x, ref_x), "ss err", (got - want).abs().max().item(),
              "plan", ops.gemm_plan(M, N, K, 1))
        w2 = (torch.randn(768, N, device=dev, generator=g) / N**0.5).to(torch.bfloat16)
        rc = ops.row_norm(ss_in=ss[: M * p].view(M, p), ss_in_parts=p, hidden=N, eps=1e-5)
        y = ops.gemm(x, w2, rownorm=rc)
        inv = torch.rsqrt((x.float() ** 2).mean(1) + 1e-5)
        ref = inv[:, None] * (x.float() @ w2.float().T)
        torch.cuda.synchronize()
        print("  consumer err", (y.float() - ref).abs().max().item(), "scale", ref.abs().max().item(), "plan", ops.gemm_plan(M, 768, N, 0))
