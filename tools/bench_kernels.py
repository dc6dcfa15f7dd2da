"""Micro-benchmarks of individual kernels (CUDA events, warm-up, L2 flush)."""

from __future__ import annotations

import argparse
import os
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2503_06433_b200 import ops  # noqa: E402

L2_FLUSH = torch.empty(0)


def timed(fn, iters=20, warmup=3, flush=True):
    global L2_FLUSH
    if L2_FLUSH.numel() == 0:
        L2_FLUSH = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    times = []
    for _ in range(iters):
        if flush:
            L2_FLUSH.zero_()
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        times.append(s.elapsed_time(e))
    times.sort()
    return times[len(times) // 2]


def bench_gemm(shapes):
    out = []
    for M, N, K, bn in shapes:
        a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        w = (torch.randn(N, K, device="cuda") / K**0.5).to(torch.bfloat16)
        c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        ms = timed(lambda: ops.gemm(a, w, out=c, block_n=bn))
        ms_t = timed(lambda: torch.matmul(a, w.T, out=c))
        fl = 2.0 * M * N * K
        out.append(dict(M=M, N=N, K=K, bn=bn, ms=ms, tflops=fl / ms / 1e9, torch_ms=ms_t,
                        torch_tflops=fl / ms_t / 1e9))
        print(json.dumps(out[-1]), flush=True)
    return out


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--what", default="gemm")
    args = ap.parse_args()
    if args.what == "attn":
        import numpy as np

        for lens in ([1024] * 16, [1024] * 4, [4096] * 2):
            nq, nk, d = 32, 8, 128
            T = sum(lens)
            qkv = torch.randn(T, (nq + 2 * nk) * d, device="cuda").to(torch.bfloat16)
            cu = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int32, device="cuda")
            out = torch.empty(T, nq * d, dtype=torch.bfloat16, device="cuda")
            fl = sum(2 * 2 * L * L / 2 * d * nq for L in lens)
            for v in ((0,) if os.environ.get("SSB_ATTN_ONLY0") else (0, 2, 1)):
                ms = timed(lambda: ops.prefill_attention(qkv, nq, nk, d, cu, max(lens), out, d ** -0.5, variant=v))
                print(json.dumps({"lens": f"{len(lens)}x{lens[0]}", "variant": v, "ms": ms,
                                  "tflops": fl / ms / 1e9, "poly": os.environ.get("SSB_ATTN_POLY", "0")}),
                      flush=True)
    if args.what == "mc":
        MC1, TWO = 1 << 16, 1 << 18
        shapes = [(8192, 6144, 4096), (8192, 28672, 4096), (8192, 4096, 14336), (512, 6144, 4096),
                  (512, 4096, 4096), (512, 28672, 4096), (512, 4096, 14336), (512, 128256, 4096)]
        bench_gemm([(M, N, K, MC1) for M, N, K in shapes] + [(M, N, K, TWO) for M, N, K in shapes]
                   + [(M, N, K, TWO | 256) for M, N, K in shapes[3:]])
    if args.what == "gemm":
        bench_gemm([
            (16384, 6144, 4096, 0), (16384, 4096, 4096, 0), (16384, 28672, 4096, 0),
            (16384, 4096, 14336, 0), (512, 6144, 4096, 0), (512, 4096, 4096, 0),
            (512, 28672, 4096, 0), (512, 4096, 14336, 0), (512, 128256, 4096, 0),
            (512, 4096, 4096, 128), (512, 4096, 4096, 64),
        ])


def bench_splitk():
    """Forced (mode, bn, splits) sweep vs the auto plan on decode shapes."""
    from paper_2503_06433_b200._lib import SSB_GEMM_2SM, SSB_GEMM_SPLIT_SHIFT, SSB_GEMM_STREAMK, SSB_GEMM_TAIL

    only = os.environ.get("SSB_SWEEP_SHAPES")  # "M,N,K;M,N,K" restricts the sweep

    ws = torch.zeros(256 << 20, dtype=torch.uint8, device="cuda")
    shapes = [(M, N, K) for M in (512, 256) for N, K in
              ((6144, 4096), (4096, 4096), (28672, 4096), (4096, 14336), (128256, 4096), (768, 4096), (4096, 512),
               (3584, 4096), (4096, 1792), (16032, 4096))]
    shapes += [(16384, 6144, 4096), (16384, 4096, 14336), (2048, 4096, 4096)]
    if only:
        shapes = [tuple(int(x) for x in sh.split(",")) for sh in only.split(";")]
    for M, N, K in shapes:
        a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        w = (torch.randn(N, K, device="cuda") / K**0.5).to(torch.bfloat16)
        c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        fl = 2.0 * M * N * K
        res = []
        plan, need = ops.gemm_plan(M, N, K, workspace_bytes=64 << 20)
        ms = timed(lambda: ops.gemm(a, w, out=c, workspace=ws[: 64 << 20]))
        res.append(("auto", plan, ms))
        ms_t = timed(lambda: torch.matmul(a, w.T, out=c))
        res.append(("cublas", None, ms_t))
        for mode in (0, 2):
            for bn in (128, 192, 224, 256):
                for sp in ((1,) if M > 4096 else (1, 2, 3, 4, 6, 8)):
                    if K // 64 // sp < 2:
                        continue
                    for tail in ((0, 1) if sp > 1 else (0,)):
                        flag = bn | (sp << SSB_GEMM_SPLIT_SHIFT) | (SSB_GEMM_2SM if mode == 2 else 0)
                        flag |= SSB_GEMM_TAIL if tail else 0
                        try:
                            ms = timed(lambda: ops.gemm(a, w, out=c, block_n=flag, workspace=ws), iters=10)
                        except Exception as e:  # noqa: BLE001
                            continue
                        res.append((f"m{mode}b{bn}s{sp}" + ("t" if tail else ""), None, ms))
                if M <= 2048:
                    flag = bn | SSB_GEMM_STREAMK | (SSB_GEMM_2SM if mode == 2 else 0)
                    try:
                        ms = timed(lambda: ops.gemm(a, w, out=c, block_n=flag, workspace=ws), iters=10)
                        res.append((f"m{mode}b{bn}sk", None, ms))
                    except Exception:  # noqa: BLE001
                        pass
        best = min(res[2:], key=lambda r: r[2])
        print(json.dumps({"M": M, "N": N, "K": K, "auto_plan": res[0][1], "auto_ms": res[0][2],
                          "auto_tflops": fl / res[0][2] / 1e9, "cublas_ms": ms_t, "cublas_tflops": fl / ms_t / 1e9,
                          "best": best[0], "best_ms": best[2], "best_tflops": fl / best[2] / 1e9,
                          "all": {r[0]: round(r[2] * 1e3, 1) for r in res[2:]}}), flush=True)


if __name__ == "__main__" and "--what" in sys.argv and sys.argv[sys.argv.index("--what") + 1] == "splitk":
    bench_splitk()


def bench_decode_attn():
    """Decode attention at the bench shape (8B: 512 sequences, ctx 1152,
    32/8 heads, 32-layer pool of 64-token blocks), algorithmic GB/s."""
    ctx = int(os.environ.get("DEC_CTX", "1152"))
    B = int(os.environ.get("DEC_B", str(512 * 1152 // ctx)))  # same KV bytes by default
    nq, nk, d, BS = 32, 8, 128, 64
    L = int(os.environ.get("DEC_LAYERS", "32"))
    seq_tables = os.environ.get("DEC_SEQ", "0") == "1"
    nb = B * (ctx // BS + 2)
    pool = torch.empty(nb * L * 2 * nk * BS * d, dtype=torch.bfloat16, device="cuda")
    pool.view(torch.int16)[:: 1 << 20].zero_()
    ids = torch.arange(nb, device="cuda") if seq_tables else torch.randperm(nb, device="cuda", dtype=torch.int64)
    tables = ids[: B * (ctx // BS + 2)].to(torch.int32).view(B, -1)
    ctxs = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
    qkv = torch.randn(B, (nq + 2 * nk) * d, device="cuda").to(torch.bfloat16)
    out = torch.empty(B, nq * d, dtype=torch.bfloat16, device="cuda")
    layer = min(17, L - 1)
    ms = timed(lambda: ops.decode_attention(qkv, nq, nk, pool, (L, nk, BS, d), nb, layer, tables, ctxs, out,
                                            d ** -0.5), iters=30, flush=False)
    gb = B * ctx * 2 * nk * d * 2 / 1e9
    print(json.dumps({"what": "decode_attn", "ms": ms, "gbs": gb / ms * 1e3, "B": B, "ctx": ctx,
                      "stages": os.environ.get("SSB_DECODE_STAGES", "3"), "ctas": os.environ.get("SSB_DECODE_CTAS", "0"),
                      "variant": os.environ.get("SSB_DECODE_ATTN_VARIANT", "0"), "layers": L,
                      "sequential_blocks": seq_tables}), flush=True)


if __name__ == "__main__" and "--what" in sys.argv and sys.argv[sys.argv.index("--what") + 1] == "decode":
    bench_decode_attn()


def bench_l2_prefetch():
    """Does an L2-resident weight make the M = 512 decode projections faster?
    Each decode projection runs right after decode attention streamed ~2 GB of
    KV through L2 (weights cold, from HBM).  Time o_proj / QKV / down after
    (a) a 2 GiB streaming read (cold weights) and (b) the same read followed
    by a pass over the weight (weights L2-resident), CUDA events on the GEMM."""
    ws = torch.zeros(64 << 20, dtype=torch.uint8, device="cuda")
    junk = torch.empty(1 << 30, dtype=torch.bfloat16, device="cuda").uniform_()
    for M, N, K in ((512, 4096, 4096), (512, 6144, 4096), (512, 4096, 14336)):
        a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        w = (torch.randn(N, K, device="cuda") / K**0.5).to(torch.bfloat16)
        c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        res = {}
        for warm in (0, 1):
            ts = []
            for _ in range(15):
                junk.sum()
                if warm:
                    w.view(torch.int32).amax()  # pulls w through L2
                s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                s_.record()
                ops.gemm(a, w, out=c, workspace=ws)
                e_.record()
                e_.synchronize()
                ts.append(s_.elapsed_time(e_))
            ts.sort()
            res["warm" if warm else "cold"] = ts[len(ts) // 2] * 1e3
        print(json.dumps({"what": "l2_prefetch", "M": M, "N": N, "K": K, "us": res}), flush=True)


if __name__ == "__main__" and "--what" in sys.argv and sys.argv[sys.argv.index("--what") + 1] == "l2pf":
    bench_l2_prefetch()
