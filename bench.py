"""Benchmark: offline PP-prefill -> NVLink re-shard -> TP-decode throughput.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One *step* is one complete offline batch through the public API
(``execute()``): BASELINE.json configs[1] — Llama-3-8B shape, random-init bf16,
512 prompts x 1024 in / 256 out — prefilled under PP=N, re-sharded (weights +
KV over NVLink) and decoded under TP=N on N GPUs of one node (N=1: the same
batch on one GPU, the re-shard degenerates to the identity).  The metric is
the reference's: output tokens / makespan (sim.py:720, :736), whole box.

Timing: W untimed warm-up batches, then K timed batches, each bracketed by a
barrier + cuda synchronize, device-timed with CUDA events on the launching
stream, max over ranks.  Inputs (16 GB weights + 86 GB KV at N=1) are far
larger than L2, so no flush is needed.  ``value`` uses prompt ids already in
HBM; ``e2e`` runs the same API with prompts in pinned host memory (H2D inside
the timed region) and reads every generated token back (D2H).

For N>1 the driver launches this file under torchrun (one process per GPU,
NCCL).  ``--impl reference`` times the CPU restatement of the path (the
reference shardsim has no executable numeric path) on the
host cores, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOAD = {"arch": "llama3-8b", "prompts": 512, "input_len": 1024, "output_len": 256}


def _peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": d["hbm_gbs"], "bf16_tflops": d["bf16_tflops"],
                "bf16_tflops_sustained": d.get("bf16_tflops_sustained", d["bf16_tflops"]), "source": "measured"}
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "source": "fallback"}


class ClockSampler:
    """nvidia-smi clocks/throttle sampling during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int) -> None:
        self.index = index
        self.rows: list[list[str]] = []
        self.proc = None
        self.thread = None

    def start(self) -> None:
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return

        def pump():
            for line in self.proc.stdout:
                self.rows.append([x.strip() for x in line.split(",")])

        self.thread = threading.Thread(target=pump, daemon=True)
        self.thread.start()

    def stop(self) -> dict:
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.thread is not None:
            self.thread.join(timeout=2)
        rows = [r for r in self.rows if len(r) >= 9]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = sorted(float(r[1]) for r in rows if r[1].replace(".", "").isdigit())
        mx = max(float(r[2]) for r in rows if r[2].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v.strip().lower() == "active"})
        loaded = [x for x in sm if x > 0.5 * mx] or sm
        return {"sm_mhz": loaded[len(loaded) // 2], "sm_max_mhz": mx, "reasons": reasons, "samples": len(rows),
                "power_w_max": max(float(r[3]) for r in rows if r[3].replace(".", "").isdigit())}


# ------------------------------------------------------------------ ours --
def run_ours(args) -> None:
    import torch

    from paper_2503_06433_b200 import PRESETS, ParallelismConfig, Request, SchedulingPolicy, execute, replay_check
    from paper_2503_06433_b200 import _lib
    from paper_2503_06433_b200.comm import SoloComm, TorchComm
    from paper_2503_06433_b200.engine import synthetic_prompts
    from paper_2503_06433_b200.runtime import Worker
    from paper_2503_06433_b200.specs import HardwareSpec, RingAllReduce

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    n = args.gpus
    if world != n:
        raise SystemExit(f"--gpus {n} but WORLD_SIZE={world}")
    # one GPU per rank; ranks beyond the device count share GPUs (gloo test runs)
    local = local % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist

        # SSB_DIST_BACKEND=gloo: ranks sharing one GPU (the multi-rank path
        # exercised on a single-GPU box; TorchComm stages CUDA tensors through
        # host memory) -- never the measured configuration
        backend = os.environ.get("SSB_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
        comm = TorchComm()
    else:
        comm = SoloComm()
    arch = PRESETS[args.arch]
    model = arch.model_spec()
    props = torch.cuda.get_device_properties(dev)
    peaks = _peaks()
    hw = HardwareSpec(num_gpus=n, hbm_bandwidth=peaks["hbm_gbs"] * 1e9, peak_flops=peaks["bf16_tflops"] * 1e12,
                      gpu_memory=float(props.total_memory), host_memory_per_gpu=256e9, host_link_bandwidth=64e9,
                      allreduce=RingAllReduce(770e9))
    cfg_p = ParallelismConfig(1, n, 1)
    cfg_d = ParallelismConfig(n, 1, 1)
    reqs = [Request(i, args.input_len, args.output_len) for i in range(args.prompts)]
    prompts_np = synthetic_prompts(reqs, arch.vocab)
    prompts_dev = [torch.from_numpy(p).to(dev) for p in prompts_np]
    prompts_pinned = [torch.from_numpy(p).pin_memory() for p in prompts_np]
    worker = Worker(arch, comm, 1, dev, seed=0, max_pos=args.input_len + args.output_len + 64)

    def one(prompts):
        return execute(model, hw, reqs, SchedulingPolicy.TRANSITION_MINIMIZING, cfg_p, cfg_d, arch=arch,
                       prompts=prompts, comm=comm, device=dev, worker=worker, max_prefill_tokens=args.prefill_tokens)

    def timed(prompts, k, nvtx=None):
        times, reports = [], []
        for _ in range(k):
            comm.barrier()
            torch.cuda.synchronize(dev)
            s = torch.cuda.Event(enable_timing=True)
            e = torch.cuda.Event(enable_timing=True)
            if nvtx:  # ncu --nvtx --nvtx-include "<name>/" selects exactly these launches
                torch.cuda.nvtx.range_push(nvtx)
            s.record()
            rep = one(prompts)
            e.record()
            if nvtx:
                torch.cuda.nvtx.range_pop()
            comm.barrier()
            torch.cuda.synchronize(dev)
            times.append(s.elapsed_time(e) / 1e3)
            reports.append(rep)
        t = torch.tensor(times, dtype=torch.float64, device=dev)
        if world > 1:
            import torch.distributed as dist

            if dist.get_backend() == "gloo":
                t = t.cpu()
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t.tolist(), reports

    # warm-up (also initialises weights/pool and JIT-free kernels)
    timed(prompts_dev, args.warmup)
    sampler = ClockSampler(local)
    sampler.start()
    launches0 = _lib.STATS.count
    times, reports = timed(prompts_dev, args.steps, nvtx="timed_step")
    launches = (_lib.STATS.count - launches0) // max(args.steps, 1)
    clocks = sampler.stop()
    e2e_times, e2e_reports = timed(prompts_pinned, max(1, min(args.steps, 2)))
    # per-kernel shares inside one instrumented batch
    kern = profile_kernels(one, prompts_dev, arch, args, dev, comm, world)

    out_tokens = args.prompts * args.output_len
    mean_t = sum(times) / len(times)
    value = out_tokens / mean_t
    e2e_t = sum(e2e_times) / len(e2e_times)
    rep = reports[-1]
    verdict = replay_check(rep)
    if rank != 0:
        if world > 1:
            import torch.distributed as dist

            dist.destroy_process_group()
        return
    # roofline of the dominant kernel: the tcgen05 GEMM on the prefill
    # projections (tensor-bound; the largest share of the batch)
    g = kern.get("gemm_prefill", {})
    peak = peaks["bf16_tflops_sustained"]
    achieved = g.get("tflops")
    traffic, alg_bytes = _gemm_prefill_traffic(arch, args)
    roofline = {"bound": "tensor", "kernel": "gemm_bf16_sm100 (tcgen05), prefill projections at M=16384 tokens",
                "achieved": achieved, "peak": peak,
                "unit": "TFLOP/s", "frac": (achieved / peak) if achieved else None, "traffic": traffic,
                "traffic_algorithmic_bytes": alg_bytes,
                "traffic_source": "ncu --set full, DRAM read+write bytes per launch, mean of the 4 projections of "
                                  "one prefill layer (profiles/r01/ncu_full_gemm_prefill.json)",
                "all_gemm_tflops": kern.get("gemm", {}).get("tflops"),
                "peak_source": f"{peaks['source']} bf16_tflops_sustained"}
    da = kern.get("decode_attention", {})
    reshard_s = rep.reshard_time
    line = {
        "metric": "offline output tokens/sec (whole box), PP-prefill -> re-shard -> TP-decode",
        "value": value,
        "unit": "tokens/s",
        "n_gpus": n,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": mean_t * 1e3,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (random-init weights, uniform prompt ids seed 1)",
        "config": {
            "workload": f"{args.arch} {args.prompts} prompts x {args.input_len} in / {args.output_len} out, "
                        f"prefill tp1.pp{n} -> decode tp{n}.pp1 (BASELINE.json configs[1] shape)",
            "prompts": args.prompts, "input_len": args.input_len, "output_len": args.output_len,
            "parallelism": f"pp{n}->tp{n}", "l2": "inputs >> L2 (weights+KV ~102 GB at N=1); no flush",
            "policy": "transition-min (b200-native: KV kept in HBM, re-sharded over NVLink)",
            "prefill_tokens_per_forward": args.prefill_tokens if n == 1 else "1 prompt per micro-batch",
            "gpu": props.name,
        },
        "e2e": {"value": out_tokens / e2e_t, "unit": "tokens/s",
                "h2d_bytes_per_step": int(sum(p.numel() * 4 for p in prompts_pinned)),
                "d2h_bytes_per_step": int(args.prompts * (args.output_len + 1) * 4)},
        "gpu_launches": launches,
        "roofline": roofline,
        "kernels": kern,
        "phases_s": {"prefill": rep.prefill_time, "reshard": reshard_s, "decode": rep.decode_time,
                     "other": rep.stalled_transfer_time, "makespan": rep.makespan},
        "reshard": {"bytes_sent_per_gpu": rep.measured.get("reshard_bytes_sent"),
                    "wall_s": reshard_s,
                    "gbs_per_gpu": (rep.measured.get("reshard_bytes_sent", 0) / reshard_s / 1e9) if reshard_s else None,
                    "share_of_e2e": reshard_s / rep.makespan},
        "replay_check": bool(verdict),
        "reference_model_prediction": _predict(model, hw, cfg_p, cfg_d, args),
        "clocks": clocks,
        "decode_attention_hbm_frac": (da.get("gbs", 0) / peaks["hbm_gbs"]) if da else None,
    }
    if n == 1:
        line["reshard_micro"] = reshard_microbench(worker, arch, args, peaks)
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args, arch, sample_in=args.cpu_sample_in)
    print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def _gemm_prefill_traffic(arch, args):
    """(mean ncu DRAM bytes per launch, mean algorithmic bytes per launch) of
    the prefill projections.  The DRAM bytes come from the committed ncu
    capture of the bench command; algorithmic = A + B + C (+ residual)."""
    p = ROOT / "profiles" / "r01" / "ncu_full_gemm_prefill.json"
    traffic = None
    if p.exists():
        rows = json.loads(p.read_text())
        unit = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}

        def val(x):
            v, u = x.split()
            return float(v) * unit[u]

        b = [val(r["dram__bytes_read.sum"]) + val(r["dram__bytes_write.sum"]) for r in rows]
        traffic = sum(b) / len(b) if b else None
    M, H, F = min(args.prefill_tokens, args.prompts * args.input_len), arch.hidden, arch.ffn
    qkv = (arch.num_query_heads + 2 * arch.num_kv_heads) * arch.head_dim
    alg = [M * H + qkv * H + M * qkv, M * H + H * H + 2 * M * H, M * H + 2 * F * H + M * F, M * F + H * F + 2 * M * H]
    return traffic, 2.0 * sum(alg) / len(alg)


def _predict(model, hw, cfg_p, cfg_d, args) -> dict:
    """The reference's analytic model (perf.py restated) on the same B200
    HardwareSpec: what shardsim.simulate would charge for this batch."""
    from paper_2503_06433_b200.perf import predict_phases

    p = predict_phases(model, hw, cfg_p, cfg_d, args.input_len, args.output_len, args.prompts)
    p["tokens_per_s"] = args.prompts * args.output_len / (p["prefill_s"] + p["decode_s"])
    return p


def reshard_microbench(worker, arch, args, peaks, sweep=(2, 4, 8)) -> dict:
    """BASELINE configs[4] on one GPU: the per-GPU re-shard work of the 8B
    batch at PP{g}->TP{g} for g in 2/4/8 — KV (every resident block of one
    GPU: pack into per-peer staging, unpack from staging into the decode
    geometry) and weights (copy2d pack of the pieces every peer needs, unpack
    of the pieces this GPU receives) — timed per kernel with CUDA events.  The
    NVLink transfer between them needs peers; at N=1 it is absent, so this
    reports the pack/unpack HBM rate and the per-GPU NVLink floor the transfer
    would have (bytes leaving the GPU / 770 GB/s measured peer bandwidth)."""
    import torch

    from paper_2503_06433_b200 import ops
    from paper_2503_06433_b200.layout import kv_geometry, repartition_pieces, weight_layout
    from paper_2503_06433_b200.reshard import kv_exchange
    from paper_2503_06433_b200.runtime import _copy_desc_rows
    from paper_2503_06433_b200.specs import ParallelismConfig

    dev = worker.device
    bs = 64
    cell = 2 * bs * arch.head_dim
    chunk = 256

    def timed(fns):
        for f in fns[:2]:
            f()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for f in fns:
            f()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / 1e3

    rows = []
    for gpus in [g for g in sweep if arch.num_layers % g == 0 and arch.num_kv_heads % g == 0]:
        # every GPU holds every block of the batch, sliced to its layers (PP)
        # or heads (TP): the per-GPU pool is 1/g of the batch's KV
        nb = args.prompts * (-(-(args.input_len + args.output_len) // bs))
        src = kv_geometry(arch, 1, gpus, nb, bs)
        dst = kv_geometry(arch, gpus, 1, nb, bs)
        need = nb * src.block_elems
        pool = worker.pool[:need] if worker.pool is not None and worker.pool.numel() >= need else \
            torch.empty(need, dtype=torch.bfloat16, device=dev)
        ex = kv_exchange(arch.model_spec(), ParallelismConfig(1, gpus, 1), ParallelismConfig(gpus, 1, 1), 0)
        stage = torch.empty(chunk * src.block_elems + 8, dtype=torch.bfloat16, device=dev)

        def peers(rects, nid):
            out, off = [], 0
            for r in rects:
                out.append((r.l0, r.nl, r.h0, r.nh, off * 2))
                off += nid * r.cells * cell
            return out

        ids_all = torch.arange(nb, dtype=torch.int32, device=dev)
        chunks = [ids_all[c : c + chunk] for c in range(0, nb, chunk)]
        t_pack = timed([lambda ids=ids: ops.kv_reshard_pack(pool, src.as_tuple(), ids, peers(ex.send, ids.numel()),
                                                            stage) for ids in chunks])
        t_unpack = timed([lambda ids=ids: ops.kv_reshard_unpack(pool, dst.as_tuple(), ids,
                                                                peers(ex.recv, ids.numel()), stage) for ids in chunks])
        kv_bytes = need * 2
        kv_leaving = kv_bytes * (gpus - 1) // gpus
        # weights: GPU 0's pieces for every peer (pack) and from every peer (unpack)
        old = [weight_layout(arch, 1, gpus, q) for q in range(gpus)]
        new = [weight_layout(arch, gpus, 1, q) for q in range(gpus)]
        send, recv, s_pos, r_pos, w_leaving = [], [], 0, 0, 0
        for q in range(gpus):
            for pc in repartition_pieces(old[0], new[q]):
                send.append((pc.src_off * 2, s_pos * 2, pc.src_ld * 2, pc.cols * 2, pc.rows, pc.cols * 2))
                s_pos += pc.numel
                w_leaving += 2 * pc.numel if q else 0
            for pc in repartition_pieces(old[q], new[0]):
                recv.append((r_pos * 2, pc.dst_off * 2, pc.cols * 2, pc.dst_ld * 2, pc.rows, pc.cols * 2))
                r_pos += pc.numel
        a_old = torch.empty(old[0].arena_elems, dtype=torch.bfloat16, device=dev)
        a_new = torch.empty(new[0].arena_elems, dtype=torch.bfloat16, device=dev)
        sbuf = torch.empty(max(s_pos, 8), dtype=torch.bfloat16, device=dev)
        rbuf = torch.empty(max(r_pos, 8), dtype=torch.bfloat16, device=dev)
        sd, stot = _copy_desc_rows(send)
        rd, rtot = _copy_desc_rows(recv)
        sd_d, rd_d = torch.from_numpy(sd).to(dev), torch.from_numpy(rd).to(dev)
        t_wpack = timed([lambda: ops.copy2d_batched(a_old, sbuf, sd_d, stot)] * 3) / 3
        t_wunpack = timed([lambda: ops.copy2d_batched(rbuf, a_new, rd_d, rtot)] * 3) / 3
        leaving = kv_leaving + w_leaving
        rows.append({
            "gpus": gpus, "transition": f"pp{gpus}->tp{gpus}",
            "kv_bytes_per_gpu": kv_bytes, "kv_bytes_leaving": kv_leaving,
            "weight_bytes_per_gpu": 2 * old[0].arena_elems, "weight_bytes_leaving": w_leaving,
            "kv_pack_s": t_pack, "kv_unpack_s": t_unpack, "w_pack_s": t_wpack, "w_unpack_s": t_wunpack,
            "kv_pack_hbm_gbs": 2 * kv_bytes / t_pack / 1e9, "kv_unpack_hbm_gbs": 2 * kv_bytes / t_unpack / 1e9,
            "w_pack_hbm_gbs": 2 * 2 * s_pos / t_wpack / 1e9, "w_unpack_hbm_gbs": 2 * 2 * r_pos / t_wunpack / 1e9,
            "kv_pack_hbm_frac": 2 * kv_bytes / t_pack / 1e9 / peaks["hbm_gbs"],
            "kv_unpack_hbm_frac": 2 * kv_bytes / t_unpack / 1e9 / peaks["hbm_gbs"],
            "bytes_leaving_gpu": leaving, "nvlink_floor_s": leaving / 770e9,
            "pack_unpack_s_vs_nvlink_floor": (t_pack + t_unpack + t_wpack + t_wunpack) / (leaving / 770e9),
        })
        del pool, stage, a_old, a_new, sbuf, rbuf
    return {
        "workload": f"{arch.name} weights + KV of {args.prompts}x{args.input_len + args.output_len} tokens, "
                    f"per-GPU share at PP{{g}}->TP{{g}} (BASELINE configs[4])",
        "sweep": rows,
        "note": "transfer over NVLink not measurable with 1 GPU; pack of chunk i+1 and unpack of chunk i-1 overlap "
                "the all-to-all of chunk i, so the transition is bound by max(pack+unpack, NVLink floor)",
    }


def profile_kernels(one, prompts, arch, args, dev, comm, world) -> dict:
    """One instrumented batch: every library launch bracketed by CUDA events
    on its stream; per-kernel time share, algorithmic FLOPs/bytes and rates."""
    import torch

    from paper_2503_06433_b200 import _lib

    def tagger(name, a):
        # every tcgen05 GEMM launch (plain, QKV+RoPE+KV-append, LM head+argmax)
        # by phase: decode projections run at M = resident batch (<= prompts),
        # prefill at packed tokens (the prefill LM head at M = prompts of a
        # micro-batch is counted with decode: same skinny shape class)
        if name in ("ssb_gemm_bf16", "ssb_gemm_bf16_ws", "ssb_gemm_bf16_rn"):
            M, N, K = a[4], a[5], a[6]
        elif name == "ssb_gemm_qkv_rope_kv":
            M, K = a[3], a[4]
            N = (a[8] + 2 * a[9]) * a[10]
        elif name == "ssb_gemm_lm_head_argmax":
            M, N, K = a[2], a[3], a[4]
        else:
            return name.replace("ssb_", ""), 0, 0
        return ("gemm_prefill" if M > args.prompts else "gemm_decode"), 2.0 * M * N * K, 0

    _lib.STATS.records = []
    _lib.STATS.tagger = tagger
    _lib.STATS.timing = True
    comm.barrier()
    torch.cuda.synchronize(dev)
    s = torch.cuda.Event(enable_timing=True)
    e = torch.cuda.Event(enable_timing=True)
    s.record()
    one(prompts)
    e.record()
    torch.cuda.synchronize(dev)
    _lib.STATS.timing = False
    total = s.elapsed_time(e) / 1e3
    agg: dict = {}
    for tag, a, b, fl, by in _lib.STATS.records:
        d = agg.setdefault(tag, {"launches": 0, "s": 0.0, "flops": 0.0})
        d["launches"] += 1
        d["s"] += a.elapsed_time(b) / 1e3
        d["flops"] += fl
    _lib.STATS.records = []
    g = {"launches": 0, "s": 0.0, "flops": 0.0}
    for tag in ("gemm_prefill", "gemm_decode"):
        for k in g:
            g[k] += agg.get(tag, {}).get(k, 0)
    if g["launches"]:
        agg["gemm"] = g
    # algorithmic bytes of decode attention: every step reads ctx tokens of K and V per layer
    n = world
    kv_tok_layer = 2 * (arch.num_kv_heads // n) * arch.head_dim * 2
    ctx_sum = sum(args.input_len + k for k in range(1, args.output_len + 1)) * args.prompts
    dec_bytes = ctx_sum * kv_tok_layer * arch.num_layers
    out = {"_batch_s": total}
    for tag, d in sorted(agg.items(), key=lambda kv: -kv[1]["s"]):
        r = {"launches": d["launches"], "s": d["s"], "share": d["s"] / total}
        if tag == "gemm":
            r["note"] = "all tcgen05 GEMM launches (= gemm_prefill + gemm_decode)"
        if d["flops"]:
            r["tflops"] = d["flops"] / d["s"] / 1e12
        if tag == "decode_attention":
            r["bytes"] = dec_bytes
            r["gbs"] = dec_bytes / d["s"] / 1e9
        out[tag] = r
    return out


# ------------------------------------------------------- CPU baseline --
_CPU_WEIGHTS: dict = {}


def cpu_baseline(args, arch, sample_in: int = 256, batch: int = 8) -> dict:
    """The CPU restatement (oracle/llama.py, fp32 torch, all host threads) on
    a bounded sample of the workload: one prompt of ``sample_in`` tokens
    through the full model (prefill cost per token), then one decode step of
    ``batch`` new tokens (the GEMM shapes of a batch-``batch`` decode step).
    Extrapolated to the whole batch: T = P*S_in*t_tok + S_out*(P/batch)*t_step,
    value = P*S_out / T (GEMM-dominated, linear in tokens)."""
    import torch

    from oracle import llama as lo

    threads = os.cpu_count() or 1
    torch.set_num_threads(threads)
    oa = lo.Arch(arch.num_layers, arch.hidden, arch.num_query_heads, arch.num_kv_heads, arch.head_dim, arch.ffn,
                 arch.vocab, arch.rope_theta, arch.rms_eps)
    if arch.name not in _CPU_WEIGHTS:
        _CPU_WEIGHTS[arch.name] = _cpu_weights(arch)
    orc = lo.LlamaOracle(oa, seed=0, bf16_faithful=False, max_pos=sample_in + batch + 8,
                         weights=_CPU_WEIGHTS[arch.name])
    prompt = np.random.default_rng(1).integers(0, arch.vocab, size=sample_in).astype(np.int64)
    cache: dict = {}
    t0 = time.perf_counter()
    orc.tp, orc._decoding = 1, False
    logits = orc._forward(torch.from_numpy(prompt), torch.arange(sample_in), cache)
    t1 = time.perf_counter()
    tok = int(torch.argmax(logits))
    orc._forward(torch.full((batch,), tok), torch.arange(sample_in, sample_in + batch), cache)
    t2 = time.perf_counter()
    t_tok = (t1 - t0) / sample_in
    t_step = t2 - t1
    P, S_in, S_out = args.prompts, args.input_len, args.output_len
    total = P * S_in * t_tok + S_out * (P / batch) * t_step
    return {"value": P * S_out / total, "unit": "tokens/s", "cores": threads, "kind": "port",
            "sample": f"1 prompt x {sample_in} tokens prefilled + one {batch}-token decode step through all "
                      f"{arch.num_layers} layers of {arch.name} (oracle/llama.py fp32 on bf16 weights); "
                      f"extrapolated to {P} x {S_in}/{S_out} as P*S_in*t_tok + S_out*(P/{batch})*t_step",
            "measured_prefill_s": t1 - t0, "measured_decode_step_s": t_step}


def _cpu_weights(arch):
    """bf16 weights for the CPU restatement, generated by the counter-based
    init on the GPU when one is present (bit-identical to oracle.init_model,
    which would take minutes in numpy at 8B), else by the oracle itself."""
    import torch

    from oracle import llama as lo

    names = list(lo.tensor_specs(lo.Arch(arch.num_layers, arch.hidden, arch.num_query_heads, arch.num_kv_heads,
                                         arch.head_dim, arch.ffn, arch.vocab, arch.rope_theta)).keys())
    if not torch.cuda.is_available():
        return None
    from paper_2503_06433_b200.comm import SoloComm
    from paper_2503_06433_b200.runtime import Worker
    from paper_2503_06433_b200.specs import ParallelismConfig

    w = Worker(arch, SoloComm(), 1, torch.device("cuda", torch.cuda.current_device()), seed=0, max_pos=64)
    w.init_weights(ParallelismConfig(1, 1, 1))
    out = {}
    h, d = arch.hidden, arch.head_dim
    nq, nk = arch.num_query_heads, arch.num_kv_heads
    for name in names:
        if name.startswith("L"):
            layer, key = name.split(".", 1)
            p = layer + "."
            if key in ("wq", "wk", "wv"):
                t = w.w(p + "wqkv")
                r0 = {"wq": 0, "wk": nq * d, "wv": (nq + nk) * d}[key]
                r1 = r0 + (nq * d if key == "wq" else nk * d)
                out[name] = t[r0:r1].cpu()
            elif key in ("w1", "w3"):
                t = w.w(p + "w13").view(-1, 2, 32, h)
                out[name] = t[:, 0 if key == "w1" else 1].reshape(-1, h).cpu()
            else:
                out[name] = w.w(p + key).cpu().reshape(-1)[: w.w(p + key).numel()].view(w.w(p + key).shape)
        else:
            out[name] = w.w(name).cpu()
    del w
    torch.cuda.empty_cache()
    return _F32View(out)


class _F32View(dict):
    """bf16 tensors handed to the oracle as fp32 on access (keeps host RAM at 2 B/param)."""

    def __getitem__(self, k):
        return dict.__getitem__(self, k).float()


# ------------------------------------------------------------ reference --
def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2503_06433_b200 import PRESETS

    arch = PRESETS[args.arch]
    import torch

    vals = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        cb = cpu_baseline(args, arch, sample_in=args.cpu_sample_in)
        if i >= args.warmup:
            vals.append((cb, time.perf_counter() - t0))
    v = sum(c["value"] for c, _ in vals) / len(vals)
    step_s = sum(t for _, t in vals) / len(vals)
    c0 = vals[-1][0]
    line = {
        "impl": "reference",
        "metric": "offline output tokens/sec (whole box), PP-prefill -> re-shard -> TP-decode",
        "value": v, "unit": "tokens/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": step_s * 1e3, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": f"{args.arch} {args.prompts} prompts x {args.input_len} in / {args.output_len} out",
                   "note": "reference shardsim is an analytic simulator with no numeric path; its CPU "
                           "implementation of the path is the oracle restatement (oracle/llama.py)"},
        "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": c0["cores"], "kind": "port", "sample": c0["sample"]},
        "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--arch", default=WORKLOAD["arch"])
    ap.add_argument("--prompts", type=int, default=WORKLOAD["prompts"])
    ap.add_argument("--input-len", type=int, default=WORKLOAD["input_len"])
    ap.add_argument("--output-len", type=int, default=WORKLOAD["output_len"])
    ap.add_argument("--prefill-tokens", type=int, default=16384)
    ap.add_argument("--cpu-sample-in", type=int, default=256)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
