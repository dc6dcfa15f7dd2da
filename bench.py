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
METRIC = "offline output tokens/sec (whole box), PP-prefill -> re-shard -> TP-decode"


def _config(args, n: int) -> dict:
    """The workload named in both arms' lines (BASELINE.json configs[1])."""
    return {
        "workload": f"{Path(args.arch).stem} {args.prompts} prompts x {args.input_len} in / {args.output_len} out, "
                    f"prefill tp1.pp{n} -> decode tp{n}.pp1 (BASELINE.json configs[1] shape)",
        "prompts": args.prompts, "input_len": args.input_len, "output_len": args.output_len,
        "parallelism": f"pp{n}->tp{n}", "l2": "inputs >> L2 (weights+KV ~102 GB at N=1); no flush",
        "policy": "transition-min (b200-native: KV kept in HBM, re-sharded over NVLink)",
        "prefill_tokens_per_forward": args.prefill_tokens if n == 1 else "1 prompt per micro-batch",
    }


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


def _arch(name: str):
    """A preset name (PRESETS) or the path of a LlamaArch YAML document."""
    from paper_2503_06433_b200 import PRESETS, load_arch

    if name in PRESETS:
        return PRESETS[name]
    if Path(name).is_file():
        return load_arch(name)
    raise SystemExit(f"--arch {name!r}: not a preset ({', '.join(PRESETS)}) nor a LlamaArch YAML file")


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
    arch = _arch(args.arch)
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
    ar_table = allreduce_table(worker, dev, world, arch)

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
                                  f"one prefill layer ({_gemm_prefill_traffic_file()})",
                "all_gemm_tflops": kern.get("gemm", {}).get("tflops"),
                "peak_source": f"{peaks['source']} bf16_tflops_sustained"}
    da = kern.get("decode_attention", {})
    reshard_s = rep.reshard_time
    line = {
        "metric": METRIC,
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
        "config": dict(_config(args, n), gpu=props.name),
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
        # prompt + output tokens per second beside the output-only metric
        "prompt_plus_output_tokens_per_s": args.prompts * (args.input_len + args.output_len) / mean_t,
    }
    if ar_table is not None:
        line["allreduce_table"] = ar_table
    if n == 1:
        line["reshard_micro"] = reshard_microbench(worker, arch, args, peaks)
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args, arch)
    print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def allreduce_table(worker, dev, world: int, arch, rows: int = 512, iters: int = 20) -> dict | None:
    """Measured all-reduce bandwidth per TP degree for the reference's
    AllReduceTable (specs.py:103-133: time = message bytes / bandwidth(tp),
    non-increasing in tp), on a decode-step message (rows x hidden bf16):
    NCCL all_reduce over ranks [0, d) for d = 2, 4, ... <= world, and the
    fused peer-memory combine (all-reduce + rmsnorm, csrc/tp_allreduce.cu) on
    the decode TP group.  Outside the timed region; device time, max over
    ranks.  None at N = 1 or without NCCL."""
    import torch
    import torch.distributed as dist

    if world < 2 or dist.get_backend() != "nccl":
        return None
    x = torch.zeros(rows, arch.hidden, dtype=torch.bfloat16, device=dev)
    nbytes = x.numel() * 2

    def device_time(fn) -> float:
        for _ in range(5):
            fn()
        torch.cuda.synchronize(dev)
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(iters):
            fn()
        e.record()
        torch.cuda.synchronize(dev)
        return s.elapsed_time(e) / iters / 1e3

    def max_over_ranks(t: float) -> float:
        tt = torch.tensor([t], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        return float(tt.item())

    out: dict = {"msg_bytes": nbytes, "rows": rows, "nccl_s": {}, "nccl_algbw": {}}
    d = 2
    while d <= world:
        grp = dist.new_group(list(range(d)))
        t = device_time(lambda: dist.all_reduce(x, group=grp)) if dist.get_rank() < d else 0.0
        t = max_over_ranks(t)
        out["nccl_s"][d] = t
        out["nccl_algbw"][d] = nbytes / t
        d *= 2
    # the AllReduceTable contract: bandwidth non-increasing in tp
    table, lo = {}, float("inf")
    for k in sorted(out["nccl_algbw"]):
        lo = min(lo, out["nccl_algbw"][k])
        table[k] = lo
    out["allreduce_table"] = table
    ar = next((a for a in worker._tp_arenas.values() if a.usable and a.comm.size == world), None)
    if ar is not None and ar.rows >= rows:
        gamma = torch.ones(arch.hidden, dtype=torch.bfloat16, device=dev)
        t = max_over_ranks(device_time(lambda: ar.combine(rows, gamma, arch.rms_eps)))
        out["fused_combine"] = {"degree": world, "s": t, "algbw": nbytes / t,
                                "note": "all-reduce + the next rmsnorm, one peer-memory kernel"}
    return out


def _gemm_prefill_traffic_file() -> str:
    for r in ("r02", "r01"):
        if (ROOT / "profiles" / r / "ncu_full_gemm_prefill.json").exists():
            return f"profiles/{r}/ncu_full_gemm_prefill.json"
    return "none"


def _gemm_prefill_traffic(arch, args):
    """(mean ncu DRAM bytes per launch, mean algorithmic bytes per launch) of
    the prefill projections.  The DRAM bytes come from the committed ncu
    capture of the bench command; algorithmic = A + B + C (+ residual)."""
    p = next((q for q in (ROOT / "profiles" / r / "ncu_full_gemm_prefill.json" for r in ("r02", "r01")) if q.exists()),
             ROOT / "profiles" / "r01" / "ncu_full_gemm_prefill.json")
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
_SLICE_WEIGHTS: dict = {}


def _slice_weights(arch) -> dict:
    """fp32 weights of ONE layer + final norm + LM head at ``arch``'s shape,
    seeded Gaussians at the init's scales (oracle/llama.py tensor_specs).
    The CPU sample's time depends on the shapes only; drawing them with
    torch on the host keeps the CPU arm free of the GPU and of this repo's
    library (the counter-based init in numpy would take ~90 s for these
    750 M elements)."""
    import torch

    from oracle import llama as lo

    key = (arch.hidden, arch.num_query_heads, arch.num_kv_heads, arch.head_dim, arch.ffn, arch.vocab)
    if key not in _SLICE_WEIGHTS:
        a1 = lo.Arch(1, arch.hidden, arch.num_query_heads, arch.num_kv_heads, arch.head_dim, arch.ffn, arch.vocab,
                     arch.rope_theta, arch.rms_eps)
        g = torch.Generator().manual_seed(0)
        w = {}
        for name, (_, rows, cols, scale) in lo.tensor_specs(a1).items():
            if name == "embed":
                continue  # the sample starts from hidden states: an embedding lookup is a gather
            w[name] = torch.ones(rows, cols) if scale == 0.0 else torch.randn(rows, cols, generator=g) * scale
        _SLICE_WEIGHTS.clear()
        _SLICE_WEIGHTS[key] = (a1, w)
    return _SLICE_WEIGHTS[key]


def cpu_port_sample(arch, s_in: int, ctx: int, batch: int = 8) -> dict:
    """One bounded sample of the CPU port of the path (oracle/llama.py, fp32
    torch on every host thread; no GPU, no repo library):

    * prefill: one prompt of ``s_in`` tokens through one full layer (causal
      attention), then the final norm + LM head of its last token;
    * decode: one decode step of ``batch`` independent sequences at context
      ``ctx`` through one full layer (batched projections and MLP, each
      sequence's attention over its own cache: LlamaOracle.layer_decode_batch),
      then the final norm + LM head of the ``batch`` rows."""
    import torch

    from oracle import llama as lo

    threads = os.cpu_count() or 1
    torch.set_num_threads(threads)
    a1, w = _slice_weights(arch)
    orc = lo.LlamaOracle(a1, seed=0, bf16_faithful=False, max_pos=max(s_in, ctx) + 8, weights=w)
    g = torch.Generator().manual_seed(1)
    hk, d = arch.num_kv_heads, arch.head_dim
    x = torch.randn(s_in, arch.hidden, generator=g)
    caches = [{0: (torch.randn(ctx - 1, hk, d, generator=g), torch.randn(ctx - 1, hk, d, generator=g))}
              for _ in range(batch)]
    xb = torch.randn(batch, arch.hidden, generator=g)
    t0 = time.perf_counter()
    y = orc._layer(x, 0, torch.arange(s_in), {})
    t1 = time.perf_counter()
    logits = orc._norm(y[-1:], w["final_norm"]) @ w["head"].T
    t2 = time.perf_counter()
    yb = orc.layer_decode_batch(xb, 0, torch.full((batch,), ctx - 1), caches)
    t3 = time.perf_counter()
    lb = orc._norm(yb, w["final_norm"]) @ w["head"].T
    t4 = time.perf_counter()
    assert torch.isfinite(logits).all() and torch.isfinite(lb).all()
    return {"prefill_layer_s": t1 - t0, "prefill_head_s": t2 - t1, "decode_layer_s": t3 - t2,
            "decode_head_s": t4 - t3, "threads": threads}


def cpu_extrapolate(arch, args, samples: list[dict], batch: int = 8) -> dict:
    """tokens/s of the whole workload from the per-layer samples: every
    prompt costs L prefill layers + one head row; every decode step of
    ``batch`` sequences costs L decode layers + ``batch`` head rows."""
    P, S_in, S_out, L = args.prompts, args.input_len, args.output_len, arch.num_layers
    mean = {k: sum(s[k] for s in samples) / len(samples) for k in samples[0] if k.endswith("_s")}
    t_prompt = L * mean["prefill_layer_s"] + mean["prefill_head_s"]
    t_step = L * mean["decode_layer_s"] + mean["decode_head_s"]
    total = P * t_prompt + S_out * math.ceil(P / batch) * t_step
    return {"value": P * S_out / total, "unit": "tokens/s", "cores": samples[0]["threads"], "kind": "port",
            "sample": f"per step: one {S_in}-token prompt through one {arch.name} layer + LM head of its last "
                      f"token, and one batch-{batch} decode step at context {S_in + S_out // 2} through one layer "
                      f"+ LM head (oracle/llama.py fp32, seeded weights, {samples[0]['threads']} threads); "
                      f"extrapolated to {P} x {S_in}/{S_out} as P*(L*t_prefill_layer + t_head) + "
                      f"S_out*ceil(P/{batch})*(L*t_decode_layer + t_head{batch})",
            "per_layer_s": mean, "extrapolated_batch_s": total}


def cpu_baseline(args, arch) -> dict:
    """The CPU port on one bounded sample (rank 0, N=1; reported beside the
    GPU line, not the target)."""
    cpu_port_sample(arch, 64, 64)  # first-touch warm-up of the weights and the thread pool
    s = cpu_port_sample(arch, args.input_len, args.input_len + args.output_len // 2)
    return cpu_extrapolate(arch, args, [s])


def reference_simulator(args, arch, n: int) -> dict:
    """The reference's own CPU path, UNMODIFIED: shardsim.simulate() from
    baseline/_ref (sim.py:748-761) on the same workload and layouts, with a
    B200 HardwareSpec from the measured peaks; single-threaded Python.  It
    predicts (models) the batch; its wall time is the reference's CPU cost of
    the path, and its replay_check validates its own log."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "shardsim").is_dir():
        return {"unavailable": "baseline/_ref (the reference install) is absent"}
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    import shardsim as ss

    peaks = _peaks()
    spec = arch.model_spec()
    model = ss.ModelSpec(num_layers=spec.num_layers, params_per_layer=spec.params_per_layer,
                         num_query_heads=spec.num_query_heads, num_kv_heads=spec.num_kv_heads,
                         head_dim=spec.head_dim, bytes_per_param=spec.bytes_per_param)
    hw = ss.HardwareSpec(num_gpus=n, hbm_bandwidth=peaks["hbm_gbs"] * 1e9, peak_flops=peaks["bf16_tflops"] * 1e12,
                         gpu_memory=_gpu_memory_bytes(), host_memory_per_gpu=256e9, host_link_bandwidth=64e9,
                         allreduce=ss.RingAllReduce(770e9))
    reqs = [ss.Request(i, args.input_len, args.output_len) for i in range(args.prompts)]
    cfg_p, cfg_d = ss.ParallelismConfig(1, n, 1), ss.ParallelismConfig(n, 1, 1)
    t0 = time.perf_counter()
    rep = ss.simulate(model, hw, reqs, ss.SchedulingPolicy.TRANSITION_MINIMIZING, cfg_p, cfg_d)
    wall = time.perf_counter() - t0
    verdict = ss.replay_check(rep)
    return {"module": ss.__file__.replace(str(ROOT) + "/", ""), "wall_s": wall, "cores": 1,
            "predicted_tokens_per_s": rep.tokens_per_second, "predicted_makespan_s": rep.makespan,
            "transitions": rep.transitions, "events": len(rep.event_log), "replay_check": bool(verdict),
            "hardware": f"B200 spec from {peaks['source']} peaks, {n} GPU(s)"}


def _gpu_memory_bytes() -> float:
    """Per-GPU HBM capacity, without touching CUDA (nvidia-smi), else 180 GB."""
    try:
        out = subprocess.run(["nvidia-smi", "--id=0", "--query-gpu=memory.total", "--format=csv,noheader,nounits"],
                             capture_output=True, text=True, timeout=30).stdout.strip()
        return float(out.splitlines()[0]) * 2**20
    except (OSError, ValueError, IndexError, subprocess.TimeoutExpired):
        return 180e9


# ------------------------------------------------------------ reference --
def run_reference(args) -> None:
    """The reference arm: the CPU implementation of the path on the host
    cores (the oracle port — the reference has no numeric path), rank 0
    only, no GPU and no repo library; plus the reference's own simulate()
    timed from baseline/_ref."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    arch = _arch(args.arch)
    n = args.gpus
    ctx = args.input_len + args.output_len // 2
    samples, walls = [], []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        smp = cpu_port_sample(arch, args.input_len, ctx)
        if i >= args.warmup:
            samples.append(smp)
            walls.append(time.perf_counter() - t0)
    cb = cpu_extrapolate(arch, args, samples)
    v = cb["value"]
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": v, "unit": "tokens/s", "n_gpus": n, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": sum(walls) / len(walls) * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded weights and activations of the shape)",
        "config": _config(args, n),
        "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": cb["cores"], "kind": "port", "sample": cb["sample"]},
        "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "per_layer_s": cb["per_layer_s"],
        "reference_simulator": reference_simulator(args, arch, n),
        "note": "the reference (shardsim) is an analytic simulator with no numeric path; the CPU implementation "
                "of the path is the oracle port (oracle/llama.py), timed per layer and extrapolated; "
                "reference_simulator times the reference's own simulate() on the same workload",
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
