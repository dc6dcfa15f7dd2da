"""Generate the golden fixtures of tests/golden/ by running the REFERENCE
(shardsim, imported read-only from /root/reference/pkg/src) in this container.

    python tests/golden/make_golden.py

The fixtures pin the restated config/planning API and the CPU oracle to the
reference's own outputs; /root/reference does not exist on the GPU box, so the
tests read only these JSON files.
"""

from __future__ import annotations

import json
import random
import sys
from pathlib import Path

sys.dont_write_bytecode = True
REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))

import shardsim  # noqa: E402
from shardsim import (  # noqa: E402
    ConfigError,
    HardwareSpec,
    KVLayout,
    ModelSpec,
    ParallelismConfig,
    Request,
    RingAllReduce,
    SchedulingPolicy,
    SimOptions,
    kv_bytes_per_token,
    max_batch_size,
    replay_check,
    simulate,
    total_weight_bytes,
    validate_config,
)
from shardsim.reshard import contiguous_runs, kv_reshard_route, shard_map, weight_reload_plan  # noqa: E402

OUT = Path(__file__).resolve().parent
GiB = 1024**3


def model_doc(m: ModelSpec) -> dict:
    return dict(num_layers=m.num_layers, params_per_layer=m.params_per_layer, num_query_heads=m.num_query_heads,
                num_kv_heads=m.num_kv_heads, head_dim=m.head_dim, bytes_per_param=m.bytes_per_param,
                activation_bytes_per_token=m.activation_bytes_per_token,
                allreduces_per_layer=m.allreduces_per_layer)


def hw_doc(h: HardwareSpec) -> dict:
    return dict(num_gpus=h.num_gpus, hbm_bandwidth=h.hbm_bandwidth, peak_flops=h.peak_flops,
                gpu_memory=h.gpu_memory, host_memory_per_gpu=h.host_memory_per_gpu,
                host_link_bandwidth=h.host_link_bandwidth,
                allreduce_model={"kind": "ring", "interconnect_bandwidth": h.allreduce.interconnect_bandwidth})


def random_cases(n: int, seed: int):
    rnd = random.Random(seed)
    cases = []
    for _ in range(n):
        h_kv = rnd.choice([2, 4, 8])
        layers = rnd.choice([4, 8, 12, 24])
        m = ModelSpec(num_layers=layers, params_per_layer=rnd.randint(1_000, 10_000_000), num_query_heads=h_kv * 2,
                      num_kv_heads=h_kv, head_dim=rnd.choice([16, 64]))
        tp = rnd.choice([t for t in (1, 2, 4, 8) if h_kv % t == 0])
        pp = rnd.choice([p for p in (1, 2, 4) if layers % p == 0])
        dp = rnd.choice([1, 2])
        cases.append((m, ParallelismConfig(tp, pp, dp)))
    return cases


# the BASELINE.json shapes (params_per_layer = total/L)
SHAPES = {
    "tiny": ModelSpec(num_layers=2, params_per_layer=1_114_752, num_query_heads=4, num_kv_heads=4, head_dim=64),
    "llama3-8b": ModelSpec(num_layers=32, params_per_layer=250_945_664, num_query_heads=32, num_kv_heads=8,
                           head_dim=128),
    "llama2-13b": ModelSpec(num_layers=40, params_per_layer=325_396_608, num_query_heads=40, num_kv_heads=40,
                            head_dim=128),
    "llama3-70b": ModelSpec(num_layers=80, params_per_layer=881_921_332, num_query_heads=64, num_kv_heads=8,
                            head_dim=128),
}


def b200_fleet(n: int) -> HardwareSpec:
    return HardwareSpec(num_gpus=n, hbm_bandwidth=8e12, peak_flops=2.25e15, gpu_memory=180e9,
                        host_memory_per_gpu=256e9, host_link_bandwidth=64e9, allreduce=RingAllReduce(9e11))


def planning_golden() -> dict:
    out = {"shard_map": [], "weight_reload": [], "kv_route": [], "scalars": [], "contiguous_runs": [],
           "parse": [], "validate": []}
    cases = random_cases(120, 7)
    for name, m in SHAPES.items():
        for tp, pp in [(1, 1), (1, 2), (2, 1), (1, 4), (4, 1), (1, 8), (8, 1), (2, 2), (2, 4), (4, 2)]:
            if m.num_kv_heads % tp == 0 and m.num_layers % pp == 0:
                cases.append((m, ParallelismConfig(tp, pp, 1)))
    for m, cfg in cases:
        sm = shard_map(m, cfg)
        out["shard_map"].append({"model": model_doc(m), "cfg": [cfg.tp, cfg.pp, cfg.dp],
                                 "shards": [[s.gpu_id, s.replica_id, s.layer_begin, s.layer_end, s.kv_head_begin,
                                             s.kv_head_end, s.weight_bytes] for s in sm.shards],
                                 "table": sm.table()})
        hw = b200_fleet(cfg.num_gpus)
        for other in [ParallelismConfig(1, cfg.tp * cfg.pp, cfg.dp), ParallelismConfig(cfg.tp * cfg.pp, 1, cfg.dp),
                      cfg]:
            try:
                plan = weight_reload_plan(m, hw, cfg, other)
                res = {"bytes": list(plan.bytes_per_gpu), "wall": plan.wall_time}
            except ConfigError as e:
                res = {"error": type(e).__name__}
            out["weight_reload"].append({"model": model_doc(m), "hw": hw_doc(hw), "old": [cfg.tp, cfg.pp, cfg.dp],
                                         "new": [other.tp, other.pp, other.dp], "result": res})
            for seq in (1, 17, 1024):
                try:
                    route = kv_reshard_route(m, cfg, other, seq)
                    res = {"out": [[d.gpu_id, d.layer_begin, d.layer_end, d.kv_head_begin, d.kv_head_end, d.bytes]
                                   for d in route.swap_out],
                           "in": [[d.gpu_id, d.layer_begin, d.layer_end, d.kv_head_begin, d.kv_head_end, d.bytes]
                                  for d in route.swap_in]}
                except (ConfigError, ValueError) as e:
                    res = {"error": type(e).__name__}
                out["kv_route"].append({"model": model_doc(m), "p": [cfg.tp, cfg.pp, cfg.dp],
                                        "d": [other.tp, other.pp, other.dp], "seq": seq, "result": res})
        out["scalars"].append({"model": model_doc(m), "kv_bytes_per_token": kv_bytes_per_token(m),
                               "total_weight_bytes": total_weight_bytes(m)})
        for seq in (1, 1280):
            try:
                mb = max_batch_size(m, hw, cfg, seq)
            except ConfigError as e:
                mb = type(e).__name__
            out["validate"].append({"model": model_doc(m), "hw": hw_doc(hw), "cfg": [cfg.tp, cfg.pp, cfg.dp],
                                    "seq": seq, "feasible": bool(validate_config(m, hw, cfg)),
                                    "reason": validate_config(m, hw, cfg).reason, "max_batch": mb})
    for layout in (KVLayout.HND, KVLayout.NHD):
        for seq in (1, 2, 1024):
            for h, tp in [(4, 1), (4, 2), (8, 8), (8, 4)]:
                out["contiguous_runs"].append([layout.value, seq, h, tp, contiguous_runs(layout, seq, h, tp)])
    for text in ["tp8.pp1", "tp1.pp8.dp2", "TP2.PP2", "pp4.tp2", "tp8", "tp1.qq2", "tpX.pp1", "tp0.pp1"]:
        try:
            c = ParallelismConfig.parse(text)
            out["parse"].append([text, [c.tp, c.pp, c.dp]])
        except ConfigError:
            out["parse"].append([text, "ConfigError"])
    return out


def sim_golden() -> dict:
    """Reference simulate() runs whose event logs pin replay_check and the
    schedule shape the real engine must reproduce."""
    out = []
    runs = [
        ("tiny", 2, (1, 2), (2, 1), 8, 64, 32, 180e9, 256e9),
        ("tiny", 2, (1, 2), (2, 1), 8, 64, 32, 2e9, 2e9),
        ("llama3-8b", 8, (1, 8), (8, 1), 512, 1024, 256, 180e9, 256e9),
        ("llama3-8b", 1, (1, 1), (1, 1), 64, 1024, 256, 180e9, 256e9),
    ]
    for name, n, p, d, nreq, s_in, s_out, gmem, hmem in runs:
        m = SHAPES[name]
        hw = HardwareSpec(num_gpus=n, hbm_bandwidth=8e12, peak_flops=2.25e15, gpu_memory=gmem,
                          host_memory_per_gpu=hmem, host_link_bandwidth=64e9, allreduce=RingAllReduce(9e11))
        reqs = [Request(i, s_in, s_out) for i in range(nreq)]
        rep = simulate(m, hw, reqs, SchedulingPolicy.TRANSITION_MINIMIZING, ParallelismConfig(*p),
                       ParallelismConfig(*d))
        kinds: dict[str, int] = {}
        for e in rep.event_log:
            kinds[e.kind] = kinds.get(e.kind, 0) + 1
        entry = {"shape": name, "model": model_doc(m), "hw": hw_doc(hw), "p": list(p), "d": list(d), "n": nreq,
                 "in": s_in, "out": s_out, "transitions": rep.transitions, "kinds": kinds,
                 "tokens_per_second": rep.tokens_per_second, "makespan": rep.makespan,
                 "config": rep.config, "replay_ok": bool(replay_check(rep))}
        if nreq <= 8:
            entry["events"] = [json.loads(e.serialize()) for e in rep.event_log]
        out.append(entry)
    return {"runs": out}


def _fleet(model: ModelSpec, gpu_seqs: float, cpu_seqs: float, seq_tokens: int, num_gpus: int = 1,
           dp: int = 1) -> HardwareSpec:
    """The reference tests' sim_fleet (pkg/tests/conftest.py:88-110): each
    replica's GPU tier holds exactly gpu_seqs sequences of seq_tokens, the
    shared CPU tier cpu_seqs."""
    k = seq_tokens * kv_bytes_per_token(model)
    return HardwareSpec(num_gpus=num_gpus, hbm_bandwidth=1e12, peak_flops=1e14,
                        gpu_memory=(total_weight_bytes(model) + gpu_seqs * k) * dp / num_gpus,
                        host_memory_per_gpu=max(cpu_seqs, 1e-9) * k / num_gpus, host_link_bandwidth=1.6e10,
                        allreduce=RingAllReduce(1.6e10))


# BASELINE configs[0]'s tiny LLaMA (2 layers, hidden 256, 4 heads, d=64, ffn
# 768, vocab 1024) as the reference ModelSpec: params_per_layer folded as
# total/L (paper_2503_06433_b200.arch.LlamaArch.model_spec)
TINY = ModelSpec(num_layers=2, params_per_layer=1114752, num_query_heads=4, num_kv_heads=4, head_dim=64)


def _event_rows(rep) -> list:
    """The schedule of a run without its clock: (kind, seq, replica, payload
    fields that describe the schedule)."""
    rows = []
    for e in rep.event_log:
        p = e.payload
        keep = {k: (list(v) if isinstance(v, tuple) else v) for k, v in p.items()
                if k in ("phase", "index", "direction", "seqs", "batch", "tokens")}
        rows.append([e.kind, e.seq_id, e.gpu_id, keep])
    return rows


def schedule_golden() -> dict:
    """Reference simulate() schedules on the tiny LLaMA that the real engine
    reproduces (tests/test_schedule_gpu.py): the [4,4] two-cycle case
    (test_sim.py:79-101), the transition law (test_sim.py:103-117), the
    decode- and prefill-prioritized policies, pipeline decode (ceil(n/pp)
    micro-batches) and DP replicas."""
    out = []
    lens8 = [(24, 8), (24, 3), (24, 5), (24, 2), (24, 7), (24, 4), (24, 6), (24, 1)]
    cases = [
        # name, policy, p, d, n_gpus, dp, gpu_seqs, cpu_seqs, seq_tokens, lens, force_mixed
        ("tm_4_4", "transition-min", (1, 1, 1), (1, 1, 1), 1, 1, 2, 4, 32, [(24, 8)] * 8, False),
        ("tm_pp2_tp2", "transition-min", (1, 2, 1), (2, 1, 1), 2, 1, 2, 4, 32, [(24, 8)] * 8, False),
        ("decode_prio", "decode", (1, 1, 1), (1, 1, 1), 1, 1, 3, 0, 32, lens8, False),
        ("decode_prio_pp2", "decode", (1, 2, 1), (1, 2, 1), 2, 1, 5, 0, 32, lens8, False),
        ("decode_prio_dp2", "decode", (1, 1, 2), (1, 1, 2), 2, 2, 2, 0, 32, lens8, False),
        ("prefill_prio", "prefill", (1, 1, 1), (1, 1, 1), 1, 1, 3, 0, 32, lens8, False),
        ("prefill_prio_mixed", "prefill", (1, 2, 1), (2, 1, 1), 2, 1, 3, 0, 32, lens8, True),
    ]
    for n, cpu, gpu in [(8, 3, 1), (5, 2, 2), (7, 7, 3), (1, 1, 1), (10, 4, 2), (6, 1, 3)]:
        cases.append((f"law_{n}_{cpu}_{gpu}", "transition-min", (1, 1, 1), (1, 1, 1), 1, 1, gpu, cpu, 19,
                      [(16, 3)] * n, False))
    for name, pol, p, d, ng, dp, gs, cs, toks, lens, mixed in cases:
        hw = _fleet(TINY, gs, cs, toks, num_gpus=ng, dp=dp)
        reqs = [Request(i, a, b) for i, (a, b) in enumerate(lens)]
        rep = simulate(TINY, hw, reqs, SchedulingPolicy(pol), ParallelismConfig(*p), ParallelismConfig(*d),
                       SimOptions(force_mixed=mixed))
        out.append({"name": name, "policy": pol, "p": list(p), "d": list(d), "num_gpus": ng,
                    "gpu_memory": hw.gpu_memory, "host_memory_per_gpu": hw.host_memory_per_gpu,
                    "host_link_bandwidth": hw.host_link_bandwidth, "lens": [list(x) for x in lens],
                    "force_mixed": mixed, "transitions": rep.transitions, "replay_ok": bool(replay_check(rep)),
                    "events": _event_rows(rep)})
    return {"model": model_doc(TINY), "runs": out}


def perf_golden() -> dict:
    """Reference cost-model values (perf.py) the restated model must equal."""
    from shardsim import perf
    from shardsim.perf import Mode, Phase

    out = []
    rnd = random.Random(11)
    for (m, cfg) in random_cases(60, 3) + [(SHAPES["llama3-8b"], ParallelismConfig(8, 1, 1)),
                                          (SHAPES["llama3-8b"], ParallelismConfig(1, 8, 1))]:
        hw = b200_fleet(cfg.num_gpus)
        for phase in (Phase.PREFILL, Phase.DECODE):
            for mode in (Mode.ROOFLINE, Mode.ADDITIVE):
                b, s = rnd.choice([1, 3, 16]), rnd.choice([1, 17, 1024])
                lens = [rnd.randint(1, 600) for _ in range(rnd.randint(1, 5))]
                out.append({
                    "model": model_doc(m), "hw": hw_doc(hw), "cfg": [cfg.tp, cfg.pp, cfg.dp], "phase": phase.value,
                    "mode": mode.value, "b": b, "s": s, "lens": lens,
                    "layer": perf.layer_time(m, hw, cfg, b, s, phase, mode).as_dict(),
                    "batch": perf.layer_time_batch(m, hw, cfg, lens, phase, mode).as_dict(),
                    "stage": perf.stage_time(m, hw, cfg, b * 4, s, phase, mode),
                    "tinv": perf.throughput_inverse(m, hw, cfg, b * 4, s, phase, mode),
                })
    return {"cases": out}


def main() -> None:
    (OUT / "perf.json").write_text(json.dumps(perf_golden(), sort_keys=True))
    (OUT / "planning.json").write_text(json.dumps(planning_golden(), sort_keys=True))
    (OUT / "simulate.json").write_text(json.dumps(sim_golden(), sort_keys=True))
    (OUT / "schedule.json").write_text(json.dumps(schedule_golden(), sort_keys=True))
    print("wrote", OUT / "planning.json", OUT / "simulate.json", "with shardsim", shardsim.__version__)


if __name__ == "__main__":
    main()
