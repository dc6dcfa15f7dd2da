"""Command line front end: ``python -m paper_2503_06433_b200 <command>``.

Mirrors the reference CLI (/root/reference/pkg/src/shardsim/cli.py:50-106,
:133-160, :213-245) for the re-sharding path:

  execute  the real-hardware counterpart of ``shardsim simulate``: same flags
           (--model/--hw/--trace/--policy/--prefill-cfg/--decode-cfg/
           --events-csv, ...) plus --arch; one process per GPU under torchrun
           (NCCL) or a single GPU; prints the SimReport document and checks
           the event log with replay_check.
  plan     shard maps, the reference weight reload plan, and the per-peer
           NVLink exchange bytes of a layout switch.
  predict  the reference cost model's prediction for a constant-length batch.

Errors print {"error_kind", "message"} JSON on stderr and exit 1 (cli.py:236-245).
Traces are the reference's JSONL (input_len, output_len, optional id), with an
optional "prompt" list of token ids per record (synthetic ids otherwise).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
from pathlib import Path

from .report import Mode, SchedulingPolicy, SimOptions, replay_check
from .specs import ConfigError, KVLayout, ParallelismConfig, Request, load_hardware_spec, load_model_spec

_POLICIES = {p.value: p for p in SchedulingPolicy}


class TraceError(ValueError):
    """A trace file is malformed (workload.py:19-20)."""


def parse_trace(path: str | Path) -> tuple[list[Request], list | None]:
    """JSONL records in file order; missing ids become the record index
    (workload.py:53-85); an optional "prompt" field carries token ids."""
    try:
        lines = Path(path).read_text(encoding="utf-8").splitlines()
    except OSError as exc:
        raise TraceError(f"cannot open trace {path}: {exc}") from exc
    reqs, prompts = [], []
    for i, line in enumerate(lines):
        if not line.strip():
            continue
        try:
            rec = json.loads(line)
        except json.JSONDecodeError as exc:
            raise TraceError(f"{path}:{i + 1}: invalid JSON ({exc})") from exc
        if not isinstance(rec, dict) or "input_len" not in rec or "output_len" not in rec:
            raise TraceError(f"{path}:{i + 1}: record needs input_len and output_len")
        try:
            reqs.append(Request(rec.get("id", len(reqs)), rec["input_len"], rec["output_len"]))
        except ConfigError as exc:
            raise TraceError(f"{path}:{i + 1}: {exc}") from exc
        prompts.append(rec.get("prompt"))
    if not reqs:
        raise TraceError(f"{path}: empty trace")
    if all(p is None for p in prompts):
        return reqs, None
    if any(p is None for p in prompts):
        raise TraceError(f"{path}: either every record or none carries a prompt")
    return reqs, prompts


def build_parser() -> argparse.ArgumentParser:
    parser = argparse.ArgumentParser(prog="paper_2503_06433_b200")
    sub = parser.add_subparsers(dest="command", required=True)

    p = sub.add_parser("execute", help="run a trace for real: PP prefill -> NVLink re-shard -> TP decode")
    p.add_argument("--model", required=True, help="ModelSpec document (YAML/JSON)")
    p.add_argument("--hw", required=True, help="HardwareSpec document (YAML/JSON)")
    p.add_argument("--arch", required=True, help="LlamaArch preset name or YAML document")
    p.add_argument("--trace", required=True)
    p.add_argument("--policy", choices=sorted(_POLICIES), default="transition-min")
    p.add_argument("--prefill-cfg", required=True, help="e.g. tp1.pp8.dp1")
    p.add_argument("--decode-cfg", required=True, help="e.g. tp8.pp1.dp1")
    p.add_argument("--no-overlap", action="store_true")
    p.add_argument("--nhd", action="store_true")
    p.add_argument("--p2p", action="store_true")
    p.add_argument("--mode", choices=["roofline", "additive"], default="roofline")
    p.add_argument("--force-mixed", action="store_true")
    p.add_argument("--seed", type=int, default=0)
    p.add_argument("--events-csv", help="write the event log to this CSV file")
    p.add_argument("--outputs", help="write generated token ids (JSON) to this file")
    p.add_argument("--tm-mode", choices=["native", "reference"], default="native",
                   help="transition-minimizing: keep fitting KV in HBM (native) or route every wave "
                        "through the host tier (the reference's schedule)")

    p = sub.add_parser("plan", help="shard maps, reload plan and NVLink exchange of a layout switch")
    p.add_argument("--model", required=True)
    p.add_argument("--hw", required=True)
    p.add_argument("--cfg", required=True)
    p.add_argument("--new-cfg")
    p.add_argument("--tokens", type=int, default=1, help="KV tokens for the exchange byte matrix")

    p = sub.add_parser("predict", help="reference cost-model prediction of a constant-length batch")
    p.add_argument("--model", required=True)
    p.add_argument("--hw", required=True)
    p.add_argument("--prefill-cfg", required=True)
    p.add_argument("--decode-cfg", required=True)
    p.add_argument("--prompts", type=int, required=True)
    p.add_argument("--input-len", type=int, required=True)
    p.add_argument("--output-len", type=int, required=True)
    return parser


def _load_arch(text: str):
    from .arch import PRESETS, load_arch

    return PRESETS[text] if text in PRESETS else load_arch(text)


def _cmd_execute(args) -> int:
    import torch

    from .comm import SoloComm, TorchComm
    from .engine import execute

    model = load_model_spec(args.model)
    hw = load_hardware_spec(args.hw)
    arch = _load_arch(args.arch)
    reqs, prompts = parse_trace(args.trace)
    options = SimOptions(overlap=not args.no_overlap, mode=Mode(args.mode), charge_p2p=args.p2p,
                         kv_layout=KVLayout.NHD if args.nhd else KVLayout.HND, force_mixed=args.force_mixed,
                         seed=args.seed)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local % max(torch.cuda.device_count(), 1))
    if world > 1:
        import torch.distributed as dist

        # SSB_DIST_BACKEND=gloo: ranks sharing one GPU (multi-rank test runs)
        if os.environ.get("SSB_DIST_BACKEND", "nccl") == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
        comm = TorchComm()
    else:
        comm = SoloComm()
    rep = execute(model, hw, reqs, _POLICIES[args.policy], ParallelismConfig.parse(args.prefill_cfg),
                  ParallelismConfig.parse(args.decode_cfg), options, arch=arch, seed=args.seed, prompts=prompts,
                  comm=comm, tm_mode=args.tm_mode)
    verdict = replay_check(rep)
    if not verdict:
        raise RuntimeError(f"replay check failed: {verdict.violation}")
    if comm.rank == 0:
        if args.events_csv:
            rep.write_events_csv(args.events_csv)
        if args.outputs:
            Path(args.outputs).write_text(json.dumps({str(k): v for k, v in rep.outputs.items()}))
        print(rep.to_document())
    return 0


def _cmd_plan(args) -> int:
    from .reshard import kv_exchange_matrix, shard_map, weight_reload_plan

    model = load_model_spec(args.model)
    hw = load_hardware_spec(args.hw)
    cfg = ParallelismConfig.parse(args.cfg)
    print(shard_map(model, cfg).table())
    if args.new_cfg:
        new = ParallelismConfig.parse(args.new_cfg)
        plan = weight_reload_plan(model, hw, cfg, new)
        doc = {"reference_reload": {"bytes_per_gpu": list(plan.bytes_per_gpu), "wall_time_s": plan.wall_time},
               "nvlink_kv_exchange_bytes": kv_exchange_matrix(model, cfg, new, args.tokens)}
        print(json.dumps(doc, indent=2))
    return 0


def _cmd_predict(args) -> int:
    from .perf import predict_phases

    model = load_model_spec(args.model)
    hw = load_hardware_spec(args.hw)
    doc = predict_phases(model, hw, ParallelismConfig.parse(args.prefill_cfg),
                         ParallelismConfig.parse(args.decode_cfg), args.input_len, args.output_len, args.prompts)
    doc["output_tokens_per_s"] = args.prompts * args.output_len / (doc["prefill_s"] + doc["decode_s"])
    print(json.dumps(doc, indent=2, sort_keys=True))
    return 0


_COMMANDS = {"execute": _cmd_execute, "plan": _cmd_plan, "predict": _cmd_predict}


def main(argv: list[str] | None = None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return _COMMANDS[args.command](args)
    except (ConfigError, TraceError, ValueError, OSError, RuntimeError) as exc:
        print(json.dumps({"error_kind": type(exc).__name__, "message": str(exc)}), file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
