"""Per-GPU HBM plan of the BASELINE configurations on 8 x B200 (180 GB each;
VERDICT r1 "Next round" 8): weights under the prefill and the decode layout
(the largest GPU of the replica), the runtime reserve the engine subtracts
before sizing the KV pool (runtime.runtime_reserve: re-partition transient,
prefill activations, workspaces, slack), and the KV pool that is left, in
64-token blocks and in resident 1024+256-token sequences per replica.

Pure arithmetic on the layouts the engine allocates (layout.weight_layout,
layout.kv_geometry); no GPU.

    python tools/memory_plan.py [--json profiles/r02/memory_plan.json]
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2503_06433_b200 import PRESETS, ParallelismConfig  # noqa: E402
from paper_2503_06433_b200.layout import kv_geometry, weight_layout  # noqa: E402
from paper_2503_06433_b200.runtime import runtime_reserve  # noqa: E402

HBM = 180e9
CASES = [
    ("llama3-8b", ParallelismConfig(1, 1, 1), ParallelismConfig(1, 1, 1), "configs[1] at N=1"),
    ("llama3-8b", ParallelismConfig(1, 8, 1), ParallelismConfig(8, 1, 1), "configs[1]: PP8 -> TP8"),
    ("llama2-13b", ParallelismConfig(1, 4, 1), ParallelismConfig(4, 1, 1), "configs[2]: PP4 -> TP4 (4 GPUs)"),
    ("llama2-13b", ParallelismConfig(1, 4, 2), ParallelismConfig(4, 1, 2), "configs[2]: PP4 -> TP4 x DP2"),
    ("llama3-70b", ParallelismConfig(1, 8, 1), ParallelismConfig(8, 1, 1), "configs[3]: PP8 -> TP8 (+ host tier)"),
]


def plan(arch_name: str, cfg_p: ParallelismConfig, cfg_d: ParallelismConfig, note: str,
         max_prefill_tokens: int = 16384, block_size: int = 64, seq_tokens: int = 1280) -> dict:
    arch = PRESETS[arch_name]
    gpus = cfg_p.gpus_per_replica
    rows = []
    for g in range(gpus):
        w_p = weight_layout(arch, cfg_p.tp, cfg_p.pp, g).arena_elems * 2
        w_d = weight_layout(arch, cfg_d.tp, cfg_d.pp, g).arena_elems * 2
        res = runtime_reserve(arch, g, cfg_p, cfg_d, max_prefill_tokens, block_size)
        rows.append((max(w_p, w_d), w_p, w_d, res))
    worst = max(rows, key=lambda r: r[0] + r[3]["total"])
    weights, w_p, w_d, res = worst
    block = kv_geometry(arch, cfg_p.tp, cfg_p.pp, 1, block_size).block_elems * 2
    pool = HBM - weights - res["total"]
    blocks = int(pool // block)
    per_seq = -(-seq_tokens // block_size)
    return {
        "model": arch_name, "layout": f"{cfg_p.label()} -> {cfg_d.label()}", "note": note,
        "gpus_per_replica": gpus, "replicas": cfg_p.dp,
        "weights_gb": {"prefill_layout": w_p / 1e9, "decode_layout": w_d / 1e9},
        "reserve_gb": {k: v / 1e9 for k, v in res.items()},
        "kv_block_bytes_per_gpu": block,
        "kv_pool_gb": pool / 1e9, "kv_blocks_per_gpu": blocks,
        "resident_seqs_per_replica": blocks // per_seq,
        "peak_gb": (weights + res["total"] + blocks * block) / 1e9,
    }


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--json", type=Path)
    args = ap.parse_args()
    out = [plan(*c) for c in CASES]
    hdr = f"{'model':11} {'layout':28} {'W_p':>6} {'W_d':>6} {'transient':>9} {'act':>5} {'ws':>5} " \
          f"{'KV pool':>8} {'blocks':>7} {'seqs':>6} {'peak':>6}  (GB per GPU, worst GPU)"
    print(hdr)
    for r in out:
        rs = r["reserve_gb"]
        print(f"{r['model']:11} {r['layout']:28} {r['weights_gb']['prefill_layout']:6.1f} "
              f"{r['weights_gb']['decode_layout']:6.1f} {rs['weight_transient']:9.1f} {rs['activations']:5.1f} "
              f"{rs['workspaces']:5.1f} {r['kv_pool_gb']:8.1f} {r['kv_blocks_per_gpu']:7d} "
              f"{r['resident_seqs_per_replica']:6d} {r['peak_gb']:6.1f}")
    if args.json:
        args.json.write_text(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
