"""Summarise the ncu captures of tools/profile.sh into profiles/<round>/.

    python tools/summarise_profiles.py gpurun_out/prof profiles/r01

* launches.csv.gz (one timed batch, every kernel, gpu__time_duration) ->
  launch_shares.json: per-kernel launch count, summed time, share, median.
* <name>.ncu-rep (--set full) -> ncu_full_<name>.json: the counters the
  roofline needs per launch (duration, DRAM bytes, tensor-pipe and DRAM
  utilisation, occupancy, registers, smem, clocks) and the grid.
"""

from __future__ import annotations

import csv
import gzip
import io
import json
import statistics
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

KEEP = [
    "Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
    "dram__bytes_write.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
    "l1tex__m_xbar2l1tex_read_bytes.sum", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.avg.per_second", "dram__cycles_elapsed.avg.per_second",
]


def _to_seconds(v: float, unit: str) -> float:
    return v * {"nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}.get(unit, 1e-9)


def launches(path: Path) -> dict:
    text = gzip.open(path, "rt").read() if path.suffix == ".gz" else path.read_text()
    lines = text.splitlines()
    start = next(i for i, ln in enumerate(lines) if ln.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    agg: dict = defaultdict(list)
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"].split("(")[0].replace("void ", "")
        agg[name].append(_to_seconds(float(r["Metric Value"].replace(",", "")), r["Metric Unit"]))
    total = sum(sum(v) for v in agg.values())
    out = {"launches": sum(len(v) for v in agg.values()), "total_s": total, "kernels": {}}
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out["kernels"][k] = {"launches": len(v), "s": sum(v), "share": sum(v) / total,
                             "median_us": statistics.median(v) * 1e6}
    return out


def full(rep: Path) -> list[dict]:
    proc = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True,
                          check=True)
    rows = list(csv.reader(io.StringIO(proc.stdout)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    out = []
    for r in data:
        d = {}
        for key in KEEP:
            if key in hdr:
                i = hdr.index(key)
                d[key] = f"{r[i]} {units[i]}".strip()
        out.append(d)
    return out


def main() -> None:
    src, dst = Path(sys.argv[1]), Path(sys.argv[2])
    dst.mkdir(parents=True, exist_ok=True)
    for p in [src / "launches.csv.gz", src / "launches.csv"]:
        if p.exists():
            (dst / "launch_shares.json").write_text(json.dumps(launches(p), indent=1))
            if p.suffix == ".gz":
                (dst / "launches.csv.gz").write_bytes(p.read_bytes())
            break
    for rep in sorted(src.glob("*.ncu-rep")):
        (dst / f"ncu_full_{rep.stem}.json").write_text(json.dumps(full(rep), indent=1))
    print(sorted(x.name for x in dst.iterdir()))


if __name__ == "__main__":
    main()
