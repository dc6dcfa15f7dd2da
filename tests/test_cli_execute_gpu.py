"""``python -m paper_2503_06433_b200 execute`` end to end (SURVEY §8(f) row
4, mirroring the reference's ``shardsim simulate`` CLI, cli.py:133-160):
reference-schema ModelSpec / HardwareSpec documents, a JSONL trace, the
SimReport document on stdout, the events CSV and the generated token ids —
on one GPU, as two torchrun processes (gloo, PP2 -> TP2 on the test box's
single GPU), and the JSON error path."""

from __future__ import annotations

import csv
import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import yaml

from engine_helpers import check_greedy
from paper_2503_06433_b200 import PRESETS
from paper_2503_06433_b200.specs import Request

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent
LENS = [(40, 6), (17, 3), (64, 5), (5, 4)]


def _files(tmp: Path, prompts: bool) -> dict:
    arch = PRESETS["tiny"]
    m = arch.model_spec()
    (tmp / "model.yaml").write_text(yaml.safe_dump({
        "num_layers": m.num_layers, "params_per_layer": m.params_per_layer, "num_query_heads": m.num_query_heads,
        "num_kv_heads": m.num_kv_heads, "head_dim": m.head_dim}))
    (tmp / "hw.yaml").write_text(yaml.safe_dump({
        "num_gpus": 1, "hbm_bandwidth": 8e12, "peak_flops": 2.25e15, "gpu_memory": 2e9,
        "host_memory_per_gpu": 2e9, "host_link_bandwidth": 64e9,
        "allreduce_model": {"kind": "ring", "interconnect_bandwidth": 9e11}}))
    (tmp / "hw2.yaml").write_text((tmp / "hw.yaml").read_text().replace("num_gpus: 1", "num_gpus: 2"))
    rng = np.random.default_rng(5)
    with open(tmp / "trace.jsonl", "w") as fh:
        for i, (a, b) in enumerate(LENS):
            rec = {"id": f"r{i}", "input_len": a, "output_len": b}
            if prompts:
                rec["prompt"] = rng.integers(0, arch.vocab, size=a).tolist()
            fh.write(json.dumps(rec) + "\n")
    return {"model": tmp / "model.yaml", "hw": tmp / "hw.yaml", "hw2": tmp / "hw2.yaml", "trace": tmp / "trace.jsonl"}


def _prompts(trace: Path):
    return [np.asarray(json.loads(l)["prompt"], dtype=np.int32) for l in trace.read_text().splitlines()]


def test_execute_single_gpu(cuda, tmp_path):
    f = _files(tmp_path, prompts=True)
    out, ev = tmp_path / "out.json", tmp_path / "events.csv"
    cmd = [sys.executable, "-m", "paper_2503_06433_b200", "execute", "--model", str(f["model"]), "--hw", str(f["hw"]),
           "--arch", "tiny", "--trace", str(f["trace"]), "--prefill-cfg", "tp1.pp1.dp1", "--decode-cfg",
           "tp1.pp1.dp1", "--outputs", str(out), "--events-csv", str(ev)]
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    doc = json.loads(p.stdout)
    assert doc["transitions"] == 1 and doc["tokens_per_second"] > 0
    outputs = json.loads(out.read_text())
    assert set(outputs) == {f"r{i}" for i in range(len(LENS))}
    rows = list(csv.reader(open(ev)))
    # one CSV row per sequence of each event (the reference's events CSV)
    assert rows[0] == ["timestamp_s", "event", "seq_id", "gpu_id", "bytes"]
    assert sum(r[1] == "decode_step" for r in rows[1:]) == sum(b for _, b in LENS)
    reqs = [Request(f"r{i}", a, b) for i, (a, b) in enumerate(LENS)]
    check_greedy(PRESETS["tiny"], reqs, _prompts(f["trace"]), outputs, 1, 1)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_execute_two_ranks_pp2_to_tp2(cuda, tmp_path):
    f = _files(tmp_path, prompts=True)
    out = tmp_path / "out.json"
    env = dict(os.environ, SSB_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), "-m", "paper_2503_06433_b200", "execute",
           "--model", str(f["model"]), "--hw", str(f["hw2"]), "--arch", "tiny", "--trace", str(f["trace"]),
           "--prefill-cfg", "tp1.pp2.dp1", "--decode-cfg", "tp2.pp1.dp1", "--outputs", str(out),
           "--tm-mode", "reference"]
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert p.returncode == 0, p.stderr[-3000:]
    doc = json.loads(p.stdout)  # rank 0 prints the report document
    assert doc["transitions"] >= 1
    outputs = json.loads(out.read_text())
    reqs = [Request(f"r{i}", a, b) for i, (a, b) in enumerate(LENS)]
    check_greedy(PRESETS["tiny"], reqs, _prompts(f["trace"]), outputs, 1, 2, pp_prefill=2)


def test_execute_error_is_json(cuda, tmp_path):
    f = _files(tmp_path, prompts=False)
    cmd = [sys.executable, "-m", "paper_2503_06433_b200", "execute", "--model", str(f["model"]), "--hw", str(f["hw"]),
           "--arch", "tiny", "--trace", str(f["trace"]), "--prefill-cfg", "tp1.pp3.dp1", "--decode-cfg",
           "tp1.pp1.dp1"]
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert p.returncode == 1
    err = json.loads(p.stderr.strip().splitlines()[-1])
    assert err["error_kind"] == "ConfigError"
