"""bench.py's output contract, at N=1 and as 2 torchrun ranks (gloo: both
ranks share the test box's single GPU; the driver's N>1 runs use NCCL), on
the tiny config so it finishes in seconds."""

from __future__ import annotations

import json
import os
import socket
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent
ARGS = ["--arch", "tiny", "--prompts", "8", "--input-len", "64", "--output-len", "8", "--steps", "1", "--warmup", "3",
        "--no-cpu-baseline", "--prefill-tokens", "512"]
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
        "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "roofline", "clocks"}


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _last_json(out: str) -> dict:
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert lines, out[-2000:]
    return json.loads(lines[-1])


def test_bench_single_gpu_contract(cuda):
    p = subprocess.run([sys.executable, "bench.py", *ARGS], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    line = _last_json(p.stdout)
    assert KEYS <= set(line)
    assert line["n_gpus"] == 1 and line["value"] > 0 and line["gpu_launches"] > 0
    assert set(line["e2e"]) >= {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"}
    assert set(line["roofline"]) >= {"bound", "achieved", "peak", "unit", "frac", "traffic"}
    assert line["replay_check"] is True
    assert "sweep" in line["reshard_micro"]


def test_bench_two_ranks_contract(cuda):
    env = dict(os.environ, SSB_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2", *ARGS]
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    assert p.returncode == 0, p.stderr[-3000:]
    line = _last_json(p.stdout)
    assert KEYS <= set(line)
    assert line["n_gpus"] == 2 and line["config"]["parallelism"] == "pp2->tp2"
    assert line["replay_check"] is True
    # the PP2 -> TP2 transition moved weights and KV between the two ranks
    assert line["reshard"]["bytes_sent_per_gpu"] > 0


def test_bench_eight_ranks_contract(cuda, tmp_path):
    """bench.py --gpus 8 as 8 torchrun processes (gloo; all on the test box's
    one GPU) on an 8-layer head_dim-128 GQA model: the PP8 -> TP8 layout the
    driver's 8-GPU run takes, through the same process-level code path
    (TorchComm groups, PP send/recv, all-to-all re-shard, TP all-reduce /
    all-gather).  The line must follow the contract and rank 0's re-shard
    bytes must equal the placement-rule volume (SURVEY A.3's rules)."""
    import yaml

    from engine_helpers import expected_kv_bytes_per_token_sent, expected_weight_bytes_sent
    from paper_2503_06433_b200 import LlamaArch

    arch = LlamaArch("l8-d128", 8, 512, 16, 8, 128, 1024, 2048, rope_theta=500000.0)
    path = tmp_path / "l8.yaml"
    path.write_text(yaml.safe_dump(arch.as_dict()))
    prompts, s_in, s_out = 8, 64, 8
    args = ["--arch", str(path), "--prompts", str(prompts), "--input-len", str(s_in), "--output-len", str(s_out),
            "--steps", "1", "--warmup", "3", "--no-cpu-baseline", "--prefill-tokens", "512"]
    env = dict(os.environ, SSB_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "8", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "8", *args]
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=1500, env=env)
    assert p.returncode == 0, p.stderr[-3000:]
    line = _last_json(p.stdout)
    assert KEYS <= set(line)
    assert line["n_gpus"] == 8 and line["config"]["parallelism"] == "pp8->tp8"
    assert line["replay_check"] is True and line["value"] > 0
    blocks = prompts * -(-(s_in + s_out) // 64)
    kv = expected_kv_bytes_per_token_sent(arch, (1, 8), (8, 1), 0) * 64 * blocks
    w = expected_weight_bytes_sent(arch, (1, 8), (8, 1), 0)
    assert line["reshard"]["bytes_sent_per_gpu"] == kv + w
