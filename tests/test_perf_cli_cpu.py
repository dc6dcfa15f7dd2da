"""Restated cost model == reference perf.py (golden), and the CLI's
plan/predict/error paths (cli.py conventions: JSON errors, exit 1)."""

from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

import pytest

from paper_2503_06433_b200 import ModelSpec, ParallelismConfig
from paper_2503_06433_b200 import perf
from paper_2503_06433_b200.cli import TraceError, main, parse_trace
from paper_2503_06433_b200.report import Mode
from paper_2503_06433_b200.specs import hardware_spec_from_mapping

ROOT = Path(__file__).resolve().parent.parent
GOLD = json.loads((ROOT / "tests" / "golden" / "perf.json").read_text())


def test_cost_model_matches_reference():
    assert len(GOLD["cases"]) > 100
    for c in GOLD["cases"]:
        m = ModelSpec(**c["model"])
        hw = hardware_spec_from_mapping(c["hw"])
        cfg = ParallelismConfig(*c["cfg"])
        ph, mode = perf.Phase(c["phase"]), Mode(c["mode"])
        assert perf.layer_time(m, hw, cfg, c["b"], c["s"], ph, mode).as_dict() == pytest.approx(c["layer"], rel=1e-12)
        assert perf.layer_time_batch(m, hw, cfg, c["lens"], ph, mode).as_dict() == pytest.approx(c["batch"], rel=1e-12)
        assert perf.stage_time(m, hw, cfg, c["b"] * 4, c["s"], ph, mode) == pytest.approx(c["stage"], rel=1e-12)
        assert perf.throughput_inverse(m, hw, cfg, c["b"] * 4, c["s"], ph, mode) == pytest.approx(c["tinv"], rel=1e-12)


def test_cli_plan_and_predict(capsys):
    args = ["--model", str(ROOT / "configs/model_llama3_8b.yaml"), "--hw", str(ROOT / "configs/b200_x8.yaml")]
    assert main(["plan", *args, "--cfg", "tp1.pp8", "--new-cfg", "tp8.pp1", "--tokens", "1"]) == 0
    out = capsys.readouterr().out
    doc = json.loads(out[out.index("{"):])
    mat = doc["nvlink_kv_exchange_bytes"]
    assert len(mat) == 8 and all(v == 2048 for row in mat for v in row)  # 16 KiB/token split 8 ways
    assert main(["predict", *args, "--prefill-cfg", "tp1.pp8", "--decode-cfg", "tp8.pp1", "--prompts", "512",
                 "--input-len", "1024", "--output-len", "256"]) == 0
    pred = json.loads(capsys.readouterr().out)
    assert pred["prefill_s"] > 0 and pred["decode_s"] > 0


def test_cli_errors_are_json(tmp_path):
    bad = tmp_path / "t.jsonl"
    bad.write_text('{"input_len": 4}\n')
    with pytest.raises(TraceError):
        parse_trace(bad)
    proc = subprocess.run([sys.executable, "-m", "paper_2503_06433_b200", "plan", "--model",
                           str(ROOT / "configs/model_llama3_8b.yaml"), "--hw", str(ROOT / "configs/b200_x8.yaml"),
                           "--cfg", "tp3.pp1"], capture_output=True, text=True, cwd=ROOT)
    assert proc.returncode == 1
    err = json.loads(proc.stderr.strip().splitlines()[-1])
    assert err["error_kind"] == "ConfigError" and "tp=3" in err["message"]


def test_trace_with_prompts(tmp_path):
    t = tmp_path / "t.jsonl"
    t.write_text('{"id": "a", "input_len": 3, "output_len": 2, "prompt": [1, 2, 3]}\n'
                 '{"input_len": 2, "output_len": 1, "prompt": [5, 6]}\n')
    reqs, prompts = parse_trace(t)
    assert [r.id for r in reqs] == ["a", 1] and prompts == [[1, 2, 3], [5, 6]]


def test_calibration_physical_spec_and_model_error(tmp_path):
    """tools/calibrate.py writes a PHYSICAL HardwareSpec (the measured peaks,
    nothing fitted) that the reference-schema loader accepts, attributes the
    reference model's prefill error to its d^2 attention term (x64 at
    head_dim 128; with the conventional causal count the model is within
    10 % of the measured prefill), and turns a multi-GPU line's measured
    all-reduce bandwidths into an AllReduceTable ("map") spec."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    from paper_2503_06433_b200.specs import AllReduceTable, load_hardware_spec

    root = Path(__file__).resolve().parent.parent
    line = root / "profiles" / "r02" / "bench_n1_first.log"
    peaks = tmp_path / "peaks.json"
    peaks.write_text(json.dumps({"hbm_gbs": 6551.4, "bf16_tflops_sustained": 1388.1, "when": "test"}))
    scale = tmp_path / "scale.json"
    scale.write_text(json.dumps({"allreduce_table": {"allreduce_table": {"2": 3.1e11, "4": 2.6e11, "8": 2.2e11}}}))
    out = tmp_path / "hw.yaml"
    p = subprocess.run([sys.executable, str(root / "tools" / "calibrate.py"), str(line), str(scale), "--peaks",
                        str(peaks), "--yaml", str(out)], capture_output=True, text=True, timeout=120)
    assert p.returncode == 0, p.stderr
    res = json.loads(p.stdout)
    assert res["prefill_compute_terms"]["d2_over_conventional"] == 64.0
    assert abs(res["reference_model_conventional_attention"]["prefill_error"]) < 0.10
    assert abs(res["reference_model"]["decode_error"]) < 0.10
    assert res["reference_model"]["prefill_error"] > 0.5  # the d^2 term, attributed rather than fitted away
    hw = load_hardware_spec(out)
    assert hw.peak_flops == 1.3881e15 and hw.hbm_bandwidth == 6.5514e12
    assert isinstance(hw.allreduce, AllReduceTable) and hw.allreduce.bandwidth(8) == 2.2e11


def test_memory_plan_fits_every_baseline_layout():
    """Per-GPU HBM plan (tools/memory_plan.py): on every BASELINE layout the
    worst GPU's weights + runtime reserve (re-partition transient, prefill
    activations, workspaces, slack) leave a KV pool for hundreds of resident
    1024+256-token sequences; 70B PP8->TP8 included (its pool is what the
    engine sizes, no hand cap)."""
    import sys
    from pathlib import Path

    sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tools"))
    import memory_plan

    for case in memory_plan.CASES:
        r = memory_plan.plan(*case)
        assert r["kv_pool_gb"] > 100 and r["resident_seqs_per_replica"] >= 500, r
        assert abs(r["peak_gb"] - 180) < 1.0
        rs = r["reserve_gb"]
        assert rs["total"] < 30 and rs["weight_transient"] >= 0
