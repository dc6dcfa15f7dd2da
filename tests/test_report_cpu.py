"""report.py (Event / SimReport / replay_check) against the reference's own
event logs (tests/golden/simulate.json, produced by shardsim.simulate): the
restated checker accepts them and rejects the same tampering the reference's
tests inject (test_sim.py:194-221)."""

from __future__ import annotations

import dataclasses
import json
from pathlib import Path

from paper_2503_06433_b200.report import Event, SimReport, TieredKVState, replay_check

GOLD = json.loads((Path(__file__).parent / "golden" / "simulate.json").read_text())


def _report(run) -> SimReport:
    evs = []
    for e in run["events"]:
        extra = tuple((k, tuple(v) if isinstance(v, list) else v) for k, v in e["extra"])
        evs.append(Event(t=float(e["t"]), kind=e["kind"], seq_id=e["seq_id"], gpu_id=e["gpu_id"], bytes=e["bytes"],
                         extra=extra))
    return SimReport(makespan=run["makespan"], requests_per_second=0.0, tokens_per_second=run["tokens_per_second"],
                     prefill_time=0.0, decode_time=0.0, reshard_time=0.0, stalled_transfer_time=0.0,
                     transitions=run["transitions"], event_log=tuple(evs), config=run["config"],
                     final_kv_state=TieredKVState(0, 0))


def test_reference_logs_pass():
    runs = [r for r in GOLD["runs"] if "events" in r]
    assert runs
    for run in runs:
        assert run["replay_ok"]
        rep = _report(run)
        assert replay_check(rep), replay_check(rep).violation
        # serialisation is byte-identical to the reference's Event.serialize
        for ev, raw in zip(rep.event_log, run["events"]):
            assert json.loads(ev.serialize()) == raw


def test_tampered_logs_rejected():
    run = next(r for r in GOLD["runs"] if "events" in r)
    rep = _report(run)
    log = list(rep.event_log)
    idx = next(i for i, e in enumerate(log) if e.kind == "swap_out_complete")
    rogue = Event(t=log[idx].t, kind="decode_step", gpu_id=0, extra=(("seqs", (log[idx].seq_id,)),))
    bad = dataclasses.replace(rep, event_log=tuple(log[: idx + 1] + [rogue] + log[idx + 1 :]))
    v = replay_check(bad)
    assert not v and "decode before residency" in v.violation
    k = int(rep.config["cpu_kv_capacity_bytes"]) + 1
    log2 = list(log)
    log2.insert(idx, Event(t=log[idx].t, kind="prefill_complete", seq_id="ghost", gpu_id=0, bytes=k,
                           extra=(("input_len", 1), ("output_len", 1))))
    log2.insert(idx + 1, Event(t=log[idx].t, kind="swap_out_complete", seq_id="ghost", gpu_id=0, bytes=k))
    v = replay_check(dataclasses.replace(rep, event_log=tuple(log2)))
    assert not v and "tier overflow" in v.violation
    # dropping a release leaks bytes / leaves a sequence unreleased
    log3 = [e for i, e in enumerate(log) if not (e.kind == "kv_release" and e.seq_id == 0)]
    assert not replay_check(dataclasses.replace(rep, event_log=tuple(log3)))
