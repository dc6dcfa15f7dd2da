"""Engine result types and the event-log replay checker.

Same names, fields, serialisation and checks as the reference simulator so a
real B200 run is a drop-in for ``simulate()``'s report and passes the
reference's own ``replay_check`` unchanged — /root/reference/pkg/src/shardsim/sim.py:
  SimulationError  :40-41     SchedulingPolicy :44-47    Residency :50-54
  TieredKVState    :57-72     SimOptions       :75-96    Event     :99-125
  SimReport        :128-176   ReplayVerdict    :183-190  replay_check :764-837
Event.gpu_id holds the data-parallel REPLICA index, as in the reference.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field
from enum import Enum

from .specs import KVLayout


class SimulationError(ValueError):
    """The requested run is impossible (empty workload, unbufferable request, ...)."""


class SchedulingPolicy(Enum):
    PREFILL_PRIORITIZED = "prefill"
    DECODE_PRIORITIZED = "decode"
    TRANSITION_MINIMIZING = "transition-min"


class Mode(Enum):
    """Composition rule of the reference cost model (perf.py:28-32); carried in
    SimOptions for API compatibility — real runs measure instead."""

    ROOFLINE = "roofline"
    ADDITIVE = "additive"


class Residency(Enum):
    GPU = "gpu"
    CPU = "cpu"
    IN_TRANSIT = "in_transit"
    RELEASED = "released"


@dataclass
class TieredKVState:
    """Byte ledger of the GPU and host KV tiers plus per-sequence residency."""

    gpu_capacity: float
    cpu_capacity: float
    gpu_used: int = 0
    cpu_used: int = 0
    inflight_out: int = 0
    inflight_in: int = 0
    residency: dict = field(default_factory=dict)

    def check(self) -> None:
        assert 0 <= self.gpu_used <= self.gpu_capacity + 1e-6, "gpu tier overflow"
        assert 0 <= self.cpu_used <= self.cpu_capacity + 1e-6, "cpu tier overflow"
        assert self.inflight_out >= 0 and self.inflight_in >= 0


@dataclass(frozen=True)
class SimOptions:
    overlap: bool = True
    mode: Mode = Mode.ROOFLINE
    charge_p2p: bool = False
    kv_layout: KVLayout = KVLayout.HND
    nhd_efficiency: float = 0.5
    full_duplex: bool = True
    force_mixed: bool = False
    seed: int = 0

    def as_dict(self) -> dict:
        return {
            "overlap": self.overlap,
            "mode": self.mode.value,
            "charge_p2p": self.charge_p2p,
            "kv_layout": self.kv_layout.value,
            "nhd_efficiency": self.nhd_efficiency,
            "full_duplex": self.full_duplex,
            "force_mixed": self.force_mixed,
            "seed": self.seed,
        }


@dataclass(frozen=True)
class Event:
    """One timestamped record; gpu_id holds the data-parallel replica index."""

    t: float
    kind: str
    seq_id: int | str | None = None
    gpu_id: int | None = None
    bytes: int | None = None
    extra: tuple[tuple[str, object], ...] = ()

    @property
    def payload(self) -> dict:
        return dict(self.extra)

    def serialize(self) -> str:
        doc = {"t": repr(self.t), "kind": self.kind, "seq_id": self.seq_id, "gpu_id": self.gpu_id,
               "bytes": self.bytes, "extra": [[k, v] for k, v in self.extra]}
        return json.dumps(doc, sort_keys=True)


def _cell(v) -> str:
    return "" if v is None else str(v)


@dataclass
class SimReport:
    makespan: float
    requests_per_second: float
    tokens_per_second: float
    prefill_time: float
    decode_time: float
    reshard_time: float
    stalled_transfer_time: float
    transitions: int
    event_log: tuple[Event, ...]
    config: dict
    final_kv_state: TieredKVState
    # B200 additions (not in the reference report): generated token ids per
    # request and measured transfer statistics.
    outputs: dict = field(default_factory=dict)
    measured: dict = field(default_factory=dict)

    def to_document(self) -> str:
        doc = {
            "makespan_s": self.makespan,
            "requests_per_second": self.requests_per_second,
            "tokens_per_second": self.tokens_per_second,
            "prefill_time_s": self.prefill_time,
            "decode_time_s": self.decode_time,
            "reshard_time_s": self.reshard_time,
            "stalled_transfer_time_s": self.stalled_transfer_time,
            "transitions": self.transitions,
            "num_events": len(self.event_log),
            "config": self.config,
        }
        return json.dumps(doc, indent=2, sort_keys=True)

    def events_csv(self) -> str:
        lines = ["timestamp_s,event,seq_id,gpu_id,bytes"]
        for ev in self.event_log:
            seqs = ev.payload.get("seqs")
            ids = seqs if seqs else (ev.seq_id,)
            for sid in ids:
                lines.append(f"{ev.t!r},{ev.kind},{_cell(sid)},{_cell(ev.gpu_id)},{_cell(ev.bytes)}")
        return "\n".join(lines) + "\n"

    def write_events_csv(self, path) -> None:
        with open(path, "w", encoding="utf-8") as fh:
            fh.write(self.events_csv())

    def serialize_events(self) -> str:
        return "\n".join(ev.serialize() for ev in self.event_log)


@dataclass(frozen=True)
class ReplayVerdict:
    ok: bool
    violation: str | None = None
    event_index: int | None = None

    def __bool__(self) -> bool:
        return self.ok


def replay_check(report: SimReport) -> ReplayVerdict:
    """Re-validate KV conservation, tier capacity and decode counts from the
    event log alone (same rules as sim.py:764-837)."""
    gpu_cap = report.config["gpu_kv_capacity_bytes"]
    cpu_cap = report.config["cpu_kv_capacity_bytes"]
    used = {"gpu": 0, "cpu": 0}
    state: dict = {}
    size: dict = {}
    done: dict = {}
    want: dict = {}
    last_t = 0.0
    for i, ev in enumerate(report.event_log):
        if ev.t < last_t - 1e-12:
            return ReplayVerdict(False, "timestamps decrease", i)
        last_t = max(last_t, ev.t)
        sid, k = ev.seq_id, ev.kind
        if k == "prefill_complete":
            if sid in state:
                return ReplayVerdict(False, f"prefill repeated for {sid!r}", i)
            state[sid], size[sid], done[sid] = Residency.GPU, ev.bytes, 0
            want[sid] = ev.payload["output_len"]
            used["gpu"] += ev.bytes
        elif k == "swap_out_complete":
            if state.get(sid) is not Residency.GPU:
                return ReplayVerdict(False, f"swap-out of non-resident {sid!r}", i)
            state[sid] = Residency.CPU
            used["gpu"] -= ev.bytes
            used["cpu"] += ev.bytes
        elif k == "swap_in_start":
            if state.get(sid) is not Residency.CPU:
                return ReplayVerdict(False, f"swap-in of non-buffered {sid!r}", i)
            state[sid] = Residency.IN_TRANSIT
            used["cpu"] -= ev.bytes
        elif k == "swap_in_complete":
            if state.get(sid) is not Residency.IN_TRANSIT:
                return ReplayVerdict(False, f"swap-in completion without start for {sid!r}", i)
            state[sid] = Residency.GPU
            used["gpu"] += ev.bytes
        elif k == "decode_step":
            for s in ev.payload["seqs"]:
                if state.get(s) is not Residency.GPU:
                    return ReplayVerdict(False, f"decode before residency for {s!r}", i)
                done[s] += 1
                if done[s] > want[s]:
                    return ReplayVerdict(False, f"decode overrun for {s!r}", i)
        elif k == "kv_release":
            if state.get(sid) is not Residency.GPU:
                return ReplayVerdict(False, f"release of non-resident {sid!r}", i)
            if done[sid] != want[sid]:
                return ReplayVerdict(False, f"release before completion for {sid!r}", i)
            state[sid] = Residency.RELEASED
            used["gpu"] -= ev.bytes
        if used["gpu"] > gpu_cap + 1e-6 or used["gpu"] < 0:
            return ReplayVerdict(False, "tier overflow (gpu)", i)
        if used["cpu"] > cpu_cap + 1e-6 or used["cpu"] < 0:
            return ReplayVerdict(False, "tier overflow (cpu)", i)
    if len(state) != report.config["num_requests"]:
        return ReplayVerdict(False, f"saw {len(state)} sequences, expected {report.config['num_requests']}")
    for sid, st in state.items():
        if st is not Residency.RELEASED:
            return ReplayVerdict(False, f"sequence {sid!r} never released")
        if done[sid] != want[sid]:
            return ReplayVerdict(False, f"sequence {sid!r} decoded {done[sid]} of {want[sid]}")
    if used["gpu"] or used["cpu"]:
        return ReplayVerdict(False, "kv bytes leaked")
    return ReplayVerdict(True)
