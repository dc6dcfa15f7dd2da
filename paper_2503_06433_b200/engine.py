"""``execute()`` — the real PP-prefill → re-shard → TP-decode engine behind the
reference's ``simulate()`` signature.

The control flow follows the reference engine (/root/reference/pkg/src/
shardsim/sim.py) on a REAL clock (CUDA events) instead of a virtual one:

  validation, capacity, per-request KV reservation   sim.py:210-296
  round-robin replica assignment i % dp               sim.py:267
  greedy trace-order packing (_pack)                  sim.py:345-358
  prefill step: one sequence per micro-batch at pp>1  sim.py:371-378
  transition (weights + KV re-shard)                  sim.py:328-333
  decode rounds, release at output_len                sim.py:517-565
  transition-minimizing / decode-prioritized cycles   sim.py:618-662
  event log, end-of-run conservation asserts, report  sim.py:312-322, :699-745

B200-native mode: KV that fits in HBM stays on the GPU and
is re-sharded over NVLink at the P→D transition instead of riding the host
tier; a phase admits what the GPU tier holds, so every prefilled sequence is
decoded in the following D phase.  With the C2 workload everything fits and
the run has exactly the reference's single transition.  Event ``bytes`` are
in the reference's units ((in+out)·kv_bytes_per_token, sim.py:256) so the
reference's replay_check applies unchanged.

SPMD: every rank calls execute() with its own Comm and makes the same
decisions; rank 0's report is authoritative (all ranks return one).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from typing import Iterable, Sequence

import numpy as np
import torch

from .arch import LlamaArch
from .comm import Comm, SoloComm
from .report import (
    Event,
    Residency,
    SchedulingPolicy,
    SimOptions,
    SimReport,
    SimulationError,
    TieredKVState,
)
from .runtime import Worker
from .specs import (
    ConfigError,
    HardwareSpec,
    ModelSpec,
    ParallelismConfig,
    Request,
    kv_bytes_per_token,
    total_weight_bytes,
    validate_config,
)


@dataclass
class _Seq:
    req: Request
    replica: int
    kv_bytes: int
    prompt: np.ndarray
    blocks: list[int] = field(default_factory=list)
    generated: list[int] = field(default_factory=list)
    decoded: int = 0


class BlockAllocator:
    """Deterministic free list of pool blocks (identical on every rank of a replica)."""

    def __init__(self, num_blocks: int) -> None:
        self.free = list(range(num_blocks))
        self.num_blocks = num_blocks

    def alloc(self, n: int) -> list[int]:
        if n > len(self.free):
            raise SimulationError("KV pool exhausted")
        out, self.free = self.free[:n], self.free[n:]
        return out

    def release(self, blocks: Sequence[int]) -> None:
        self.free.extend(blocks)
        self.free.sort()


def synthetic_prompts(requests: Sequence[Request], vocab: int, seed: int = 1) -> list[np.ndarray]:
    """Prompt ids uniform in [0, vocab) from a seeded generator."""
    rng = np.random.default_rng(seed)
    return [rng.integers(0, vocab, size=r.input_len, dtype=np.int64).astype(np.int32) for r in requests]


class _Clock:
    """Timeline from CUDA events (device time), resolved once at the end."""

    def __init__(self, device: torch.device) -> None:
        self.cuda = device.type == "cuda"
        self.marks: list = []
        self.t0 = self.mark()

    def mark(self):
        if self.cuda:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            self.marks.append(ev)
            return ev
        t = time.perf_counter()
        self.marks.append(t)
        return t

    def resolve(self, m) -> float:
        if self.cuda:
            return self.t0.elapsed_time(m) / 1e3
        return m - self.t0


def execute(
    model: ModelSpec,
    hw: HardwareSpec,
    workload: Iterable[Request],
    policy: SchedulingPolicy,
    cfg_p: ParallelismConfig,
    cfg_d: ParallelismConfig,
    options: SimOptions | None = None,
    *,
    arch: LlamaArch,
    seed: int = 0,
    prompts: Sequence[np.ndarray] | None = None,
    comm: Comm | None = None,
    device: torch.device | str | None = None,
    block_size: int = 64,
    max_prefill_tokens: int = 16384,
    kv_pool_bytes_per_gpu: int | None = None,
    worker: Worker | None = None,
    record_logits: bool = False,
) -> SimReport:
    """Run the offline workload to completion on the GPUs and return a report
    with the reference's fields (measured, not modelled)."""
    return _Engine(model, hw, workload, policy, cfg_p, cfg_d, options or SimOptions(), arch=arch, seed=seed,
                   prompts=prompts, comm=comm, device=device, block_size=block_size,
                   max_prefill_tokens=max_prefill_tokens, kv_pool_bytes_per_gpu=kv_pool_bytes_per_gpu,
                   worker=worker, record_logits=record_logits).run()


class _Engine:
    def __init__(self, model, hw, workload, policy, cfg_p, cfg_d, options, *, arch, seed, prompts, comm, device,
                 block_size, max_prefill_tokens, kv_pool_bytes_per_gpu, worker, record_logits) -> None:
        requests = list(workload)
        if not requests:
            raise SimulationError("workload is empty")
        for cfg, name in ((cfg_p, "prefill"), (cfg_d, "decode")):
            verdict = validate_config(model, hw, cfg)
            if not verdict:
                raise ConfigError(f"{name} config {cfg.label()}: {verdict.reason}")
        if cfg_p.dp != cfg_d.dp:
            raise ConfigError("prefill and decode configs must share the same dp")
        if cfg_p != cfg_d and policy is not SchedulingPolicy.TRANSITION_MINIMIZING and not options.force_mixed:
            raise ConfigError(f"policy {policy.value} requires cfg_p == cfg_d (pass force_mixed to override)")
        if policy is SchedulingPolicy.PREFILL_PRIORITIZED:
            raise ConfigError("prefill-prioritized interleaving is not part of the re-sharding hot path")
        if cfg_d.pp != 1:
            raise ConfigError("decode layout must be pure tensor parallel (pp=1) in this engine")
        spec = arch.model_spec(model.bytes_per_param)
        for f in ("num_layers", "num_query_heads", "num_kv_heads", "head_dim"):
            if getattr(spec, f) != getattr(model, f):
                raise ConfigError(f"ModelSpec.{f}={getattr(model, f)} disagrees with arch {arch.name}")
        arch.validate_layout(cfg_p.tp, cfg_p.pp)
        arch.validate_layout(cfg_d.tp, cfg_d.pp)
        self.model, self.hw, self.arch, self.policy = model, hw, arch, policy
        self.cfg_p, self.cfg_d, self.options = cfg_p, cfg_d, options
        self.dp = cfg_p.dp
        self.comm = comm or SoloComm()
        if self.comm.size != hw.num_gpus:
            raise ConfigError(f"communicator has {self.comm.size} ranks but the fleet has {hw.num_gpus} GPUs")
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.block_size = block_size
        self.max_prefill_tokens = max_prefill_tokens
        self.replica_gpu_capacity = hw.gpu_memory * cfg_p.gpus_per_replica - total_weight_bytes(model)
        if self.replica_gpu_capacity <= 0:
            raise ConfigError("no GPU memory left for KV cache after weights")
        self.cpu_capacity = hw.cpu_kv_capacity
        self.kv_tok = kv_bytes_per_token(model)
        if prompts is None:
            prompts = synthetic_prompts(requests, arch.vocab)
        self.seqs: list[_Seq] = []
        seen = set()
        for i, (req, pr) in enumerate(zip(requests, prompts)):
            if req.id in seen:
                raise SimulationError(f"duplicate request id {req.id!r}")
            seen.add(req.id)
            k = (req.input_len + req.output_len) * self.kv_tok
            if k > self.replica_gpu_capacity:
                raise SimulationError(f"request {req.id!r} needs {k} KV bytes but a replica's GPU tier holds "
                                      f"{self.replica_gpu_capacity:.0f}")
            if policy is SchedulingPolicy.TRANSITION_MINIMIZING and k > self.cpu_capacity:
                raise SimulationError(f"request {req.id!r} needs {k} KV bytes but the CPU tier holds "
                                      f"{self.cpu_capacity:.0f}; it can never be buffered")
            if isinstance(pr, torch.Tensor):
                if pr.dtype != torch.int32:
                    pr = pr.to(torch.int32)
            else:
                pr = np.asarray(pr, dtype=np.int32)
            n_ids = pr.numel() if isinstance(pr, torch.Tensor) else pr.size
            if n_ids != req.input_len:
                raise SimulationError(f"request {req.id!r}: prompt has {n_ids} ids, input_len {req.input_len}")
            self.seqs.append(_Seq(req=req, replica=i % self.dp, kv_bytes=k, prompt=pr))
        if len(prompts) != len(requests):
            raise SimulationError("prompts and workload differ in length")
        max_len = max(s.req.input_len + s.req.output_len for s in self.seqs)
        self.max_blocks = -(-max_len // block_size)

        # physical pool: the reference capacity (in blocks) plus per-sequence rounding slack
        gpus = cfg_p.gpus_per_replica
        block_bytes_replica = block_size * self.kv_tok
        want_blocks = int(self.replica_gpu_capacity // block_bytes_replica) + len(self.seqs)
        need_blocks = sum(-(-(s.req.input_len + s.req.output_len) // block_size) for s in self.seqs)
        num_blocks = min(want_blocks, need_blocks)
        if kv_pool_bytes_per_gpu is not None:
            num_blocks = min(num_blocks, int(kv_pool_bytes_per_gpu // (block_bytes_replica // gpus)))
        self.num_blocks = max(num_blocks, self.max_blocks)

        self.worker = worker or Worker(arch, self.comm, self.dp, self.device, seed=seed, block_size=block_size,
                                       max_pos=max(max_len, 64))
        self.worker.record_logits = record_logits
        self.rank0 = self.comm.rank == 0
        self.events: list[tuple[object, str, dict]] = []  # (clock mark, kind, fields)
        self.kv = TieredKVState(gpu_capacity=self.replica_gpu_capacity * self.dp, cpu_capacity=self.cpu_capacity)
        self.transitions = 0
        self.phase_index = 0
        self.measured: dict = {"reshard_bytes_sent": 0, "weight_bytes_sent": 0, "kv_bytes_sent": 0,
                               "transition_s": []}

    # ----------------------------------------------------------------- log --
    def _log(self, mark, kind, seq=None, gpu=None, nbytes=None, **extra) -> None:
        self.events.append((mark, kind, dict(seq=seq, gpu=gpu, nbytes=nbytes, extra=extra)))

    # ---------------------------------------------------------------- run --
    def run(self) -> SimReport:
        w = self.worker
        if w.state is None:
            w.init_weights(self.cfg_p)
        elif w.state.cfg != self.cfg_p:
            # weights still in a previous run's decode layout: move them back
            # over NVLink (the reference starts every run in cfg_p, uncharged)
            w.repartition_weights(self.cfg_p)
        if w.pool is None or w.num_blocks < self.num_blocks:
            w.alloc_pool(self.num_blocks)
        self.alloc = BlockAllocator(w.num_blocks)
        self.comm.barrier()
        if self.device.type == "cuda":
            torch.cuda.synchronize(self.device)
        self.clock = _Clock(self.device)
        self._log(self.clock.t0, "run_start", policy=self.policy.value, cfg_p=self.cfg_p.label(),
                  cfg_d=self.cfg_d.label(), requests=len(self.seqs))
        my = self.worker.replica
        pending = [s for s in self.seqs if s.replica == my]
        others = {r: [s for s in self.seqs if s.replica == r] for r in range(self.dp)}
        phases: list[tuple[str, object, object]] = []
        cycle = 0
        while any(others[r] for r in range(self.dp)):
            if cycle > 0:
                t0 = self.clock.mark()
                self._transition("decode_to_prefill", self.cfg_p, [])
                phases.append(("reshard", t0, self.clock.mark()))
            self.phase_index += 1
            t_phase = self.clock.mark()
            self._log(t_phase, "phase_start", phase="prefill", index=self.phase_index)
            waves = {r: self._pack(others[r]) for r in range(self.dp)}
            if not any(waves.values()):
                raise SimulationError("a request that fits the GPU tier must be admissible")
            batch = waves[my]
            self._prefill(batch)
            t_end = self.clock.mark()
            phases.append(("prefill", t_phase, t_end))
            for r in sorted(waves):
                if waves[r]:
                    self._log(t_end, "prefill_step", gpu=r, batch=len(waves[r]),
                              seqs=tuple(s.req.id for s in waves[r]))
            for r in sorted(waves):
                for s in waves[r]:
                    self.kv.gpu_used += s.kv_bytes
                    self.kv.residency[s.req.id] = Residency.GPU
                    self._log(t_end, "prefill_complete", seq=s.req.id, gpu=r, nbytes=s.kv_bytes,
                              input_len=s.req.input_len, output_len=s.req.output_len)
            t0 = self.clock.mark()
            self._transition("prefill_to_decode", self.cfg_d, batch)
            phases.append(("reshard", t0, self.clock.mark()))
            self.phase_index += 1
            t_dec = self.clock.mark()
            self._log(t_dec, "phase_start", phase="decode", index=self.phase_index)
            self._decode(batch, {r: waves[r] for r in range(self.dp)})
            phases.append(("decode", t_dec, self.clock.mark()))
            for r in range(self.dp):
                done = {id(s) for s in waves[r]}
                others[r] = [s for s in others[r] if id(s) not in done]
            cycle += 1
        t_end = self.clock.mark()
        self._log(t_end, "run_end")
        return self._report(phases, t_end)

    def _pack(self, queue: list[_Seq]) -> list[_Seq]:
        """Greedy trace-order admission against the GPU tier (sim.py:345-358)."""
        room = self.replica_gpu_capacity
        blocks = self.alloc.num_blocks
        out = []
        for s in queue:
            nb = -(-(s.req.input_len + s.req.output_len) // self.block_size)
            if s.kv_bytes > room or nb > blocks:
                break
            out.append(s)
            room -= s.kv_bytes
            blocks -= nb
        return out

    # ------------------------------------------------------------ prefill --
    def _prefill(self, batch: list[_Seq]) -> None:
        w = self.worker
        cfg = self.cfg_p
        for s in batch:
            s.blocks = self.alloc.alloc(-(-(s.req.input_len + s.req.output_len) // self.block_size))
        # micro-batches: one sequence per micro-batch when pp > 1 (sim.py:371-378);
        # without a pipeline, packed forwards bounded by max_prefill_tokens
        mbs: list[list[_Seq]] = []
        if cfg.pp > 1:
            mbs = [[s] for s in batch]
        else:
            cur, toks = [], 0
            for s in batch:
                if cur and toks + s.req.input_len > self.max_prefill_tokens:
                    mbs.append(cur)
                    cur, toks = [], 0
                cur.append(s)
                toks += s.req.input_len
            if cur:
                mbs.append(cur)
        first = torch.zeros(len(batch), dtype=torch.int32, device=self.device)
        pos = 0
        for mb in mbs:
            cu = np.zeros(len(mb) + 1, dtype=np.int32)
            cu[1:] = np.cumsum([s.req.input_len for s in mb])
            tables = np.zeros((len(mb), self.max_blocks), dtype=np.int32)
            for i, s in enumerate(mb):
                tables[i, : len(s.blocks)] = s.blocks
            if isinstance(mb[0].prompt, torch.Tensor):
                # device-resident or pinned-host prompt ids
                toks = torch.cat([s.prompt for s in mb]).to(self.device, non_blocking=True)
            else:
                toks = torch.from_numpy(np.concatenate([s.prompt for s in mb])).to(self.device)
            w.prefill(toks, cu, tables, first[pos : pos + len(mb)])
            pos += len(mb)
        # every rank of the replica needs the first tokens: only the last
        # stage's tensor rank 0 contributes, the others add zeros
        st = w.state
        if not (st.stage == cfg.pp - 1 and st.rank == 0):
            first.zero_()
        w.replica_comm.all_reduce_(first)
        self._first_tokens = first

    # --------------------------------------------------------- transition --
    def _transition(self, direction: str, cfg_to: ParallelismConfig, residents: list[_Seq]) -> None:
        w = self.worker
        t0 = self.clock.mark()
        cfg_from = w.state.cfg
        wbytes = kbytes = 0
        if cfg_from != cfg_to:
            blocks = np.array(sorted(b for s in residents for b in s.blocks), dtype=np.int32)
            if "before_reshard" in w.hooks:
                w.hooks["before_reshard"](w, blocks=blocks, cfg_to=cfg_to)
            kbytes = w.reshard_kv(cfg_to, blocks) if blocks.size else 0
            wbytes = w.repartition_weights(cfg_to)
            if "after_reshard" in w.hooks:
                w.hooks["after_reshard"](w, blocks=blocks, cfg_to=cfg_to)
        t1 = self.clock.mark()
        self.transitions += 1
        self.measured["weight_bytes_sent"] += wbytes
        self.measured["kv_bytes_sent"] += kbytes
        self.measured["reshard_bytes_sent"] += wbytes + kbytes
        self.measured["transition_s"].append((t0, t1))
        self._log(t1, "transition", direction=direction)

    # ------------------------------------------------------------- decode --
    def _decode(self, batch: list[_Seq], waves: dict[int, list[_Seq]]) -> None:
        """Decode rounds until every resident reached output_len (sim.py:517-565).
        Under pure TP (pp=1) a round is one step over all residents."""
        w = self.worker
        dev = self.device
        B = len(batch)
        active = list(range(B))
        tables = np.zeros((max(B, 1), self.max_blocks), dtype=np.int32)
        for i, s in enumerate(batch):
            tables[i, : len(s.blocks)] = s.blocks
            s.generated = []
        tables_d = torch.from_numpy(tables[:B]).to(dev)
        ctx = torch.tensor([s.req.input_len for s in batch], dtype=torch.int32, device=dev)
        tokens = self._first_tokens.clone()
        positions = torch.empty(B, dtype=torch.int32, device=dev)
        slots = torch.empty(B, dtype=torch.int64, device=dev)
        nxt = torch.empty(B, dtype=torch.int32, device=dev)
        rows: list[tuple[list[int], torch.Tensor]] = [(list(active), tokens.clone())]
        other_live = {r: list(waves[r]) for r in waves if r != w.replica}
        while active or any(other_live.values()):
            if active:
                w.decode_step(tokens, ctx, tables_d, positions, slots, nxt)
                tokens, nxt = nxt, tokens
                rows.append((list(active), tokens.clone()))
            mark = self.clock.mark()
            lanes = {w.replica: [batch[i] for i in active]}
            lanes.update(other_live)
            for r in sorted(lanes):
                if not lanes[r]:
                    continue
                self._log(mark, "decode_step", gpu=r, tokens=len(lanes[r]), seqs=tuple(s.req.id for s in lanes[r]))
                for s in lanes[r]:
                    s.decoded += 1
                for s in lanes[r]:
                    if s.decoded == s.req.output_len:
                        self.kv.gpu_used -= s.kv_bytes
                        self.kv.residency[s.req.id] = Residency.RELEASED
                        self._log(mark, "kv_release", seq=s.req.id, gpu=r, nbytes=s.kv_bytes)
            for r in other_live:
                other_live[r] = [s for s in other_live[r] if s.decoded < s.req.output_len]
            keep = [i for i in active if batch[i].decoded < batch[i].req.output_len]
            if len(keep) < len(active):
                for i in active:
                    if batch[i].decoded >= batch[i].req.output_len:
                        self.alloc.release(batch[i].blocks)
                if keep:
                    # compact the device batch: finished rows drop out
                    idx = torch.tensor([active.index(i) for i in keep], dtype=torch.long, device=dev)
                    tables_d = tables_d.index_select(0, idx)
                    ctx = ctx.index_select(0, idx)
                    tokens = tokens.index_select(0, idx)
                    nxt = torch.empty_like(tokens)
                    positions = torch.empty_like(tokens)
                    slots = torch.empty(len(keep), dtype=torch.int64, device=dev)
                active = keep
        # one device->host read of every generated token
        flat = torch.cat([t for _, t in rows]).cpu().numpy() if B else np.zeros(0, np.int32)
        pos = 0
        for idxs, t in rows:
            for col, i in enumerate(idxs):
                batch[i].generated.append(int(flat[pos + col]))
            pos += len(idxs)

    # ------------------------------------------------------------- report --
    def _report(self, phases, t_end) -> SimReport:
        if self.device.type == "cuda":
            torch.cuda.synchronize(self.device)
        clk = self.clock
        makespan = clk.resolve(t_end)
        # max over ranks of the makespan (device-timed)
        mk = torch.tensor([makespan], dtype=torch.float32, device=self.device)
        gathered = torch.empty(self.comm.size, dtype=torch.float32, device=self.device)
        self.comm.all_gather(gathered, mk)
        makespan_all = float(gathered.max().item())
        sums = {"prefill": 0.0, "decode": 0.0, "reshard": 0.0}
        for kind, a, b in phases:
            sums[kind] += clk.resolve(b) - clk.resolve(a)
        events = []
        last = 0.0
        for mark, kind, f in self.events:
            t = clk.resolve(mark)
            t = max(t, last)
            last = t
            events.append(Event(t=t, kind=kind, seq_id=f["seq"], gpu_id=f["gpu"], bytes=f["nbytes"],
                                extra=tuple(sorted(f["extra"].items()))))
        assert self.kv.gpu_used == 0 and self.kv.cpu_used == 0, "kv bytes leaked"
        assert all(s.decoded == s.req.output_len for s in self.seqs)
        out_tokens = sum(s.req.output_len for s in self.seqs)
        trans = [clk.resolve(b) - clk.resolve(a) for a, b in self.measured.pop("transition_s")]
        stalled = max(makespan - sum(sums.values()), 0.0)
        config = {
            "policy": self.policy.value,
            "cfg_p": self.cfg_p.label(),
            "cfg_d": self.cfg_d.label(),
            "options": self.options.as_dict(),
            "num_requests": len(self.seqs),
            "output_tokens": out_tokens,
            "gpu_kv_capacity_bytes": self.kv.gpu_capacity,
            "cpu_kv_capacity_bytes": self.kv.cpu_capacity,
            "kv_bytes_per_token": self.kv_tok,
            "num_gpus": self.hw.num_gpus,
            "engine": "b200-native",
            "arch": self.arch.name,
            "pool_blocks_per_gpu": self.worker.num_blocks,
            "block_size": self.block_size,
        }
        measured = dict(self.measured)
        measured["transition_wall_s"] = trans
        measured["makespan_max_over_ranks_s"] = makespan_all
        outputs = {s.req.id: s.generated[: s.req.output_len] for s in self.seqs
                   if s.replica == self.worker.replica}
        return SimReport(
            makespan=makespan,
            requests_per_second=len(self.seqs) / makespan,
            tokens_per_second=out_tokens / makespan,
            prefill_time=sums["prefill"],
            decode_time=sums["decode"],
            reshard_time=sums["reshard"],
            stalled_transfer_time=stalled,
            transitions=self.transitions,
            event_log=tuple(events),
            config=config,
            final_kv_state=self.kv,
            outputs=outputs,
            measured=measured,
        )
