"""``execute()`` — the real PP-prefill → re-shard → TP-decode engine behind the
reference's ``simulate()`` signature.

The control flow follows the reference engine (/root/reference/pkg/src/
shardsim/sim.py) on a REAL clock (CUDA events) instead of a virtual one:

  validation, capacity, per-request KV reservation   sim.py:210-296
  round-robin replica assignment i % dp               sim.py:267
  greedy trace-order packing (_pack)                  sim.py:345-358
  prefill step: one sequence per micro-batch at pp>1  sim.py:371-378
  swap-out to the host tier overlapped with prefill   sim.py:382-385, :417-429
  transition (weights + KV re-shard)                  sim.py:328-333
  decode rounds, release at output_len                sim.py:517-565
  FIFO prefetcher, continuous swap-in during decode   sim.py:436-513, :591-614
  transition-minimizing cycles                        sim.py:618-642
  event log, end-of-run conservation asserts, report  sim.py:312-322, :699-745

B200-native mode: KV that fits in HBM stays on the GPU and
is re-sharded over NVLink at the P→D transition; sequences beyond the GPU
tier are prefilled into a small reserve of pool blocks and swapped out to the
pinned host tier (HND, shared by the replica's GPUs).  P→D fires when the GPU
tier plus the host tier are full or work runs out.  During decode the
prefetcher swaps buffered sequences back in under the DECODE layout on a copy
stream and they join the running batch.  Event ``bytes`` are in the
reference's units ((in+out)·kv_bytes_per_token, sim.py:256) so the
reference's replay_check applies unchanged.

SPMD: every rank calls execute() with its own Comm and makes the same
decisions — admission of a swapped-in sequence happens a fixed number of
decode steps after its transfer started (the compute stream waits on the
transfer's event), never on a host-side timing query — so all ranks of a
replica always step the same batch.
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


@dataclass(eq=False)
class _Seq:
    req: Request
    replica: int
    kv_bytes: int
    prompt: object
    nblocks: int = 0
    blocks: list[int] = field(default_factory=list)
    generated: list[int] = field(default_factory=list)
    decoded: int = 0
    overflow: bool = False       # prefilled into the reserve and buffered in the host tier
    slot: int = -1
    first_token: int = 0
    admit_step: int = -1
    ticket: object = None


class BlockAllocator:
    """Deterministic free list of pool blocks (identical on every rank of a replica)."""

    def __init__(self, num_blocks: int) -> None:
        self.free = list(range(num_blocks))
        self.num_blocks = num_blocks

    @property
    def available(self) -> int:
        return len(self.free)

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
        self.t0 = self.mark()

    def mark(self):
        if self.cuda:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record()
            return ev
        return time.perf_counter()

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
    swap_in_flight: int = 4,
) -> SimReport:
    """Run the offline workload to completion on the GPUs and return a report
    with the reference's fields (measured, not modelled)."""
    return _Engine(model, hw, workload, policy, cfg_p, cfg_d, options or SimOptions(), arch=arch, seed=seed,
                   prompts=prompts, comm=comm, device=device, block_size=block_size,
                   max_prefill_tokens=max_prefill_tokens, kv_pool_bytes_per_gpu=kv_pool_bytes_per_gpu,
                   worker=worker, record_logits=record_logits, swap_in_flight=swap_in_flight).run()


class _Engine:
    def __init__(self, model, hw, workload, policy, cfg_p, cfg_d, options, *, arch, seed, prompts, comm, device,
                 block_size, max_prefill_tokens, kv_pool_bytes_per_gpu, worker, record_logits,
                 swap_in_flight) -> None:
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
        self.swap_in_flight = max(1, swap_in_flight)
        self.replica_gpu_capacity = hw.gpu_memory * cfg_p.gpus_per_replica - total_weight_bytes(model)
        if self.replica_gpu_capacity <= 0:
            raise ConfigError("no GPU memory left for KV cache after weights")
        self.cpu_capacity = hw.cpu_kv_capacity
        self.kv_tok = kv_bytes_per_token(model)
        if prompts is None:
            prompts = synthetic_prompts(requests, arch.vocab)
        if len(prompts) != len(requests):
            raise SimulationError("prompts and workload differ in length")
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
                pr = pr if pr.dtype == torch.int32 else pr.to(torch.int32)
                n_ids = pr.numel()
            else:
                pr = np.asarray(pr, dtype=np.int32)
                n_ids = pr.size
            if n_ids != req.input_len:
                raise SimulationError(f"request {req.id!r}: prompt has {n_ids} ids, input_len {req.input_len}")
            nb = -(-(req.input_len + req.output_len) // block_size)
            self.seqs.append(_Seq(req=req, replica=i % self.dp, kv_bytes=k, prompt=pr, nblocks=nb))
        max_len = max(s.req.input_len + s.req.output_len for s in self.seqs)
        self.max_blocks = -(-max_len // block_size)
        self.max_prompt = max(s.req.input_len for s in self.seqs)

        # physical pool: the reference capacity (in blocks) plus rounding slack,
        # never more than the whole workload needs
        gpus = cfg_p.gpus_per_replica
        block_bytes_replica = block_size * self.kv_tok
        # every replica's ranks size the same pool (shadow allocators mirror
        # the other replicas' schedules): the largest replica's share decides
        by_replica = [[s for s in self.seqs if s.replica == r] for r in range(self.dp)]
        want_blocks = int(self.replica_gpu_capacity // block_bytes_replica) + max(len(q) for q in by_replica)
        need_blocks = max(sum(s.nblocks for s in q) for q in by_replica)
        num_blocks = min(want_blocks, need_blocks)
        if kv_pool_bytes_per_gpu is not None:
            num_blocks = min(num_blocks, int(kv_pool_bytes_per_gpu // (block_bytes_replica // gpus)))
        self.num_blocks = max(num_blocks, self.max_blocks)
        # host tier: needed when a replica's demand exceeds its GPU tier
        demand = max(sum(s.kv_bytes for s in self.seqs if s.replica == r) for r in range(self.dp))
        self.use_tier = (demand > self.replica_gpu_capacity or need_blocks > self.num_blocks) and self.cpu_capacity > 0
        # reserve for prefilling overflow sequences before they are swapped out
        self.reserve_seqs = 1 if cfg_p.pp > 1 else max(1, min(4, self.max_prefill_tokens // max(self.max_prompt, 1)))
        self.reserve_blocks = self.reserve_seqs * self.max_blocks if self.use_tier else 0
        self.reserve_bytes = self.reserve_seqs * max(s.kv_bytes for s in self.seqs) if self.use_tier else 0
        if self.use_tier and self.reserve_blocks >= self.num_blocks:
            raise SimulationError("GPU KV pool too small to stage a prefill for the host tier")

        self.worker = worker or Worker(arch, self.comm, self.dp, self.device, seed=seed, block_size=block_size,
                                       max_pos=max(max_len, 64))
        self.worker.record_logits = record_logits
        self.events: list[tuple[object, str, dict]] = []  # (clock mark, kind, fields)
        self.kv = TieredKVState(gpu_capacity=self.replica_gpu_capacity * self.dp, cpu_capacity=self.cpu_capacity)
        self.transitions = 0
        self.phase_index = 0
        self.measured: dict = {"reshard_bytes_sent": 0, "weight_bytes_sent": 0, "kv_bytes_sent": 0,
                               "transition_s": [], "swapped_out": 0, "swap_bytes_per_gpu": 0}
        self.tier = None

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
        if self.use_tier:
            self._setup_tier()
        self.comm.barrier()
        if self.device.type == "cuda":
            torch.cuda.synchronize(self.device)
        self.clock = _Clock(self.device)
        self._log(self.clock.t0, "run_start", policy=self.policy.value, cfg_p=self.cfg_p.label(),
                  cfg_d=self.cfg_d.label(), requests=len(self.seqs))
        pending = {r: [s for s in self.seqs if s.replica == r] for r in range(self.dp)}
        phases: list[tuple[str, object, object]] = []
        cycle = 0
        while any(pending[r] for r in range(self.dp)):
            if cycle > 0:
                t0 = self.clock.mark()
                self._transition("decode_to_prefill", self.cfg_p, [])
                phases.append(("reshard", t0, self.clock.mark()))
            self.phase_index += 1
            t_phase = self.clock.mark()
            self._log(t_phase, "phase_start", phase="prefill", index=self.phase_index)
            cpu_room = self.cpu_capacity - self.kv.cpu_used
            waves: dict[int, list[_Seq]] = {}
            for r in range(self.dp):
                waves[r] = self._pack(pending[r], cpu_room)
                cpu_room -= sum(s.kv_bytes for s in waves[r] if s.overflow)
            if not any(waves.values()):
                raise SimulationError("a request that fits the GPU tier must be admissible")
            t_end = self._prefill_phase(waves)
            phases.append(("prefill", t_phase, t_end))
            residents = [s for s in waves[self.worker.replica] if not s.overflow]
            t0 = self.clock.mark()
            self._transition("prefill_to_decode", self.cfg_d, residents)
            phases.append(("reshard", t0, self.clock.mark()))
            self.phase_index += 1
            t_dec = self.clock.mark()
            self._log(t_dec, "phase_start", phase="decode", index=self.phase_index)
            self._decode_phase(waves)
            phases.append(("decode", t_dec, self.clock.mark()))
            for r in range(self.dp):
                done = {id(s) for s in waves[r]}
                pending[r] = [s for s in pending[r] if id(s) not in done]
            cycle += 1
        t_end = self.clock.mark()
        self._log(t_end, "run_end")
        return self._report(phases, t_end)

    def _setup_tier(self) -> None:
        from .hosttier import HostTier

        w = self.worker
        per_replica_bytes = self.cpu_capacity / self.dp
        slot_bytes = self.max_prompt * self.kv_tok
        n_slots = int(per_replica_bytes // max(slot_bytes, 1))
        n_slots = min(n_slots, len([s for s in self.seqs if s.replica == w.replica]))
        gpus = self.cfg_p.gpus_per_replica
        staging = self.max_prompt * self.kv_tok // gpus
        a = self.arch
        # pinned memory is allocated once per worker and reused by later runs
        # whose slot shape matches and whose slot count it covers; a larger
        # need replaces it (the old buffer is released first: pinned host
        # memory, not HBM, is what runs out at 13B/70B scale)
        shape = (self.max_prompt, staging)
        tier = getattr(w, "_host_tier", None)
        if tier is None or tier.shape_key != shape or tier.n_slots < max(n_slots, 1):
            w._host_tier = None
            del tier
            import gc

            gc.collect()
            if self.device.type == "cuda":
                torch.cuda.synchronize(self.device)
                torch._C._host_emptyCache()  # return cached pinned blocks to the OS
            tier = HostTier(w.replica_comm, self.device, a.num_layers, a.num_kv_heads, a.head_dim,
                            self.max_prompt, max(n_slots, 1), staging)
            tier.shape_key = shape
            w._host_tier = tier
        self.tier = tier
        self.tier.free = list(range(max(n_slots, 1)))
        self.slots_total = max(n_slots, 1)
        # deterministic admission lag (decode steps) for a swap-in: transfer
        # time of one sequence's piece at the host link rate over a nominal
        # 10 ms step, rounded up (identical on every rank)
        piece = self.max_prompt * self.kv_tok / gpus
        self.swap_lag = max(1, math.ceil(piece / self.hw.host_link_bandwidth / 0.010))

    def _pack(self, queue: list[_Seq], cpu_room: float) -> list[_Seq]:
        """Greedy trace-order admission (sim.py:345-358): GPU-resident while the
        GPU tier (bytes and pool blocks, minus the staging reserve) has room,
        then buffered in the host tier while it has room."""
        room = self.replica_gpu_capacity - self.reserve_bytes
        blocks = self.alloc.available - self.reserve_blocks
        slots = len(self.tier.free) if self.tier is not None else 0
        out = []
        spill = False
        for s in queue:
            if not spill and s.kv_bytes <= room and s.nblocks <= blocks:
                s.overflow = False
                room -= s.kv_bytes
                blocks -= s.nblocks
            elif self.use_tier and s.kv_bytes <= cpu_room and slots > 0 and s.nblocks <= self.reserve_blocks:
                spill = True
                s.overflow = True
                cpu_room -= s.kv_bytes
                slots -= 1
            else:
                break
            out.append(s)
        return out

    # ------------------------------------------------------------ prefill --
    def _micro_batches(self, seqs: list[_Seq], limit_seqs: int | None = None) -> list[list[_Seq]]:
        if self.cfg_p.pp > 1:
            return [[s] for s in seqs]  # one sequence per micro-batch (sim.py:371-378)
        mbs, cur, toks = [], [], 0
        for s in seqs:
            if cur and (toks + s.req.input_len > self.max_prefill_tokens or (limit_seqs and len(cur) >= limit_seqs)):
                mbs.append(cur)
                cur, toks = [], 0
            cur.append(s)
            toks += s.req.input_len
        if cur:
            mbs.append(cur)
        return mbs

    def _prefill_phase(self, waves: dict[int, list[_Seq]]):
        """Prefill this replica's wave: residents stay in HBM; overflow
        sequences go through the reserve and are swapped out to the host tier
        on the copy stream while the next micro-batch computes."""
        w = self.worker
        batch = waves[w.replica]
        residents = [s for s in batch if not s.overflow]
        overflow = [s for s in batch if s.overflow]
        first = torch.zeros(len(batch), dtype=torch.int32, device=self.device)
        index = {id(s): i for i, s in enumerate(batch)}
        for s in residents:
            s.blocks = self.alloc.alloc(s.nblocks)
        for mb in self._micro_batches(residents):
            self._run_prefill(mb, first, index)
        tickets = []
        st = w.state
        glayer0, ghead0 = st.weights.layer_begin, st.rank * st.weights.n_kv_heads
        for mb in self._micro_batches(overflow, limit_seqs=self.reserve_seqs):
            for s in mb:
                s.blocks = self.alloc.alloc(s.nblocks)
                s.slot = self.tier.alloc()
            self._run_prefill(mb, first, index)
            geo = w.geometry().as_tuple()
            for s in mb:
                blk = torch.tensor(s.blocks, dtype=torch.int32, device=self.device)
                tk = self.tier.swap_out(w.pool, geo, blk, s.req.input_len, s.slot, glayer0, ghead0, s.req.id)
                tickets.append((s, tk))
                # the gather is stream-ordered before any later prefill writes
                self.alloc.release(s.blocks)
                s.blocks = []
        if self.tier is not None:
            # every swap-out lands before the transition (ranks read each
            # other's pieces only after the transition's collectives)
            torch.cuda.current_stream(self.device).wait_stream(self.tier.copy_stream)
        # every rank of the replica needs the first tokens: only the last
        # stage's tensor rank 0 contributes, the others add zeros
        if not (st.stage == self.cfg_p.pp - 1 and st.rank == 0):
            first.zero_()
        w.replica_comm.all_reduce_(first)
        self._first = first
        firsts = first.cpu().numpy() if overflow else None
        for s in overflow:
            s.first_token = int(firsts[index[id(s)]])
        t_end = self.clock.mark()
        # log in the reference's order: step, completions, swap-outs
        for r in sorted(waves):
            if waves[r]:
                self._log(t_end, "prefill_step", gpu=r, batch=len(waves[r]), seqs=tuple(s.req.id for s in waves[r]))
        for r in sorted(waves):
            for s in waves[r]:
                if s.overflow:
                    continue
                self.kv.gpu_used += s.kv_bytes
                self.kv.residency[s.req.id] = Residency.GPU
                self._log(t_end, "prefill_complete", seq=s.req.id, gpu=r, nbytes=s.kv_bytes,
                          input_len=s.req.input_len, output_len=s.req.output_len)
        tk_by_id = {id(s): tk for s, tk in tickets}
        for r in sorted(waves):
            for s in waves[r]:
                if not s.overflow:
                    continue
                mark = tk_by_id[id(s)].done if id(s) in tk_by_id else t_end
                self.kv.gpu_used += s.kv_bytes
                self._log(mark, "prefill_complete", seq=s.req.id, gpu=r, nbytes=s.kv_bytes,
                          input_len=s.req.input_len, output_len=s.req.output_len)
                self.kv.gpu_used -= s.kv_bytes
                self.kv.cpu_used += s.kv_bytes
                self.kv.residency[s.req.id] = Residency.CPU
                self._log(mark, "swap_out_complete", seq=s.req.id, gpu=r, nbytes=s.kv_bytes)
                self.measured["swapped_out"] += 1
        return t_end

    def _run_prefill(self, mb: list[_Seq], first: torch.Tensor, index: dict) -> None:
        cu = np.zeros(len(mb) + 1, dtype=np.int32)
        cu[1:] = np.cumsum([s.req.input_len for s in mb])
        tables = np.zeros((len(mb), self.max_blocks), dtype=np.int32)
        for i, s in enumerate(mb):
            tables[i, : len(s.blocks)] = s.blocks
        if isinstance(mb[0].prompt, torch.Tensor):
            toks = torch.cat([s.prompt for s in mb]).to(self.device, non_blocking=True)
        else:
            toks = torch.from_numpy(np.concatenate([s.prompt for s in mb])).to(self.device)
        i0 = index[id(mb[0])]
        # micro-batches are contiguous in batch order
        self.worker.prefill(toks, cu, tables, first[i0 : i0 + len(mb)])

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
    def _decode_phase(self, waves: dict[int, list[_Seq]]) -> None:
        """Decode rounds until every sequence of the wave reached output_len
        (sim.py:517-565), with the FIFO prefetcher admitting host-tier
        sequences as pool blocks free up (sim.py:436-513).  All replicas'
        schedules advance in lockstep; only this rank's replica runs kernels."""
        w = self.worker
        my = w.replica
        dev = self.device
        lanes = {r: [s for s in waves[r] if not s.overflow] for r in waves}
        queues = {r: [s for s in waves[r] if s.overflow] for r in waves}
        inflight: dict[int, list[_Seq]] = {r: [] for r in waves}
        allocs = {r: (self.alloc if r == my else BlockAllocator(self.alloc.num_blocks)) for r in waves}
        for r in waves:
            if r != my:  # shadow allocators mirror the residents' blocks
                allocs[r].alloc(sum(s.nblocks for s in lanes[r]))
        gpu_room = {r: self.replica_gpu_capacity - sum(s.kv_bytes for s in lanes[r]) for r in waves}
        index = {id(s): i for i, s in enumerate(waves[my])}
        # device state of this replica's running batch
        batch: list[_Seq] = []
        tables_d = ctx = tokens = None
        rows: list[tuple[list[_Seq], torch.Tensor]] = []
        first_rows = self._first
        compute = torch.cuda.current_stream(dev)
        st = w.state
        ghead0, glayer0 = st.rank * st.weights.n_kv_heads, st.weights.layer_begin
        step = 0

        def rebuild(new_batch: list[_Seq], old: list[_Seq]):
            nonlocal tables_d, ctx, tokens
            keep = [old.index(s) for s in new_batch if s in old]
            fresh = [s for s in new_batch if s not in old]
            order = [s for s in new_batch if s in old] + fresh
            tab = np.zeros((len(order), self.max_blocks), dtype=np.int32)
            for i, s in enumerate(order):
                tab[i, : len(s.blocks)] = s.blocks
            parts_ctx, parts_tok = [], []
            if keep:
                idx = torch.tensor(keep, dtype=torch.long, device=dev)
                parts_ctx.append(ctx.index_select(0, idx))
                parts_tok.append(tokens.index_select(0, idx))
            if fresh:
                parts_ctx.append(torch.tensor([s.req.input_len for s in fresh], dtype=torch.int32, device=dev))
                ft = [first_rows[index[id(s)]].view(1) if not s.overflow else
                      torch.tensor([s.first_token], dtype=torch.int32, device=dev) for s in fresh]
                parts_tok.append(torch.cat(ft))
                rows.append((list(fresh), torch.cat(ft).clone()))
            tables_d = torch.from_numpy(tab).to(dev)
            ctx = torch.cat(parts_ctx).contiguous()
            tokens = torch.cat(parts_tok).contiguous()
            return order

        while any(lanes[r] or queues[r] or inflight[r] for r in waves):
            # 1. admissions: swap-ins whose lag expired (or, with an empty
            #    batch, the oldest in flight: the reference's wait-for-fill)
            for r in sorted(waves):
                ready = [s for s in inflight[r] if s.admit_step <= step]
                if not lanes[r] and not ready and inflight[r]:
                    ready = inflight[r][:1]
                for s in ready:
                    inflight[r].remove(s)
                    if r == my:
                        compute.wait_event(s.ticket.done)
                        self.tier.release(s.slot)
                    mark = self.clock.mark()
                    self.kv.inflight_in -= s.kv_bytes
                    self.kv.gpu_used += s.kv_bytes
                    self.kv.residency[s.req.id] = Residency.GPU
                    self._log(mark, "swap_in_complete", seq=s.req.id, gpu=r, nbytes=s.kv_bytes)
                    lanes[r].append(s)
            # 2. prefetch: FIFO while the GPU tier has room (sim.py:441-456)
            if self.tier is not None and any(queues[r] for r in waves):
                marker = torch.cuda.Event()
                marker.record(compute)
                self.tier.copy_stream.wait_event(marker)  # freed blocks are no longer read
                for r in sorted(waves):
                    while (queues[r] and len(inflight[r]) < self.swap_in_flight
                           and allocs[r].available >= queues[r][0].nblocks
                           and gpu_room[r] >= queues[r][0].kv_bytes):
                        s = queues[r].pop(0)
                        s.blocks = allocs[r].alloc(s.nblocks)
                        gpu_room[r] -= s.kv_bytes
                        s.admit_step = step + self.swap_lag
                        if r == my:
                            blk = torch.tensor(s.blocks, dtype=torch.int32, device=dev)
                            s.ticket = self.tier.swap_in(w.pool, w.geometry().as_tuple(), blk, s.req.input_len,
                                                         s.slot, glayer0, ghead0, s.req.id)
                        self.kv.cpu_used -= s.kv_bytes
                        self.kv.inflight_in += s.kv_bytes
                        self.kv.residency[s.req.id] = Residency.IN_TRANSIT
                        self._log(self.clock.mark(), "swap_in_start", seq=s.req.id, gpu=r, nbytes=s.kv_bytes)
                        inflight[r].append(s)
            if not any(lanes[r] for r in waves):
                continue  # nothing resident anywhere: the next pass admits the oldest transfer
            # 3. one decode step of every replica's batch
            if lanes[my] != batch:
                batch = rebuild(lanes[my], batch) if lanes[my] else []
                lanes[my] = list(batch)
            if batch:
                nxt = torch.empty_like(tokens)
                positions = torch.empty_like(tokens)
                slots = torch.empty(len(batch), dtype=torch.int64, device=dev)
                w.decode_step(tokens, ctx, tables_d, positions, slots, nxt)
                tokens = nxt
                rows.append((list(batch), tokens))
            step += 1
            mark = self.clock.mark()
            for r in sorted(waves):
                if not lanes[r]:
                    continue
                self._log(mark, "decode_step", gpu=r, tokens=len(lanes[r]), seqs=tuple(s.req.id for s in lanes[r]))
                for s in lanes[r]:
                    s.decoded += 1
                done = [s for s in lanes[r] if s.decoded == s.req.output_len]
                for s in done:
                    self.kv.gpu_used -= s.kv_bytes
                    self.kv.residency[s.req.id] = Residency.RELEASED
                    self._log(mark, "kv_release", seq=s.req.id, gpu=r, nbytes=s.kv_bytes)
                    allocs[r].release(s.blocks)
                    gpu_room[r] += s.kv_bytes
                if done:
                    lanes[r] = [s for s in lanes[r] if s.decoded < s.req.output_len]
        # one device->host read of every generated token of this replica
        if rows:
            flat = torch.cat([t for _, t in rows]).cpu().numpy()
            pos = 0
            for seqs, _ in rows:
                for col, s in enumerate(seqs):
                    s.generated.append(int(flat[pos + col]))
                pos += len(seqs)

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
            t = max(clk.resolve(mark), last)
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
            "host_tier": bool(self.use_tier),
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
