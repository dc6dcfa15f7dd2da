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
  decode rounds, ceil(n/pp) micro-batches at pp>1,    sim.py:517-565, :201-206
    release at output_len
  FIFO prefetcher, continuous swap-in during decode,  sim.py:436-513, :591-614
    wait-for-fill when nothing is resident
  policies: transition-minimizing cycles,             sim.py:618-642
            decode-prioritized (static batches),      sim.py:644-663
            prefill-prioritized (vLLM-style)          sim.py:666-695
  event log, end-of-run conservation asserts, report  sim.py:312-322, :699-745
  stalled transfer time = waits on the tier           sim.py:401, :602

Two transition-minimizing modes:
* ``tm_mode="native"`` (default, B200-native): KV that fits in HBM stays on
  the GPU and is re-sharded over NVLink at the P→D transition; only the
  sequences beyond the GPU tier are prefilled into a small reserve of pool
  blocks and swapped out to the pinned host tier (HND, shared by the
  replica's GPUs).  P→D fires when the GPU tier plus the host tier are full
  or work runs out.
* ``tm_mode="reference"``: the reference's schedule exactly — every prefill
  step packs against the whole GPU tier and the host room (sim.py:629),
  every prefilled sequence is swapped out (``swap_to_cpu=True``, sim.py:635)
  and comes back through the prefetcher under the decode layout.

During decode the prefetcher swaps buffered sequences back in under the
DECODE layout on a copy stream and they join the running batch.  Event
``bytes`` are in the reference's units ((in+out)·kv_bytes_per_token,
sim.py:256) so the reference's replay_check applies unchanged.

SPMD: every rank calls execute() with its own Comm and makes the same
decisions — admission of a swapped-in sequence happens a fixed number of
decode steps after its transfer started (the compute stream waits on the
transfer's event), never on a host-side timing query; every rank keeps
shadow block allocators and slot lists of the other replicas, so all ranks
log the same global schedule.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from typing import Callable, Iterable, Sequence

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
    first_token: int = 0         # host copy (buffered sequences)
    first_dev: object = None     # device view of the prefill's greedy token (resident sequences)
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


def ceil_chunks(items: list, pp: int) -> list[list]:
    """At most pp micro-batches of ceil(n/pp), the last possibly smaller
    (sim.py:201-206): the decode micro-batching of a pipeline layout."""
    if not items:
        return []
    size = math.ceil(len(items) / pp)
    return [items[i : i + size] for i in range(0, len(items), size)]


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
    swap_lag: int | None = None,
    tm_mode: str = "native",
) -> SimReport:
    """Run the offline workload to completion on the GPUs and return a report
    with the reference's fields (measured, not modelled).

    ``tm_mode``: "native" (KV that fits stays in HBM) or "reference" (every
    wave through the host tier, the reference's schedule).  ``swap_lag``:
    decode steps between a swap-in's start and its admission (default: the
    transfer time at the host link rate over a nominal 10 ms step)."""
    return _Engine(model, hw, workload, policy, cfg_p, cfg_d, options or SimOptions(), arch=arch, seed=seed,
                   prompts=prompts, comm=comm, device=device, block_size=block_size,
                   max_prefill_tokens=max_prefill_tokens, kv_pool_bytes_per_gpu=kv_pool_bytes_per_gpu,
                   worker=worker, record_logits=record_logits, swap_in_flight=swap_in_flight,
                   swap_lag=swap_lag, tm_mode=tm_mode).run()


class _Engine:
    def __init__(self, model, hw, workload, policy, cfg_p, cfg_d, options, *, arch, seed, prompts, comm, device,
                 block_size, max_prefill_tokens, kv_pool_bytes_per_gpu, worker, record_logits,
                 swap_in_flight, swap_lag, tm_mode) -> None:
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
        if tm_mode not in ("native", "reference"):
            raise ConfigError(f"tm_mode must be 'native' or 'reference', not {tm_mode!r}")
        spec = arch.model_spec(model.bytes_per_param)
        for f in ("num_layers", "num_query_heads", "num_kv_heads", "head_dim"):
            if getattr(spec, f) != getattr(model, f):
                raise ConfigError(f"ModelSpec.{f}={getattr(model, f)} disagrees with arch {arch.name}")
        arch.validate_layout(cfg_p.tp, cfg_p.pp)
        arch.validate_layout(cfg_d.tp, cfg_d.pp)
        self.model, self.hw, self.arch, self.policy = model, hw, arch, policy
        self.cfg_p, self.cfg_d, self.options = cfg_p, cfg_d, options
        self.tm_mode = tm_mode if policy is SchedulingPolicy.TRANSITION_MINIMIZING else "native"
        self.dp = cfg_p.dp
        self.comm = comm or SoloComm()
        if self.comm.size != hw.num_gpus:
            raise ConfigError(f"communicator has {self.comm.size} ranks but the fleet has {hw.num_gpus} GPUs")
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.block_size = block_size
        self.max_prefill_tokens = max_prefill_tokens
        self.swap_in_flight = max(1, swap_in_flight)
        self.swap_lag_override = swap_lag
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

        # physical pool (blocks per GPU): the reference capacity (in blocks)
        # plus rounding slack, never more than the largest replica's share
        # of the workload needs; run() caps it by the HBM left after the
        # weights and the runtime reserve
        gpus = cfg_p.gpus_per_replica
        self.block_bytes_gpu = block_size * self.kv_tok // gpus
        by_replica = [[s for s in self.seqs if s.replica == r] for r in range(self.dp)]
        want_blocks = int(self.replica_gpu_capacity // (block_size * self.kv_tok)) + max(len(q) for q in by_replica)
        self.need_blocks = max(sum(s.nblocks for s in q) for q in by_replica)
        self.num_blocks = max(min(want_blocks, self.need_blocks), self.max_blocks)
        if kv_pool_bytes_per_gpu is not None:
            self.num_blocks = max(min(self.num_blocks, int(kv_pool_bytes_per_gpu // self.block_bytes_gpu)),
                                  self.max_blocks)
        self.demand = max(sum(s.kv_bytes for s in q) for q in by_replica)

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
        self.slots: dict[int, list[int]] = {r: [] for r in range(self.dp)}
        self.stalls: list[tuple[str, object, object]] = []   # (kind, before, after) marks on the compute stream

    # ------------------------------------------------------- memory plan --
    def _plan_tier(self) -> None:
        """Host tier use and the prefill reserve for the final pool size."""
        ref_mode = self.tm_mode == "reference"
        tm = self.policy is SchedulingPolicy.TRANSITION_MINIMIZING
        self.use_tier = tm and self.cpu_capacity > 0 and (
            ref_mode or self.demand > self.replica_gpu_capacity or self.need_blocks > self.num_blocks)
        if ref_mode:
            # the whole GPU tier is the staging area of every prefill step
            self.reserve_seqs = max(1, self.num_blocks // self.max_blocks)
            self.reserve_blocks = self.num_blocks
            self.reserve_bytes = 0
            return
        # reserve for prefilling overflow sequences before they are swapped out
        self.reserve_seqs = 1 if self.cfg_p.pp > 1 else max(1, min(4, self.max_prefill_tokens // max(self.max_prompt, 1)))
        self.reserve_blocks = self.reserve_seqs * self.max_blocks if self.use_tier else 0
        self.reserve_bytes = self.reserve_seqs * max(s.kv_bytes for s in self.seqs) if self.use_tier else 0
        if self.use_tier and self.reserve_blocks >= self.num_blocks:
            raise SimulationError("GPU KV pool too small to stage a prefill for the host tier")

    def _cap_pool_by_hbm(self) -> None:
        """Bound the pool by what HBM really holds: free memory after the
        weights, minus the worker's runtime reserve (re-shard transients,
        prefill activations, workspaces).  Ranks that share a device (the
        virtual ranks of the single-GPU tests) split it; every rank adopts
        the smallest cap so the replica's pools agree."""
        w = self.worker
        if self.device.type != "cuda":
            return
        self.comm.barrier()                      # every rank's weights are allocated
        torch.cuda.synchronize(self.device)
        free, _ = torch.cuda.mem_get_info(self.device)
        free += torch.cuda.memory_reserved(self.device) - torch.cuda.memory_allocated(self.device)
        have = w.pool.numel() * 2 if w.pool is not None else 0
        bus = torch.cuda.get_device_properties(self.device).pci_bus_id
        mine = torch.tensor([float(free), float(have), float(bus)], dtype=torch.float64, device=self.device)
        got = torch.empty(3 * self.comm.size, dtype=torch.float64, device=self.device)
        self.comm.all_gather(got, mine)
        rows = got.view(-1, 3).cpu().tolist()
        caps = []
        for f, _, b in rows:
            same = [r for r in rows if r[2] == b]
            budget = min(r[0] for r in same) + sum(r[1] for r in same)
            caps.append(budget / len(same))
        reserve = w.runtime_reserve_bytes(self.cfg_p, self.cfg_d, self.max_prefill_tokens)
        cap_blocks = int(max(min(caps) - reserve, 0) // self.block_bytes_gpu)
        self.measured["pool_cap_blocks_by_hbm"] = cap_blocks
        self.measured["runtime_reserve_bytes"] = reserve
        if cap_blocks < self.num_blocks:
            if cap_blocks < self.max_blocks:
                raise SimulationError(f"HBM left after the weights and the runtime reserve ({reserve / 2**30:.1f} "
                                      f"GiB) holds {cap_blocks} KV blocks per GPU; the longest request needs "
                                      f"{self.max_blocks}")
            self.num_blocks = cap_blocks

    # ----------------------------------------------------------------- log --
    def _log(self, mark, kind, seq=None, gpu=None, nbytes=None, **extra) -> None:
        self.events.append((mark, kind, dict(seq=seq, gpu=gpu, nbytes=nbytes, extra=extra)))

    def _phase_start(self, phase: str):
        self.phase_index += 1
        t = self.clock.mark()
        self._log(t, "phase_start", phase=phase, index=self.phase_index)
        return t

    def _wait(self, kind: str, fn) -> None:
        """Make the compute stream wait (fn) and record how long it stalled."""
        a = self.clock.mark()
        fn()
        self.stalls.append((kind, a, self.clock.mark()))

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
            self._cap_pool_by_hbm()
        self._plan_tier()
        if w.pool is None or w.num_blocks < self.num_blocks:
            w.pool = None  # release the smaller pool before allocating its successor
            w.alloc_pool(self.num_blocks)
        self.allocs = {r: BlockAllocator(w.num_blocks) for r in range(self.dp)}
        self.alloc = self.allocs[w.replica]
        if self.use_tier:
            self._setup_tier()
        self.pending = {r: [s for s in self.seqs if s.replica == r] for r in range(self.dp)}
        self.running: dict[int, list[_Seq]] = {r: [] for r in range(self.dp)}   # resident, decoding
        self.queues: dict[int, list[_Seq]] = {r: [] for r in range(self.dp)}    # buffered in the host tier
        self.inflight: dict[int, list[_Seq]] = {r: [] for r in range(self.dp)}  # swap-ins under way
        self.gpu_room = {r: self.replica_gpu_capacity for r in range(self.dp)}
        self.batch: list[_Seq] = []                          # this replica's device batch (row order)
        self.d_tables = self.d_ctx = self.d_tokens = None
        self.rows: list[tuple[list[_Seq], torch.Tensor]] = []
        self.step = 0
        self.comm.barrier()
        if self.device.type == "cuda":
            torch.cuda.synchronize(self.device)
        self.clock = _Clock(self.device)
        self._log(self.clock.t0, "run_start", policy=self.policy.value, cfg_p=self.cfg_p.label(),
                  cfg_d=self.cfg_d.label(), requests=len(self.seqs))
        self.phases: list[tuple[str, object, object]] = []
        if self.policy is SchedulingPolicy.PREFILL_PRIORITIZED:
            self._run_prefill_prioritized()
        else:
            # transition-minimizing (native or reference mode) and
            # decode-prioritized (no host tier: static batches, sim.py:644-663)
            self._run_cycles()
        self._collect_tokens()
        t_end = self.clock.mark()
        self._log(t_end, "run_end")
        return self._report(t_end)

    def _any_pending(self) -> bool:
        return any(self.pending[r] for r in range(self.dp))

    def _run_cycles(self) -> None:
        """P-phase -> transition -> D-phase cycles until the workload is done
        (sim.py:618-642 and :644-663)."""
        cycle = 0
        while self._any_pending():
            if cycle > 0:
                self._transition("decode_to_prefill", self.cfg_p, [])
            t_phase = self._phase_start("prefill")
            if self.tm_mode == "reference":
                # prefill steps against the whole GPU tier until the host
                # tier is full or work runs out (sim.py:623-636)
                while True:
                    cpu_room = self.cpu_capacity - self.kv.cpu_used
                    waves = {}
                    for r in range(self.dp):
                        waves[r] = self._pack_reference(r, cpu_room)
                        cpu_room -= sum(s.kv_bytes for s in waves[r])
                    if not any(waves.values()):
                        break
                    self._prefill_phase(waves)
                    if not self._any_pending():
                        break
            else:
                cpu_room = self.cpu_capacity - self.kv.cpu_used
                waves = {}
                for r in range(self.dp):
                    waves[r] = self._pack(r, cpu_room)
                    cpu_room -= sum(s.kv_bytes for s in waves[r] if s.overflow)
                if not any(waves.values()):
                    raise SimulationError("a request that fits the GPU tier must be admissible")
                self._prefill_phase(waves)
            self.phases.append(("prefill", t_phase, self.clock.mark()))
            self._transition("prefill_to_decode", self.cfg_d, self.running[self.worker.replica])
            t_dec = self._phase_start("decode")
            self._decode_phase()
            self.phases.append(("decode", t_dec, self.clock.mark()))
            cycle += 1

    def _run_prefill_prioritized(self) -> None:
        """vLLM-style prefill priority (sim.py:666-695): prefill whatever fits
        the free GPU tier, decode until the next pending request fits, then
        switch back; residents keep decoding across the switches (their KV
        is re-sharded with the layout when cfg_p != cfg_d)."""
        me = self.worker.replica
        while True:
            waves = {r: self._pack(r, 0.0) for r in range(self.dp)}
            if any(waves.values()):
                if self.phase_index > 0:
                    self._transition("decode_to_prefill", self.cfg_p, self.running[me])
                t_phase = self._phase_start("prefill")
                self._prefill_phase(waves)
                self.phases.append(("prefill", t_phase, self.clock.mark()))
            if not any(self.running[r] for r in range(self.dp)) and not self._any_pending():
                return
            self._transition("prefill_to_decode", self.cfg_d, self.running[me])
            t_dec = self._phase_start("decode")

            def room_for_next() -> bool:
                return any(self.pending[r] and self.pending[r][0].kv_bytes <= self.gpu_room[r]
                           and self.pending[r][0].nblocks <= self.allocs[r].available for r in range(self.dp))

            self._decode_phase(stop=room_for_next if self._any_pending() else None)
            self.phases.append(("decode", t_dec, self.clock.mark()))
            if not any(self.running[r] for r in range(self.dp)) and not self._any_pending():
                return

    def _setup_tier(self) -> None:
        from .hosttier import HostTier

        w = self.worker
        per_replica_bytes = self.cpu_capacity / self.dp
        slot_bytes = self.max_prompt * self.kv_tok
        n_slots = int(per_replica_bytes // max(slot_bytes, 1))
        n_slots = max(1, min(n_slots, max(len([s for s in self.seqs if s.replica == r]) for r in range(self.dp))))
        gpus = self.cfg_p.gpus_per_replica
        staging = self.max_prompt * self.kv_tok // gpus
        a = self.arch
        # pinned memory is allocated once per worker and reused by later runs
        # whose slot shape matches and whose slot count it covers; a larger
        # need replaces it (the old buffer is released first: pinned host
        # memory, not HBM, is what runs out at 13B/70B scale)
        shape = (self.max_prompt, staging)
        tier = getattr(w, "_host_tier", None)
        if tier is None or tier.shape_key != shape or tier.n_slots < n_slots:
            w._host_tier = None
            del tier
            import gc

            gc.collect()
            if self.device.type == "cuda":
                torch.cuda.synchronize(self.device)
                torch._C._host_emptyCache()  # return cached pinned blocks to the OS
            tier = HostTier(w.replica_comm, self.device, a.num_layers, a.num_kv_heads, a.head_dim,
                            self.max_prompt, n_slots, staging)
            tier.shape_key = shape
            w._host_tier = tier
        self.tier = tier
        # slot lists of every replica (the real tier is this replica's)
        self.slots = {r: list(range(n_slots)) for r in range(self.dp)}
        # deterministic admission lag (decode steps) for a swap-in: transfer
        # time of one sequence's piece at the host link rate over a nominal
        # 10 ms step, rounded up (identical on every rank)
        piece = self.max_prompt * self.kv_tok / gpus
        lag = max(1, math.ceil(piece / self.hw.host_link_bandwidth / 0.010))
        self.swap_lag = lag if self.swap_lag_override is None else max(0, self.swap_lag_override)

    # ------------------------------------------------------------- pack --
    def _pack(self, r: int, cpu_room: float) -> list[_Seq]:
        """Greedy trace-order admission (sim.py:345-358): GPU-resident while the
        GPU tier (bytes and pool blocks, minus the staging reserve) has room,
        then buffered in the host tier while it has room."""
        room = self.gpu_room[r] - self.reserve_bytes
        blocks = self.allocs[r].available - self.reserve_blocks
        slots = len(self.slots[r]) if self.use_tier else 0
        out = []
        spill = False
        for s in self.pending[r]:
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
        self.pending[r] = self.pending[r][len(out):]
        return out

    def _pack_reference(self, r: int, cpu_room: float) -> list[_Seq]:
        """The reference's prefill-step pack (sim.py:345-358 with
        gpu_room = the whole tier, sim.py:629): greedy while the sequence
        fits the GPU tier's remaining bytes, the host tier's room, the pool
        and the tier's slots; every packed sequence is swapped out."""
        room = self.replica_gpu_capacity
        blocks = self.allocs[r].available
        slots = len(self.slots[r])
        out = []
        for s in self.pending[r]:
            if s.kv_bytes > room or s.kv_bytes > cpu_room or s.nblocks > blocks or slots == 0:
                break
            s.overflow = True
            room -= s.kv_bytes
            cpu_room -= s.kv_bytes
            blocks -= s.nblocks
            slots -= 1
            out.append(s)
        self.pending[r] = self.pending[r][len(out):]
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

    def _prefill_phase(self, waves: dict[int, list[_Seq]]) -> None:
        """One prefill step of every replica's wave: residents stay in HBM;
        overflow sequences go through the reserve and are swapped out to the
        host tier on the copy stream while the next micro-batch computes."""
        w = self.worker
        me = w.replica
        batch = waves[me]
        residents = [s for s in batch if not s.overflow]
        overflow = [s for s in batch if s.overflow]
        first = torch.zeros(max(len(batch), 1), dtype=torch.int32, device=self.device)
        index = {id(s): i for i, s in enumerate(batch)}
        for r in waves:  # every replica's residents take pool blocks (shadow allocators elsewhere)
            for s in waves[r]:
                if not s.overflow:
                    s.blocks = self.allocs[r].alloc(s.nblocks)
                    self.gpu_room[r] -= s.kv_bytes
                else:
                    s.slot = self.slots[r].pop(0)
        for mb in self._micro_batches(residents):
            self._run_prefill(mb, first, index)
        tickets = []
        st = w.state
        glayer0, ghead0 = st.weights.layer_begin, st.rank * st.weights.n_kv_heads
        for mb in self._micro_batches(overflow, limit_seqs=self.reserve_seqs):
            for s in mb:
                s.blocks = self.alloc.alloc(s.nblocks)
            self._run_prefill(mb, first, index)
            geo = w.geometry().as_tuple()
            for s in mb:
                blk = torch.tensor(s.blocks, dtype=torch.int32, device=self.device)
                tk = self.tier.swap_out(w.pool, geo, blk, s.req.input_len, s.slot, glayer0, ghead0, s.req.id)
                tickets.append((s, tk))
                # the gather is stream-ordered before any later prefill writes
                self.alloc.release(s.blocks)
                s.blocks = []
        if tickets:
            # every swap-out lands before the transition (ranks read each
            # other's pieces only after the transition's collectives): the
            # compute stream's wait is the swap-out stall (sim.py:401)
            compute = torch.cuda.current_stream(self.device)
            self._wait("swap_out", lambda: compute.wait_stream(self.tier.copy_stream))
        # every rank of the replica needs the first tokens: only the last
        # stage's tensor rank 0 contributes, the others add zeros
        if not (st.stage == self.cfg_p.pp - 1 and st.rank == 0):
            first.zero_()
        w.replica_comm.all_reduce_(first)
        firsts = first.cpu().numpy() if overflow else None
        for s in residents:
            s.first_dev = first[index[id(s)]].view(1)
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
                self.running[r].append(s)
        tk_by_id = {id(s): tk for s, tk in tickets}
        # reference mode: the whole wave fits the GPU tier, so (as in
        # sim.py:403-429) every completion is logged before the swap-outs;
        # native mode stages overflow through a small reserve, one sequence
        # at a time, and logs each completion next to its swap-out
        batched = self.tm_mode == "reference"
        if batched:
            for r in sorted(waves):
                for s in waves[r]:
                    if s.overflow:
                        self.kv.gpu_used += s.kv_bytes
                        self._log(t_end, "prefill_complete", seq=s.req.id, gpu=r, nbytes=s.kv_bytes,
                                  input_len=s.req.input_len, output_len=s.req.output_len)
        for r in sorted(waves):
            for s in waves[r]:
                if not s.overflow:
                    continue
                mark = t_end if batched else (tk_by_id[id(s)].done if id(s) in tk_by_id else t_end)
                if not batched:
                    self.kv.gpu_used += s.kv_bytes
                    self._log(mark, "prefill_complete", seq=s.req.id, gpu=r, nbytes=s.kv_bytes,
                              input_len=s.req.input_len, output_len=s.req.output_len)
                self.kv.gpu_used -= s.kv_bytes
                self.kv.cpu_used += s.kv_bytes
                self.kv.residency[s.req.id] = Residency.CPU
                self._log(mark, "swap_out_complete", seq=s.req.id, gpu=r, nbytes=s.kv_bytes)
                self.queues[r].append(s)
                self.measured["swapped_out"] += 1

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
        n0 = len(self.worker.logit_log)
        self.worker.prefill(toks, cu, tables, first[i0 : i0 + len(mb)])
        if len(self.worker.logit_log) > n0:
            self.worker.logit_rows.append([s.req.id for s in mb])

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
        self.phases.append(("reshard", t0, t1))
        self._log(t1, "transition", direction=direction)

    # ------------------------------------------------------------- decode --
    def _rebuild(self, new_batch: list[_Seq]) -> None:
        """Device state (tokens, contexts, block tables) of this replica's
        batch: kept rows gathered from the old state (in their old order),
        fresh rows appended from their prefill / swap-in first tokens."""
        dev = self.device
        pos = {id(s): i for i, s in enumerate(self.batch)}
        kept = [s for s in new_batch if id(s) in pos]
        fresh = [s for s in new_batch if id(s) not in pos]
        order = kept + fresh
        tab = np.zeros((len(order), self.max_blocks), dtype=np.int32)
        for i, s in enumerate(order):
            tab[i, : len(s.blocks)] = s.blocks
        parts_ctx, parts_tok = [], []
        if kept:
            idx = torch.tensor([pos[id(s)] for s in kept], dtype=torch.long, device=dev)
            parts_ctx.append(self.d_ctx.index_select(0, idx))
            parts_tok.append(self.d_tokens.index_select(0, idx))
        if fresh:
            parts_ctx.append(torch.tensor([s.req.input_len for s in fresh], dtype=torch.int32, device=dev))
            ft = [s.first_dev if not s.overflow else torch.tensor([s.first_token], dtype=torch.int32, device=dev)
                  for s in fresh]
            parts_tok.append(torch.cat(ft))
            self.rows.append((list(fresh), torch.cat(ft).clone()))
        self.d_tables = torch.from_numpy(tab).to(dev)
        if order:
            self.d_ctx = torch.cat(parts_ctx).contiguous()
            self.d_tokens = torch.cat(parts_tok).contiguous()
        else:
            # this replica drained while others still decode (dp > 1)
            self.d_ctx = torch.zeros(0, dtype=torch.int32, device=dev)
            self.d_tokens = torch.zeros(0, dtype=torch.int32, device=dev)
        self.batch = order

    def _prefetch(self, fill: bool) -> None:
        """FIFO swap-ins while the GPU tier has room (sim.py:441-456); at most
        swap_in_flight per replica unless ``fill`` (nothing resident: start
        every transfer that fits, the reference's wait-for-fill)."""
        if self.tier is None or not any(self.queues[r] for r in range(self.dp)):
            return
        w = self.worker
        me = w.replica
        compute = torch.cuda.current_stream(self.device)
        marker = torch.cuda.Event()
        marker.record(compute)
        self.tier.copy_stream.wait_event(marker)  # freed blocks are no longer read
        st = w.state
        ghead0, glayer0 = st.rank * st.weights.n_kv_heads, st.weights.layer_begin
        for r in range(self.dp):
            q = self.queues[r]
            while (q and (fill or len(self.inflight[r]) < self.swap_in_flight)
                   and self.allocs[r].available >= q[0].nblocks and self.gpu_room[r] >= q[0].kv_bytes):
                s = q.pop(0)
                s.blocks = self.allocs[r].alloc(s.nblocks)
                self.gpu_room[r] -= s.kv_bytes
                s.admit_step = self.step + self.swap_lag
                if r == me:
                    blk = torch.tensor(s.blocks, dtype=torch.int32, device=self.device)
                    s.ticket = self.tier.swap_in(w.pool, w.geometry().as_tuple(), blk, s.req.input_len, s.slot,
                                                 glayer0, ghead0, s.req.id)
                self.kv.cpu_used -= s.kv_bytes
                self.kv.inflight_in += s.kv_bytes
                self.kv.residency[s.req.id] = Residency.IN_TRANSIT
                self._log(self.clock.mark(), "swap_in_start", seq=s.req.id, gpu=r, nbytes=s.kv_bytes)
                self.inflight[r].append(s)

    def _admit(self, fill: bool) -> None:
        """Swap-ins whose lag expired join the batch (all in flight when
        ``fill``); the compute stream waits on each transfer's event — that
        wait is the swap-in stall (sim.py:602)."""
        me = self.worker.replica
        for r in range(self.dp):
            ready = list(self.inflight[r]) if fill else [s for s in self.inflight[r] if s.admit_step <= self.step]
            for s in ready:
                self.inflight[r].remove(s)
                if r == me:
                    compute = torch.cuda.current_stream(self.device)
                    self._wait("swap_in", lambda s=s: compute.wait_event(s.ticket.done))
                self.slots[r].append(s.slot)
                self.slots[r].sort()
                mark = self.clock.mark()
                self.kv.inflight_in -= s.kv_bytes
                self.kv.gpu_used += s.kv_bytes
                self.kv.residency[s.req.id] = Residency.GPU
                self._log(mark, "swap_in_complete", seq=s.req.id, gpu=r, nbytes=s.kv_bytes)
                self.running[r].append(s)

    def _decode_phase(self, stop: Callable[[], bool] | None = None) -> None:
        """Decode rounds until every resident and buffered sequence reached
        output_len (sim.py:517-565, :605-614) — or until ``stop()`` after a
        round (prefill-prioritized).  Under a pipeline layout (pp>1) a round
        is ceil(n/pp) micro-batches, each one decode_step in the log.  All
        replicas' schedules advance in lockstep; only this rank's replica
        runs kernels."""
        w = self.worker
        me = w.replica
        pp = self.cfg_d.pp
        while any(self.running[r] or self.queues[r] or self.inflight[r] for r in range(self.dp)):
            fill = not any(self.running[r] for r in range(self.dp))
            self._prefetch(fill)
            self._admit(fill)
            if not any(self.running[r] for r in range(self.dp)):
                raise SimulationError("prefetcher wedged with work remaining")
            # one round of every replica's residents
            if [id(s) for s in self.running[me]] != [id(s) for s in self.batch]:
                self._rebuild(self.running[me])
                self.running[me] = list(self.batch)
            chunks = {r: ceil_chunks(list(self.running[r]), pp) for r in range(self.dp)}
            if self.batch:
                spans, a = [], 0
                for c in chunks[me]:
                    spans.append((a, a + len(c)))
                    a += len(c)
                nxt = torch.empty_like(self.d_tokens)
                positions = torch.empty_like(self.d_tokens)
                slots = torch.empty(len(self.batch), dtype=torch.int64, device=self.device)
                n0 = len(w.logit_log)
                w.decode_round(self.d_tokens, self.d_ctx, self.d_tables, positions, slots, nxt, spans)
                recorded = len(w.logit_log) - n0
                for k in range(recorded):
                    a, b = spans[k] if recorded == len(spans) else (0, len(self.batch))
                    w.logit_rows.append([s.req.id for s in self.batch[a:b]])
                self.d_tokens = nxt
                self.rows.append((list(self.batch), nxt))
            self.step += 1
            n_steps = max(len(c) for c in chunks.values())
            for i in range(n_steps):
                mark = self.clock.mark()
                for r in range(self.dp):
                    if i >= len(chunks[r]):
                        continue
                    chunk = chunks[r][i]
                    self._log(mark, "decode_step", gpu=r, tokens=len(chunk), seqs=tuple(s.req.id for s in chunk))
                    for s in chunk:
                        s.decoded += 1
                    for s in chunk:
                        if s.decoded == s.req.output_len:
                            self.kv.gpu_used -= s.kv_bytes
                            self.kv.residency[s.req.id] = Residency.RELEASED
                            self._log(mark, "kv_release", seq=s.req.id, gpu=r, nbytes=s.kv_bytes)
                            self.allocs[r].release(s.blocks)
                            self.gpu_room[r] += s.kv_bytes
                            self.running[r].remove(s)
            if stop is not None and stop():
                return

    def _collect_tokens(self) -> None:
        """One device->host read of every generated token of this replica.
        Under a decode pipeline only the last stage computed them: the
        replica sums (the last stage's tensor rank 0 contributes, every other
        rank zeros; the prefill first tokens are replica-wide already and
        enter through the same rank)."""
        if self.comm.size > 1:
            # every rank has issued all of its kernels before this one blocks
            # on a device->host copy: virtual ranks share the process, and a
            # pageable D2H copy can hold the driver while a peer still has to
            # launch the other half of a fused combine's barrier
            self.comm.barrier()
        if not self.rows:
            return
        flat = torch.cat([t for _, t in self.rows])
        st = self.worker.state
        if self.cfg_d.pp > 1:
            if not (st.stage == st.cfg.pp - 1 and st.rank == 0):
                flat = torch.zeros_like(flat)
            self.worker.replica_comm.all_reduce_(flat)
        host = flat.cpu().numpy()
        pos = 0
        for seqs, _ in self.rows:
            for col, s in enumerate(seqs):
                s.generated.append(int(host[pos + col]))
            pos += len(seqs)

    # ------------------------------------------------------------- report --
    def _report(self, t_end) -> SimReport:
        if self.device.type == "cuda":
            torch.cuda.synchronize(self.device)
        self.worker.check_peer_errors()
        clk = self.clock
        makespan = clk.resolve(t_end)
        # max over ranks of the makespan (device-timed)
        mk = torch.tensor([makespan], dtype=torch.float32, device=self.device)
        gathered = torch.empty(self.comm.size, dtype=torch.float32, device=self.device)
        self.comm.all_gather(gathered, mk)
        makespan_all = float(gathered.max().item())
        sums = {"prefill": 0.0, "decode": 0.0, "reshard": 0.0}
        for kind, a, b in self.phases:
            sums[kind] += clk.resolve(b) - clk.resolve(a)
        # stalls: the compute stream waiting on the tier (sim.py:401, :602)
        stall = {"swap_out": 0.0, "swap_in": 0.0}
        for kind, a, b in self.stalls:
            stall[kind] += max(clk.resolve(b) - clk.resolve(a), 0.0)
        stalled = stall["swap_out"] + stall["swap_in"]
        prefill_t = max(sums["prefill"] - stall["swap_out"], 0.0)
        # decode absorbs the host-side gaps between phase marks (microseconds)
        decode_t = max(makespan - prefill_t - sums["reshard"] - stalled, 0.0)
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
            "tm_mode": self.tm_mode,
            "arch": self.arch.name,
            "pool_blocks_per_gpu": self.worker.num_blocks,
            "block_size": self.block_size,
            "host_tier": bool(self.use_tier),
        }
        measured = dict(self.measured)
        measured["transition_wall_s"] = trans
        measured["makespan_max_over_ranks_s"] = makespan_all
        measured["stall_swap_out_s"] = stall["swap_out"]
        measured["stall_swap_in_s"] = stall["swap_in"]
        measured["stall_share_of_makespan"] = stalled / makespan if makespan else 0.0
        measured["phase_span_s"] = dict(sums)
        outputs = {s.req.id: s.generated[: s.req.output_len] for s in self.seqs
                   if s.replica == self.worker.replica}
        return SimReport(
            makespan=makespan,
            requests_per_second=len(self.seqs) / makespan,
            tokens_per_second=out_tokens / makespan,
            prefill_time=prefill_t,
            decode_time=decode_t,
            reshard_time=sums["reshard"],
            stalled_transfer_time=stalled,
            transitions=self.transitions,
            event_log=tuple(events),
            config=config,
            final_kv_state=self.kv,
            outputs=outputs,
            measured=measured,
        )
