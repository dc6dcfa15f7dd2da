"""Re-shard planning: placement, KV routes, weight transfer plans, plus the
per-peer exchange rectangles the B200 re-shard engine executes.

The first half keeps the reference's planning API (same names, dataclasses,
results and errors) — /root/reference/pkg/src/shardsim/reshard.py:
  GpuShard / ShardMap         :23-48     shard_map            :98-122
  TransferPlan                :51-65     weight_reload_plan   :125-148
  KVShardDesc / KVRoute       :68-88     _kv_shards / kv_reshard_route :151-188
  contiguous_runs             :191-201

The second half is new: the reference only *charges* KV movement on the host
link (sim.py:382, :436-488) and models weights as a host reload
(reshard.py:125-148).  Here the KV and weights move GPU-to-GPU over NVLink,
so every GPU needs, for each peer, the (layer range x head range) rectangle it
sends and receives — the pairwise intersections of the reference's swap-out
(cfg_p) and swap-in (cfg_d) descriptors.
"""

from __future__ import annotations

from dataclasses import dataclass

from .specs import ConfigError, HardwareSpec, KVLayout, ModelSpec, ParallelismConfig


@dataclass(frozen=True)
class GpuShard:
    gpu_id: int
    replica_id: int
    layer_begin: int
    layer_end: int
    kv_head_begin: int
    kv_head_end: int
    weight_bytes: int


@dataclass(frozen=True)
class ShardMap:
    cfg: ParallelismConfig
    shards: tuple[GpuShard, ...]

    def replica(self, replica_id: int) -> tuple[GpuShard, ...]:
        return tuple(s for s in self.shards if s.replica_id == replica_id)

    def table(self) -> str:
        rows = ["gpu_id  replica  layers        kv_heads      weight_bytes"]
        for s in self.shards:
            rows.append(
                f"{s.gpu_id:<7d} {s.replica_id:<8d} {f'[{s.layer_begin},{s.layer_end})':<13s} "
                f"{f'[{s.kv_head_begin},{s.kv_head_end})':<13s} {s.weight_bytes}"
            )
        return "\n".join(rows)


@dataclass(frozen=True)
class TransferPlan:
    """Bytes each GPU receives when switching configs and the wall time.

    Reference semantics (reshard.py:51-65): every GPU reloads its whole new
    shard from host memory.  The B200 engine fills ``measured_*`` fields from
    the real NVLink exchange (see execute()).
    """

    bytes_per_gpu: tuple[int, ...]
    wall_time: float
    kv_note: str = "kv re-sharding rides the host-tier swap path; not charged in this plan"

    @property
    def total_bytes(self) -> int:
        return sum(self.bytes_per_gpu)


@dataclass(frozen=True)
class KVShardDesc:
    gpu_id: int
    layer_begin: int
    layer_end: int
    kv_head_begin: int
    kv_head_end: int
    bytes: int


@dataclass(frozen=True)
class KVRoute:
    swap_out: tuple[KVShardDesc, ...]
    swap_in: tuple[KVShardDesc, ...]


def _check_divisible(model: ModelSpec, cfg: ParallelismConfig) -> None:
    if model.num_layers % cfg.pp:
        raise ConfigError(f"pp={cfg.pp} does not divide num_layers={model.num_layers}")
    if model.num_kv_heads % cfg.tp:
        raise ConfigError(f"tp={cfg.tp} does not divide num_kv_heads={model.num_kv_heads}")


def shard_map(model: ModelSpec, cfg: ParallelismConfig) -> ShardMap:
    """Blocked layers per stage, blocked KV heads per rank, GPU ids replica →
    stage → rank; a stage's weight bytes split by divmod with the remainder on
    the low ranks (reshard.py:98-122)."""
    _check_divisible(model, cfg)
    lps = model.num_layers // cfg.pp
    hpr = model.num_kv_heads // cfg.tp
    q, rem = divmod(lps * model.params_per_layer * model.bytes_per_param, cfg.tp)
    shards = tuple(
        GpuShard(
            gpu_id=(rep * cfg.pp + st) * cfg.tp + rk,
            replica_id=rep,
            layer_begin=st * lps,
            layer_end=(st + 1) * lps,
            kv_head_begin=rk * hpr,
            kv_head_end=(rk + 1) * hpr,
            weight_bytes=q + (rk < rem),
        )
        for rep in range(cfg.dp)
        for st in range(cfg.pp)
        for rk in range(cfg.tp)
    )
    return ShardMap(cfg=cfg, shards=shards)


def weight_reload_plan(model: ModelSpec, hw: HardwareSpec, cfg_old: ParallelismConfig,
                       cfg_new: ParallelismConfig) -> TransferPlan:
    """Reference transition cost: max per-GPU new shard / host link (reshard.py:125-148)."""
    if cfg_old.dp != cfg_new.dp:
        raise ConfigError(f"unsupported transition: dp may not change ({cfg_old.dp} -> {cfg_new.dp})")
    _check_divisible(model, cfg_old)
    _check_divisible(model, cfg_new)
    if cfg_old == cfg_new:
        return TransferPlan(bytes_per_gpu=(0,) * cfg_new.num_gpus, wall_time=0.0)
    per_gpu = tuple(s.weight_bytes for s in shard_map(model, cfg_new).shards)
    return TransferPlan(bytes_per_gpu=per_gpu, wall_time=max(per_gpu) / hw.host_link_bandwidth)


def _kv_shards(model: ModelSpec, cfg: ParallelismConfig, seq_len: int) -> tuple[KVShardDesc, ...]:
    cell = 2 * model.bytes_per_param * model.head_dim  # K+V of one (layer, head, token)
    one = ParallelismConfig(cfg.tp, cfg.pp, 1)
    return tuple(
        KVShardDesc(s.gpu_id, s.layer_begin, s.layer_end, s.kv_head_begin, s.kv_head_end,
                    (s.layer_end - s.layer_begin) * (s.kv_head_end - s.kv_head_begin) * seq_len * cell)
        for s in shard_map(model, one).shards
    )


def kv_reshard_route(model: ModelSpec, cfg_p: ParallelismConfig, cfg_d: ParallelismConfig,
                     seq_len: int) -> KVRoute:
    """Swap-out descriptors under cfg_p, swap-in under cfg_d (reshard.py:170-188)."""
    if seq_len < 1:
        raise ValueError("seq_len must be >= 1")
    return KVRoute(swap_out=_kv_shards(model, cfg_p, seq_len), swap_in=_kv_shards(model, cfg_d, seq_len))


def contiguous_runs(layout: KVLayout, seq_len: int, h_kv: int, tp: int) -> int:
    """Contiguous runs per (layer, sequence) shard: HND 1, NHD seq_len if tp>1."""
    if h_kv % tp:
        raise ConfigError(f"tp={tp} does not divide h_kv={h_kv}")
    if layout is KVLayout.HND or tp == 1:
        return 1
    return seq_len


# ---------------------------------------------------------------------------
# B200 additions: per-peer rectangles of the NVLink exchange.
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class Rect:
    """(layer, head) rectangle in the LOCAL coordinates of one GPU's pool."""

    l0: int
    nl: int
    h0: int
    nh: int

    @property
    def cells(self) -> int:
        return self.nl * self.nh


@dataclass(frozen=True)
class PeerExchange:
    """What GPU ``gpu`` (index inside its replica) sends to / receives from
    each peer of the replica when the KV layout switches src → dst.

    send[q]: rectangle of this GPU's src-layout pool destined to peer q.
    recv[q]: rectangle of this GPU's dst-layout pool that arrives from peer q.
    Staging buffers are per-peer contiguous, peers in gpu order.
    """

    gpu: int
    send: tuple[Rect, ...]
    recv: tuple[Rect, ...]


def _ranges(model: ModelSpec, tp: int, pp: int) -> list[tuple[int, int, int, int]]:
    return [(s.layer_begin, s.layer_end, s.kv_head_begin, s.kv_head_end)
            for s in shard_map(model, ParallelismConfig(tp, pp, 1)).shards]


def _intersect(a, b, origin) -> Rect:
    l0, l1 = max(a[0], b[0]), min(a[1], b[1])
    h0, h1 = max(a[2], b[2]), min(a[3], b[3])
    if l1 <= l0 or h1 <= h0:
        return Rect(0, 0, 0, 0)
    return Rect(l0 - origin[0], l1 - l0, h0 - origin[2], h1 - h0)


def kv_exchange(model: ModelSpec, src: ParallelismConfig, dst: ParallelismConfig, gpu: int) -> PeerExchange:
    """Per-peer send/recv rectangles of ``gpu`` for a src → dst KV re-shard.

    Equal dp and full fleet coverage force equal tp*pp (sim.py:241-243), so a
    pool block has the same byte size in both layouts and the re-shard is a
    block-local permutation across the replica's GPUs.
    """
    if src.gpus_per_replica != dst.gpus_per_replica:
        raise ConfigError("re-shard requires equal tp*pp in both layouts")
    a = _ranges(model, src.tp, src.pp)
    b = _ranges(model, dst.tp, dst.pp)
    if not 0 <= gpu < len(a):
        raise ConfigError(f"gpu {gpu} outside the replica of {len(a)} GPUs")
    send = tuple(_intersect(a[gpu], b[q], a[gpu]) for q in range(len(b)))
    recv = tuple(_intersect(a[q], b[gpu], b[gpu]) for q in range(len(a)))
    return PeerExchange(gpu=gpu, send=send, recv=recv)


def kv_exchange_matrix(model: ModelSpec, src: ParallelismConfig, dst: ParallelismConfig,
                       tokens: int) -> list[list[int]]:
    """Bytes [from gpu][to gpu] of ``tokens`` KV tokens crossing the switch."""
    cell = 2 * model.bytes_per_param * model.head_dim * tokens
    n = src.gpus_per_replica
    return [[r.cells * cell for r in kv_exchange(model, src, dst, g).send] for g in range(n)]
