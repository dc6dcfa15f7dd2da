"""Per-GPU worker: owns one GPU's weights, paged KV pool and buffers, and runs
the prefill (PP layout) and decode (TP layout) forwards and the re-shard.

One Worker per rank (process or thread); all ranks run the same SPMD program
and make identical decisions, so no control messages are exchanged — only
data moves (NCCL / ThreadComm).  Every FLOP and every byte of layout
transformation is done by libseesaw_b200.so kernels (ops.py); torch provides
allocation and streams.

What replaces what in the reference (paths under shardsim/):
  prefill micro-batch quantum  sim.py:360-432 / perf.py  -> :meth:`prefill`
  transition weight reload     sim.py:328-333, reshard.py:125-148 -> :meth:`repartition_weights`
  KV re-shard via host tier    sim.py:382, reshard.py:170-188      -> :meth:`reshard_kv`
  decode quantum               sim.py:517-565 / perf.py  -> :meth:`decode_step`
"""

from __future__ import annotations

import math
import struct
from dataclasses import dataclass

import numpy as np
import torch

from . import ops
from .arch import LlamaArch
from .comm import Comm
from .layout import KVPoolGeometry, WeightLayout, kv_geometry, logical_tensors, repartition_pieces, weight_layout
from .reshard import kv_exchange
from .specs import ModelSpec, ParallelismConfig


def rope_tables(arch: LlamaArch, max_pos: int) -> tuple[np.ndarray, np.ndarray]:
    """cos/sin [max_pos, d/2] fp32, computed in float64 on the host so the CPU
    oracle and the GPU use bit-identical tables (rotate-half RoPE)."""
    d = arch.head_dim
    inv = arch.rope_theta ** (-np.arange(0, d, 2, dtype=np.float64) / d)
    ang = np.arange(max_pos, dtype=np.float64)[:, None] * inv[None, :]
    return np.cos(ang).astype(np.float32), np.sin(ang).astype(np.float32)


def init_segment_table(layout: WeightLayout) -> tuple[np.ndarray, int]:
    """int64 [n, 8] rows of ssb_init_seg for every segment of the layout."""
    logical = logical_tensors(layout.arch)
    rows = []
    cum = 0
    for t in layout.tensors.values():
        for s in t.segments:
            lg = logical[s.logical]
            scale_bits = struct.unpack("<i", struct.pack("<f", np.float32(lg.scale)))[0]
            rows.append([
                t.offset + s.dst_row * t.cols + s.dst_col, t.cols, s.row0, s.col0, lg.cols, cum,
                (s.rows & 0xFFFFFFFF) | (s.cols << 32),
                (lg.tensor_id & 0xFFFFFFFF) | ((scale_bits & 0xFFFFFFFF) << 32),
            ])
            cum += s.rows * s.cols
    arr = np.array(rows, dtype=np.uint64).astype(np.int64) if rows else np.zeros((0, 8), np.int64)
    return arr, cum


def _copy_desc_rows(entries: list[tuple[int, int, int, int, int, int]]) -> tuple[np.ndarray, int]:
    """(src_off, dst_off, src_stride, dst_stride, rows, row_bytes) -> int64 [n, 6] with prefix."""
    out = np.zeros((len(entries), 6), dtype=np.int64)
    cum = 0
    for i, (so, do, ss, ds, rows, rb) in enumerate(entries):
        out[i] = (so, do, ss, ds, cum, (rows & 0xFFFFFFFF) | (rb << 32))
        cum += rows * rb
    return out, cum


def runtime_reserve(arch: LlamaArch, gpu: int, cfg_p: ParallelismConfig, cfg_d: ParallelismConfig,
                    max_prefill_tokens: int, block_size: int = 64, ws_bytes: int = 64 << 20,
                    chunk_bytes: int = 256 << 20) -> dict:
    """Bytes one GPU needs beyond its weights and its KV pool at the peak of
    a run, by component:
      * weight_transient: a weight re-partition holds the new arena next to
        the old one, plus two chunk buffers each way (SSB_RESHARD_CHUNK_MB);
        the KV re-shard stages 256 blocks of its rectangles twice each way
        (the larger of the two; they do not overlap);
      * activations: a max_prefill_tokens forward (h, x, qkv, attention out,
        gate/up product, row sums) and the fp32 logits of its last rows
        (decode buffers are smaller);
      * workspaces: two GEMM split-K / stream-K workspaces, the fused-TP peer
        arena and host-tier staging;
      * slack: 2 GiB for the allocator."""
    a = arch
    mx = 0
    cfgs = {cfg_p, cfg_d}
    if len(cfgs) > 1:
        new = max(weight_layout(a, c.tp, c.pp, gpu).arena_elems for c in cfgs) * 2
        mx = new + 4 * chunk_bytes
        blk = max(kv_geometry(a, c.tp, c.pp, 1, block_size).block_elems for c in cfgs) * 2
        mx = max(mx, 4 * 256 * blk)
    T = max_prefill_tokens
    tp = min(c.tp for c in cfgs)
    act = T * (2 * a.hidden + a.qkv_dim // tp + a.num_query_heads * a.head_dim // tp + a.ffn // tp) * 2
    act += 2 * T * (-(-a.hidden // 64)) * 4 + 2 * T * 4 * (a.vocab // tp) // max(T // 512, 1)
    ws = 2 * ws_bytes + 3 * T * a.hidden * 2
    slack = 2 << 30
    return {"weight_transient": int(mx), "activations": int(act), "workspaces": int(ws), "slack": slack,
            "total": int(mx + act + ws + slack)}


@dataclass
class LayoutState:
    cfg: ParallelismConfig
    gpu: int                 # index inside the replica
    stage: int
    rank: int                # tensor rank
    weights: WeightLayout
    arena: torch.Tensor
    tp_comm: Comm
    pp_prev: int | None      # replica-group index of the previous stage peer
    pp_next: int | None


class Worker:
    """One GPU of the fleet (SPMD)."""

    GEMM_WS_BYTES = 64 << 20
    RESHARD_CHUNK_BYTES = int(__import__("os").environ.get("SSB_RESHARD_CHUNK_MB", "256")) << 20

    def __init__(self, arch: LlamaArch, world: Comm, dp: int, device: torch.device, seed: int = 0,
                 block_size: int = 64, max_pos: int = 4096) -> None:
        self.arch = arch
        self.world = world
        self.device = device
        self.seed = seed
        self.block_size = block_size
        self.dp = dp
        self.per_replica = world.size // dp
        self.replica, self.gpu = divmod(world.rank, self.per_replica)
        self.replica_comm = world.subgroup([self.replica * self.per_replica + i for i in range(self.per_replica)])
        cos, sin = rope_tables(arch, max_pos)
        self.rope_cos = torch.from_numpy(cos).to(device)
        self.rope_sin = torch.from_numpy(sin).to(device)
        self.state: LayoutState | None = None
        self.pool: torch.Tensor | None = None
        self.num_blocks = 0
        self.scale = 1.0 / math.sqrt(arch.head_dim)
        self._comm_cache: dict = {}
        self._wplans: dict = {}
        self.stream = torch.cuda.current_stream(device) if device.type == "cuda" else None
        self.record_logits = False
        self.logit_log: list[torch.Tensor] = []
        self.logit_rows: list[list] = []  # request ids of each recorded forward's rows (set by the engine)
        self.stats: dict[str, float] = {}
        # test/inspection callbacks invoked by the engine: name -> fn(worker, **kw)
        self.hooks: dict = {}
        self._bufs: dict = {}
        self._side = None
        # decode overlap: two half-batch lanes on two streams; GEMM grid cap
        import os

        # measured on B200 (tools/bench_decode.py, 8B, B=512): two lanes are
        # ~3% SLOWER than one (the second weight read outweighs the overlap),
        # so the overlap is off by default
        self.decode_lanes = int(os.environ.get("SSB_DECODE_LANES", "1"))
        self.lane_gemm_cap = int(os.environ.get("SSB_LANE_GEMM_CAP", "0"))
        self.min_lane_rows = int(os.environ.get("SSB_MIN_LANE_ROWS", "64"))
        # RoPE + K/V append in the QKV GEMM epilogue (head_dim 128)
        self.fuse_rope = os.environ.get("SSB_FUSE_ROPE", "1") != "0"
        # greedy argmax in the LM-head GEMM epilogue
        self.fuse_argmax = os.environ.get("SSB_FUSE_ARGMAX", "1") != "0"
        # split-K for skinny projections (a workspace per lane)
        self.split_k = os.environ.get("SSB_SPLIT_K", "1") != "0"
        # KV re-shard with the transfer fused into the pack (peer memory)
        self.p2p_reshard = os.environ.get("SSB_RESHARD_P2P", "0") == "1"
        # TP combine (all-reduce of the row-parallel partials + the rmsnorm
        # after it) as one kernel over NVLink peer memory (tpcombine.py).
        # None = automatic: on for NCCL process groups; ThreadComm ranks need
        # one CUDA stream per thread for its device-side barrier, so tests
        # opt in.  SSB_TP_FUSED=0/1 forces it.
        env = os.environ.get("SSB_TP_FUSED")
        self.fused_tp: bool | None = None if env is None else env == "1"
        self.fused_tp_blocks = int(os.environ.get("SSB_TP_FUSED_BLOCKS", "0"))
        self._tp_arenas: dict = {}
        # RMSNorm folded into the GEMMs (single-GPU layout): the residual
        # GEMMs emit row sums of squares, the consumers scale rows by 1/rms,
        # the gains live in the consumer weights (fold_gains)
        self.fold_norm = os.environ.get("SSB_FOLD_NORM", "1") != "0"
        # TP decode with the folded norm: the combine broadcasts x plus one
        # fp32 row sum of squares instead of x and h (half the NVLink stores)
        self.tp_fold = os.environ.get("SSB_TP_FOLD", "1") != "0"
        # decode steps replayed from CUDA graphs (per batch size)
        self.cuda_graphs = os.environ.get("SSB_CUDA_GRAPH", "1") != "0"
        self._graphs: dict = {}
        self._graph_pool = None

    # ------------------------------------------------------------ layouts --
    def _tp_comm(self, cfg: ParallelismConfig, stage: int) -> Comm:
        key = ("tp", cfg.tp, cfg.pp)
        if key not in self._comm_cache:
            # every rank of the replica creates every stage's group (same order)
            groups = [self.replica_comm.subgroup([s * cfg.tp + r for r in range(cfg.tp)]) for s in range(cfg.pp)]
            self._comm_cache[key] = groups
        return self._comm_cache[key][stage]

    def make_layout(self, cfg: ParallelismConfig, arena: torch.Tensor | None = None) -> LayoutState:
        stage, rank = divmod(self.gpu, cfg.tp)
        wl = weight_layout(self.arch, cfg.tp, cfg.pp, self.gpu)
        if arena is None:
            arena = torch.empty(wl.arena_elems, dtype=torch.bfloat16, device=self.device)
        prev_ = (stage - 1) * cfg.tp + rank if stage > 0 else None
        next_ = (stage + 1) * cfg.tp + rank if stage < cfg.pp - 1 else None
        return LayoutState(cfg, self.gpu, stage, rank, wl, arena, self._tp_comm(cfg, stage), prev_, next_)

    def init_weights(self, cfg: ParallelismConfig) -> None:
        """Generate this GPU's shard of the random-init model under ``cfg``."""
        st = self.make_layout(cfg)
        table, total = init_segment_table(st.weights)
        segs = torch.from_numpy(table).to(self.device)
        ops.init_weights(st.arena, segs, total, self.seed)
        self.state = st
        if self.fold_norm:
            self.fold_gains()

    def fold_gains(self) -> None:
        """Fold every RMSNorm gain into the weights that consume the normed
        activations (W[:, k] *= gamma[k]: attn_norm -> wqkv, mlp_norm -> w13,
        final_norm -> head) and set the gains to 1 — the same model, whose
        norms are then pure 1/rms row scales that the GEMM epilogues apply
        (ssb_rownorm).  A no-op for unit gains (the synthetic init's)."""
        pairs = [(f"L{l}.attn_norm", f"L{l}.wqkv") for l in self._layers()]
        pairs += [(f"L{l}.mlp_norm", f"L{l}.w13") for l in self._layers()]
        pairs.append(("final_norm", "head"))
        for g_key, w_key in pairs:
            if not (self.has(g_key) and self.has(w_key)):
                continue
            g = self.w(g_key)
            if bool(torch.all(g == 1)):
                continue
            self.w(w_key).mul_(g.view(1, -1))
            g.fill_(1)

    def w(self, key: str) -> torch.Tensor:
        t = self.state.weights.tensors[key]
        return self.state.arena[t.offset : t.offset + t.numel].view(t.rows, t.cols)

    def has(self, key: str) -> bool:
        return key in self.state.weights.tensors

    # --------------------------------------------------------------- pool --
    def geometry(self, cfg: ParallelismConfig | None = None) -> KVPoolGeometry:
        cfg = cfg or self.state.cfg
        return kv_geometry(self.arch, cfg.tp, cfg.pp, self.num_blocks, self.block_size)

    def alloc_pool(self, num_blocks: int) -> None:
        """One allocation serves every layout: a block has the same byte size
        under any (tp, pp) with the same tp*pp."""
        self.num_blocks = num_blocks
        self._drop_graphs()
        geo = self.geometry()
        # zero-filled once: decode attention multiplies the (masked, p = 0)
        # tail of a sequence's last block by its V rows, and never-written
        # memory may hold NaN bit patterns (0 * NaN = NaN).  Afterwards a block
        # only ever holds finite KV of some sequence.
        self.pool = torch.zeros(num_blocks * geo.block_elems, dtype=torch.bfloat16, device=self.device)

    # ------------------------------------------------------- re-partition --
    def _weight_plan(self, cfg_old: ParallelismConfig, cfg_new: ParallelismConfig):
        """(pieces[p][q], chunks): what replica GPU p sends to GPU q, and the
        number of chunks the re-partition streams in — identical on every
        rank (computed from all layouts), cached per transition."""
        key = (cfg_old, cfg_new)
        plan = self._wplans.get(key)
        if plan is None:
            n = self.per_replica
            old = [weight_layout(self.arch, cfg_old.tp, cfg_old.pp, g) for g in range(n)]
            new = [weight_layout(self.arch, cfg_new.tp, cfg_new.pp, g) for g in range(n)]
            pieces = [[repartition_pieces(old[p], new[q]) for q in range(n)] for p in range(n)]
            moved = [sum(pc.numel for q in range(n) if q != p for pc in pieces[p][q]) for p in range(n)]
            moved += [sum(pc.numel for p in range(n) if p != q for pc in pieces[p][q]) for q in range(n)]
            chunks = max(1, math.ceil(2 * max(moved) / self.RESHARD_CHUNK_BYTES))
            plan = self._wplans[key] = (pieces, chunks)
        return plan

    def repartition_weights(self, cfg_new: ParallelismConfig) -> int:
        """Weight column/row re-partition over the replica group; returns the
        bytes this GPU sent to other GPUs.

        Streamed in chunks every rank agrees on (the k-th row range of every
        piece): per chunk, copy2d packs the pieces for every peer into a send
        buffer, an all-to-all moves them, copy2d unpacks into the new arena;
        the pack of chunk k+1 overlaps the all-to-all of chunk k.  Pieces this
        GPU keeps are one direct copy.  Peak HBM: old arena + new arena + two
        chunk buffers each way (SSB_RESHARD_CHUNK_MB, 256 MiB) — never a full
        send or receive copy of the shard."""
        old = self.state
        self._drop_graphs()
        pieces, K = self._weight_plan(old.cfg, cfg_new)
        new = self.make_layout(cfg_new)
        me, n = self.gpu, self.per_replica
        keep = pieces[me][me]
        if keep:
            d, tot = _copy_desc_rows([(pc.src_off * 2, pc.dst_off * 2, pc.src_ld * 2, pc.dst_ld * 2, pc.rows,
                                       pc.cols * 2) for pc in keep])
            ops.copy2d_batched(old.arena, new.arena, torch.from_numpy(d).to(self.device), tot)
        sent = 2 * sum(pc.numel for q in range(n) if q != me for pc in pieces[me][q])
        if n > 1 and sent + sum(pc.numel for p in range(n) if p != me for pc in pieces[p][me]):
            if self.p2p_reshard and self.device.type == "cuda":
                self._repartition_p2p(old, new, pieces, K)
            else:
                self._repartition_a2a(old, new, pieces, K)
        self.state = new
        return sent

    def _weight_chunk(self, pieces, k: int, K: int):
        """Send / receive copy descriptors and splits of chunk k (elements)."""
        me, n = self.gpu, self.per_replica
        send, recv, s_splits, r_splits = [], [], [], []
        s_pos = r_pos = 0
        for q in range(n):
            start = s_pos
            for pc in (pieces[me][q] if q != me else ()):
                sl = pc.row_slice(k, K)
                if sl is not None:
                    send.append((sl.src_off * 2, s_pos * 2, sl.src_ld * 2, sl.cols * 2, sl.rows, sl.cols * 2))
                    s_pos += sl.numel
            s_splits.append(s_pos - start)
            start = r_pos
            for pc in (pieces[q][me] if q != me else ()):
                sl = pc.row_slice(k, K)
                if sl is not None:
                    recv.append((r_pos * 2, sl.dst_off * 2, sl.cols * 2, sl.dst_ld * 2, sl.rows, sl.cols * 2))
                    r_pos += sl.numel
            r_splits.append(r_pos - start)
        return send, recv, s_splits, r_splits

    def _repartition_a2a(self, old: LayoutState, new: LayoutState, pieces, K: int) -> None:
        chunks = []
        for k in range(K):
            send, recv, s_splits, r_splits = self._weight_chunk(pieces, k, K)
            sd, stot = _copy_desc_rows(send)
            rd, rtot = _copy_desc_rows(recv)
            chunks.append((torch.from_numpy(sd).to(self.device), stot, s_splits,
                           torch.from_numpy(rd).to(self.device), rtot, r_splits))
        cap_s = max(max(sum(c[2]) for c in chunks), 8)
        cap_r = max(max(sum(c[5]) for c in chunks), 8)
        cuda = self.device.type == "cuda"
        nbuf = 2 if cuda and K > 1 else 1
        sends = [torch.empty(cap_s, dtype=torch.bfloat16, device=self.device) for _ in range(nbuf)]
        recvs = [torch.empty(cap_r, dtype=torch.bfloat16, device=self.device) for _ in range(nbuf)]

        def pack(k):
            sd, stot, _, _, _, _ = chunks[k]
            if stot:
                ops.copy2d_batched(old.arena, sends[k % nbuf], sd, stot)

        def unpack(k):
            _, _, _, rd, rtot, _ = chunks[k]
            if rtot:
                ops.copy2d_batched(recvs[k % nbuf], new.arena, rd, rtot)

        if not cuda or nbuf == 1:
            for k in range(K):
                pack(k)
                _, _, s_splits, _, _, r_splits = chunks[k]
                self.replica_comm.all_to_all(recvs[0], sends[0], r_splits, s_splits)
                unpack(k)
            return
        main = torch.cuda.current_stream(self.device)
        cs = self._comm_stream_()
        arrived: list = [None] * K
        free = [None] * nbuf  # event: the chunk that last used buffer b was unpacked

        def launch(k):
            b = k % nbuf
            if free[b] is not None:
                main.wait_event(free[b])
            pack(k)
            packed = torch.cuda.Event()
            packed.record(main)
            with torch.cuda.stream(cs):
                cs.wait_event(packed)
                _, _, s_splits, _, _, r_splits = chunks[k]
                self.replica_comm.all_to_all(recvs[b], sends[b], r_splits, s_splits)
                arrived[k] = torch.cuda.Event()
                arrived[k].record(cs)

        launch(0)
        for k in range(K):
            if k + 1 < K:
                launch(k + 1)
            main.wait_event(arrived[k])
            unpack(k)
            free[k % nbuf] = torch.cuda.Event()
            free[k % nbuf].record(main)
        for b in range(nbuf):
            sends[b].record_stream(cs)
            recvs[b].record_stream(cs)

    def _comm_stream_(self) -> torch.cuda.Stream:
        if getattr(self, "_comm_stream", None) is None:
            self._comm_stream = torch.cuda.Stream(self.device)
        return self._comm_stream

    def _p2p_buffer(self, elems: int):
        """This rank's peer-mapped receive buffer (>= elems bf16) and every
        peer's address of it; one allocation reused by every P2P re-shard and
        grown collectively (the size is identical on all ranks)."""
        buf = getattr(self, "_p2p", None)
        if buf is None or buf[0].numel() < elems:
            self._p2p = None  # release the old buffer and its peer mappings first
            t = torch.empty(elems, dtype=torch.bfloat16, device=self.device)
            maps: list = []
            self._p2p = (t, self.replica_comm.peer_addresses(t, maps), maps)
        return self._p2p[0], self._p2p[1]

    def _repartition_p2p(self, old: LayoutState, new: LayoutState, pieces, K: int) -> None:
        """Pack + transfer in one kernel per chunk: every piece is stored
        straight into its owner's receive buffer (IPC peer memory), at the
        section that follows the sections of the ranks before this one."""
        me, n = self.gpu, self.per_replica
        per_chunk = []
        cap = 8
        for k in range(K):
            # elements p sends q in chunk k, for every pair (the receivers' layout)
            sizes = [[sum(sl.numel for pc in pieces[p][q] if p != q for sl in [pc.row_slice(k, K)] if sl)
                      for q in range(n)] for p in range(n)]
            cap = max(cap, max(sum(sizes[p][q] for p in range(n)) for q in range(n)))
            per_chunk.append(sizes)
        recv, addrs = self._p2p_buffer(cap)
        stream = torch.cuda.current_stream(self.device)
        for k in range(K):
            sizes = per_chunk[k]
            entries = []
            for q in range(n):
                if q == me:
                    continue
                base = sum(sizes[p][q] for p in range(me))
                for pc in pieces[me][q]:
                    sl = pc.row_slice(k, K)
                    if sl is not None:
                        entries.append((sl.src_off * 2, addrs[q] + base * 2, sl.src_ld * 2, sl.cols * 2, sl.rows,
                                        sl.cols * 2))
                        base += sl.numel
            _, recv_e, _, _ = self._weight_chunk(pieces, k, K)
            stream.synchronize()
            self.replica_comm.barrier()  # every receive buffer is idle (previous chunk unpacked)
            if entries:
                pd, ptot = _copy_desc_rows(entries)
                ops.copy2d_batched(old.arena, None, torch.from_numpy(pd).to(self.device), ptot)
            stream.synchronize()
            self.replica_comm.barrier()  # every piece of chunk k landed
            if recv_e:
                rd, rtot = _copy_desc_rows(recv_e)
                ops.copy2d_batched(recv, new.arena, torch.from_numpy(rd).to(self.device), rtot)

    # ---------------------------------------------------------- KV reshard --
    def reshard_kv(self, cfg_new: ParallelismConfig, block_ids: np.ndarray, chunk_blocks: int = 256) -> int:
        """In-place KV re-layout of the listed pool blocks from the current
        layout to ``cfg_new`` (pack -> all-to-all -> unpack per chunk).
        Returns the bytes this GPU sent to other GPUs."""
        model = self.arch.model_spec()
        src_cfg = ParallelismConfig(self.state.cfg.tp, self.state.cfg.pp, 1)
        dst_cfg = ParallelismConfig(cfg_new.tp, cfg_new.pp, 1)
        ex = kv_exchange(model, src_cfg, dst_cfg, self.gpu)
        geo_s = kv_geometry(self.arch, src_cfg.tp, src_cfg.pp, self.num_blocks, self.block_size)
        geo_d = kv_geometry(self.arch, dst_cfg.tp, dst_cfg.pp, self.num_blocks, self.block_size)
        cell = 2 * self.block_size * self.arch.head_dim  # elements of one (layer, head) per block
        sent = 0
        ids_all = np.asarray(block_ids, dtype=np.int32)
        if ids_all.size == 0:
            return 0
        if self.p2p_reshard and self.device.type == "cuda" and self.per_replica > 1:
            return self._reshard_kv_p2p(model, src_cfg, dst_cfg, geo_s, geo_d, ids_all, chunk_blocks, cell)
        max_cells_s = sum(r.cells for r in ex.send)
        max_cells_r = sum(r.cells for r in ex.recv)
        chunk = min(chunk_blocks, ids_all.size)
        nbuf = 2 if self.device.type == "cuda" else 1
        sends = [torch.empty(chunk * max_cells_s * cell + 8, dtype=torch.bfloat16, device=self.device)
                 for _ in range(nbuf)]
        recvs = [torch.empty(chunk * max_cells_r * cell + 8, dtype=torch.bfloat16, device=self.device)
                 for _ in range(nbuf)]

        def plan(c0):
            ids_np = ids_all[c0 : c0 + chunk]
            nid = ids_np.size
            s_peers, r_peers, s_splits, r_splits = [], [], [], []
            so = ro = 0
            for q in range(self.per_replica):
                rs, rr = ex.send[q], ex.recv[q]
                s_peers.append((rs.l0, rs.nl, rs.h0, rs.nh, so * 2))
                r_peers.append((rr.l0, rr.nl, rr.h0, rr.nh, ro * 2))
                s_splits.append(nid * rs.cells * cell)
                r_splits.append(nid * rr.cells * cell)
                so += s_splits[-1]
                ro += r_splits[-1]
            return torch.from_numpy(ids_np).to(self.device), s_peers, r_peers, s_splits, r_splits, so

        chunks = [plan(c0) for c0 in range(0, ids_all.size, chunk)]
        for _, _, _, s_splits, _, so in chunks:
            sent += 2 * (so - s_splits[self.gpu])
        if nbuf == 1:  # host (gloo) path: strictly sequential
            for ids, s_peers, r_peers, s_splits, r_splits, _ in chunks:
                ops.kv_reshard_pack(self.pool, geo_s.as_tuple(), ids, s_peers, sends[0])
                self.replica_comm.all_to_all(recvs[0], sends[0], r_splits, s_splits)
                ops.kv_reshard_unpack(self.pool, geo_d.as_tuple(), ids, r_peers, recvs[0])
            return sent
        # software pipeline over chunks: pack(i+1) on the compute stream and
        # all-to-all(i) on the comm stream overlap; unpack(i) waits for its
        # transfer.  Chunks are disjoint block sets, so packing chunk i+1 from
        # the old layout while unpacking chunk i into the new one is safe.
        main = torch.cuda.current_stream(self.device)
        cs = self._comm_stream_()
        arrived: list = [None] * len(chunks)

        def launch(i):
            ids, s_peers, _, s_splits, r_splits, _ = chunks[i]
            b = i % nbuf
            ops.kv_reshard_pack(self.pool, geo_s.as_tuple(), ids, s_peers, sends[b])
            packed = torch.cuda.Event()
            packed.record(main)
            with torch.cuda.stream(cs):
                cs.wait_event(packed)
                self.replica_comm.all_to_all(recvs[b], sends[b], r_splits, s_splits)
                arrived[i] = torch.cuda.Event()
                arrived[i].record(cs)

        launch(0)
        for i in range(len(chunks)):
            if i + 1 < len(chunks):
                launch(i + 1)
            ids, _, r_peers, _, _, _ = chunks[i]
            main.wait_event(arrived[i])
            ops.kv_reshard_unpack(self.pool, geo_d.as_tuple(), ids, r_peers, recvs[i % nbuf])
        return sent

    def _reshard_kv_p2p(self, model, src_cfg, dst_cfg, geo_s, geo_d, ids_all, chunk_blocks, cell) -> int:
        """KV re-shard with the transfer fused into the pack: every rank's
        pack kernel stores each peer's rectangles straight into that peer's
        receive buffer (CUDA IPC peer memory over NVLink), then each rank
        unpacks its own buffer.  Per chunk: barrier (peers finished unpacking
        the previous chunk) -> pack_p2p -> barrier (all stores landed) ->
        unpack.  No send staging, no NCCL.  (SSB_RESHARD_P2P=1; not the
        default until measured on NVLink.)"""
        P, me = self.per_replica, self.gpu
        ex = [kv_exchange(model, src_cfg, dst_cfg, g) for g in range(P)]
        chunk = min(chunk_blocks, ids_all.size)
        # identical on every rank: the buffer every rank allocates and maps
        recv_cells = max(sum(r.cells for r in e.recv) for e in ex)
        recv, addrs = self._p2p_buffer(chunk_blocks * recv_cells * cell + 8)
        stream = torch.cuda.current_stream(self.device)
        sent = 0
        for c0 in range(0, ids_all.size, chunk):
            ids_np = ids_all[c0 : c0 + chunk]
            nid = int(ids_np.size)
            ids = torch.from_numpy(ids_np).to(self.device)
            peers = []
            for q in range(P):
                rs = ex[me].send[q]
                # my section in q's buffer follows the sections of ranks < me
                off = 2 * sum(nid * ex[p].send[q].cells * cell for p in range(me))
                peers.append((rs.l0, rs.nl, rs.h0, rs.nh, addrs[q] + off))
                if q != me:
                    sent += 2 * nid * rs.cells * cell
            stream.synchronize()
            self.replica_comm.barrier()  # every peer finished reading its buffer
            ops.kv_reshard_pack_p2p(self.pool, geo_s.as_tuple(), ids, peers)
            stream.synchronize()
            self.replica_comm.barrier()  # every rank's stores into my buffer landed
            r_peers, roff = [], 0
            for p in range(P):
                rr = ex[me].recv[p]
                r_peers.append((rr.l0, rr.nl, rr.h0, rr.nh, 2 * roff))
                roff += nid * rr.cells * cell
            ops.kv_reshard_unpack(self.pool, geo_d.as_tuple(), ids, r_peers, recv)
        return sent

    # ------------------------------------------------------------- forward --
    def _layers(self) -> range:
        wl = self.state.weights
        return range(wl.layer_begin, wl.layer_end)

    def _arena(self, rows: int):
        """The fused TP combine's peer arena for this layout (None: use the
        all-reduce + rmsnorm path).  Collective over the TP group."""
        st = self.state
        tp = st.tp_comm
        if tp.size == 1 or self.device.type != "cuda" or rows == 0:
            return None
        use = self.fused_tp
        if use is None:
            from .comm import TorchComm

            use = isinstance(tp, TorchComm) and not tp._host_staged
        if not use:
            return None
        from . import tpcombine
        from .comm import ThreadComm

        if isinstance(tp, ThreadComm):
            # virtual ranks share the GPU: a rank's GEMM launched early by
            # programmatic dependent launch would hold SMs (waiting on its own
            # combine) that a peer's producer needs to reach the same barrier
            ops.set_pdl(False)
        blocks = self.fused_tp_blocks or (
            16 if isinstance(tp, ThreadComm) else torch.cuda.get_device_properties(self.device).multi_processor_count)
        return tpcombine.get_arena(self._tp_arenas, tp, self.device, self.arch.hidden, rows, blocks)

    def _next_gamma(self, layer: int, final: bool):
        """The norm gain the combine after ``layer``'s MLP applies: the next
        layer's attn_norm on this stage, else final_norm when ``final``."""
        if layer + 1 < self.state.weights.layer_end:
            return self.w(f"L{layer + 1}.attn_norm")
        return self.w("final_norm") if final else None

    def _block(self, x: torch.Tensor, layer: int, attn_fn, buf: dict, rope: tuple, cap: int = 0, ar=None,
               h_ready: bool = False, final: bool = False, fold: bool = False) -> bool:
        """One transformer layer on x (in place); attn_fn(qkv, layer_local) -> attn out.
        ``rope`` = (positions, slots) of the rows: RoPE and the paged K/V
        append run in the QKV GEMM's epilogue (head_dim 128) or as a separate
        kernel.  ``cap`` bounds the GEMMs' persistent grid (decode lane overlap).

        With a peer arena ``ar`` (TP > 1, x = ar.x[:T]) the row-parallel
        projections write their partials to ar.part and each combine also
        produces the NEXT rmsnorm (ar.h): ``h_ready`` says this layer's input
        norm is already in ar.h; returns whether the next one is (the
        combine after the MLP applies the next layer's attn_norm, or
        final_norm on the last layer when ``final``).  ``fold`` (decode
        under a pure TP layout): the combines produce x and its row sums of
        squares (ar.ss) instead of h, and the consumer GEMMs apply 1/rms."""
        if ar is not None:
            if fold:
                return self._block_fused_folded(x, layer, attn_fn, buf, rope, cap, ar, h_ready)
            return self._block_fused(x, layer, attn_fn, buf, rope, cap, ar, h_ready, final)
        st = self.state
        if self.fold_norm and st.tp_comm.size == 1:
            return self._block_folded(x, layer, attn_fn, buf, rope, cap, int(h_ready))
        eps = self.arch.rms_eps
        p = f"L{layer}."
        lead = st.rank == 0
        ws = buf["ws"]
        local = layer - st.weights.layer_begin
        nq, nk = st.weights.n_q_heads, st.weights.n_kv_heads
        pos, slots = rope
        geo = self.geometry().as_tuple()
        h = ops.rmsnorm(x, self.w(p + "attn_norm"), eps, out=buf["h"])
        if self.fuse_rope and self.arch.head_dim == 128:
            qkv = ops.gemm_qkv_rope_kv(h, self.w(p + "wqkv"), buf["qkv"], nq, nk, pos, self.rope_cos, self.rope_sin,
                                       self.pool, geo, local, slots, max_ctas=cap, workspace=ws)
        else:
            qkv = ops.gemm(h, self.w(p + "wqkv"), out=buf["qkv"], max_ctas=cap, workspace=ws)
            ops.rope_kv_append(qkv, nq, nk, pos, self.rope_cos, self.rope_sin, self.pool, geo, local, slots)
        attn = attn_fn(qkv, local)
        ops.gemm(attn, self.w(p + "wo"), out=x, residual=x if lead else None, max_ctas=cap, workspace=ws)
        self._reduce_into(x)
        h = ops.rmsnorm(x, self.w(p + "mlp_norm"), eps, out=buf["h"])
        act = ops.gemm(h, self.w(p + "w13"), out=buf["act"], silu_mul=True, max_ctas=cap, workspace=ws)
        ops.gemm(act, self.w(p + "w2"), out=x, residual=x if lead else None, max_ctas=cap, workspace=ws)
        self._reduce_into(x)
        return False

    def _block_folded(self, x, layer, attn_fn, buf, rope, cap, ss_parts: int) -> int:
        """Single-GPU layer with both RMSNorms folded into the GEMMs: the
        o_proj / down_proj residual epilogues write per-tile row sums of
        squares of the new x, the QKV and gate/up GEMMs read x itself and
        scale their rows by 1/rms (gains folded into their weights).
        ``ss_parts`` > 0: buf["ss"][1] holds the previous down_proj's sums
        (else this layer's input norm runs as a kernel).  Returns the parts
        count of this layer's down_proj sums."""
        st = self.state
        eps = self.arch.rms_eps
        hid = self.arch.hidden
        p = f"L{layer}."
        ws = buf["ws"]
        local = layer - st.weights.layer_begin
        nq, nk = st.weights.n_q_heads, st.weights.n_kv_heads
        pos, slots = rope
        geo = self.geometry().as_tuple()
        T = x.shape[0]
        ss_a, ss_b = buf["ss"]
        if ss_parts:
            a_in = x
            rn = ops.row_norm(ss_in=ss_b[: T * ss_parts].view(T, ss_parts), ss_in_parts=ss_parts, hidden=hid, eps=eps)
        else:
            a_in = ops.rmsnorm(x, self.w(p + "attn_norm"), eps, out=buf["h"])
            rn = None
        if self.fuse_rope and self.arch.head_dim == 128:
            qkv = ops.gemm_qkv_rope_kv(a_in, self.w(p + "wqkv"), buf["qkv"], nq, nk, pos, self.rope_cos,
                                       self.rope_sin, self.pool, geo, local, slots, max_ctas=cap, workspace=ws,
                                       rownorm=rn)
        else:
            qkv = ops.gemm(a_in, self.w(p + "wqkv"), out=buf["qkv"], max_ctas=cap, workspace=ws, rownorm=rn)
            ops.rope_kv_append(qkv, nq, nk, pos, self.rope_cos, self.rope_sin, self.pool, geo, local, slots)
        attn = attn_fn(qkv, local)
        rn_o = ops.row_norm(ss_out=ss_a)
        ops.gemm(attn, self.w(p + "wo"), out=x, residual=x, max_ctas=cap, workspace=ws, rownorm=rn_o)
        pa = rn_o.ss_parts
        rn_m = ops.row_norm(ss_in=ss_a[: T * pa].view(T, pa), ss_in_parts=pa, hidden=hid, eps=eps)
        act = ops.gemm(x, self.w(p + "w13"), out=buf["act"], silu_mul=True, max_ctas=cap, workspace=ws,
                       rownorm=rn_m)
        rn_d = ops.row_norm(ss_out=ss_b)
        ops.gemm(act, self.w(p + "w2"), out=x, residual=x, max_ctas=cap, workspace=ws, rownorm=rn_d)
        return rn_d.ss_parts

    def _final_rownorm(self, buf: dict, T: int, ss_parts: int):
        """The final RMSNorm as the LM head's row scale (folded path)."""
        if not ss_parts:
            return None
        return ops.row_norm(ss_in=buf["ss"][1][: T * ss_parts].view(T, ss_parts), ss_in_parts=ss_parts,
                            hidden=self.arch.hidden, eps=self.arch.rms_eps)

    def _block_fused(self, x, layer, attn_fn, buf, rope, cap, ar, h_ready, final) -> bool:
        st = self.state
        eps = self.arch.rms_eps
        p = f"L{layer}."
        lead = st.rank == 0
        ws = buf["ws"]
        local = layer - st.weights.layer_begin
        nq, nk = st.weights.n_q_heads, st.weights.n_kv_heads
        pos, slots = rope
        geo = self.geometry().as_tuple()
        T = x.shape[0]
        h, part = ar.h[:T], ar.part[:T]
        if not h_ready:
            ops.rmsnorm(x, self.w(p + "attn_norm"), eps, out=h)
        if self.fuse_rope and self.arch.head_dim == 128:
            qkv = ops.gemm_qkv_rope_kv(h, self.w(p + "wqkv"), buf["qkv"], nq, nk, pos, self.rope_cos, self.rope_sin,
                                       self.pool, geo, local, slots, max_ctas=cap, workspace=ws)
        else:
            qkv = ops.gemm(h, self.w(p + "wqkv"), out=buf["qkv"], max_ctas=cap, workspace=ws)
            ops.rope_kv_append(qkv, nq, nk, pos, self.rope_cos, self.rope_sin, self.pool, geo, local, slots)
        attn = attn_fn(qkv, local)
        ops.gemm(attn, self.w(p + "wo"), out=part, residual=x if lead else None, max_ctas=cap, workspace=ws)
        ar.combine(T, self.w(p + "mlp_norm"), eps)
        act = ops.gemm(h, self.w(p + "w13"), out=buf["act"], silu_mul=True, max_ctas=cap, workspace=ws)
        ops.gemm(act, self.w(p + "w2"), out=part, residual=x if lead else None, max_ctas=cap, workspace=ws)
        g = self._next_gamma(layer, final)
        ar.combine(T, g, eps)
        return g is not None

    def _block_fused_folded(self, x, layer, attn_fn, buf, rope, cap, ar, ss_ready: bool) -> bool:
        """TP layer with the fused combine AND the folded norm: each combine
        leaves x and its per-row sum of squares (ar.ss) on every rank; the
        QKV and gate/up GEMMs read x and scale their rows by 1/rms (gains
        folded into their weights, fold_gains).  ``ss_ready``: ar.ss holds
        this layer's input sums (else its attn_norm runs as a kernel)."""
        st = self.state
        eps = self.arch.rms_eps
        hid = self.arch.hidden
        p = f"L{layer}."
        lead = st.rank == 0
        ws = buf["ws"]
        local = layer - st.weights.layer_begin
        nq, nk = st.weights.n_q_heads, st.weights.n_kv_heads
        pos, slots = rope
        geo = self.geometry().as_tuple()
        T = x.shape[0]
        part, ss = ar.part[:T], ar.ss[:T].view(T, 1)
        if ss_ready:
            a_in, rn = x, ops.row_norm(ss_in=ss, ss_in_parts=1, hidden=hid, eps=eps)
        else:
            a_in, rn = ops.rmsnorm(x, self.w(p + "attn_norm"), eps, out=ar.h[:T]), None
        if self.fuse_rope and self.arch.head_dim == 128:
            qkv = ops.gemm_qkv_rope_kv(a_in, self.w(p + "wqkv"), buf["qkv"], nq, nk, pos, self.rope_cos,
                                       self.rope_sin, self.pool, geo, local, slots, max_ctas=cap, workspace=ws,
                                       rownorm=rn)
        else:
            qkv = ops.gemm(a_in, self.w(p + "wqkv"), out=buf["qkv"], max_ctas=cap, workspace=ws, rownorm=rn)
            ops.rope_kv_append(qkv, nq, nk, pos, self.rope_cos, self.rope_sin, self.pool, geo, local, slots)
        attn = attn_fn(qkv, local)
        ops.gemm(attn, self.w(p + "wo"), out=part, residual=x if lead else None, max_ctas=cap, workspace=ws)
        ar.combine_ss(T)
        rn_m = ops.row_norm(ss_in=ss, ss_in_parts=1, hidden=hid, eps=eps)
        act = ops.gemm(x, self.w(p + "w13"), out=buf["act"], silu_mul=True, max_ctas=cap, workspace=ws,
                       rownorm=rn_m)
        ops.gemm(act, self.w(p + "w2"), out=part, residual=x if lead else None, max_ctas=cap, workspace=ws)
        ar.combine_ss(T)
        return True

    def _tp_fold(self, ar) -> bool:
        """Decode under a pure TP layout with the fused combine runs folded."""
        return ar is not None and self.fold_norm and self.tp_fold and self.state.cfg.pp == 1

    def _reduce_into(self, x: torch.Tensor) -> None:
        """Row-parallel combine: rank 0 added the residual in its GEMM epilogue,
        the others hold partial sums; the all-reduce yields residual + sum."""
        if self.state.tp_comm.size > 1:
            self.state.tp_comm.all_reduce_(x)

    def _alloc_buffers(self, T: int) -> dict:
        st = self.state
        a = self.arch
        nq, nk = st.weights.n_q_heads, st.weights.n_kv_heads
        dev = self.device
        return {
            "h": torch.empty(T, a.hidden, dtype=torch.bfloat16, device=dev),
            "qkv": torch.empty(T, (nq + 2 * nk) * a.head_dim, dtype=torch.bfloat16, device=dev),
            "attn": torch.empty(T, nq * a.head_dim, dtype=torch.bfloat16, device=dev),
            "act": torch.empty(T, st.weights.ffn_local, dtype=torch.bfloat16, device=dev),
            # folded-norm row sums of squares: [T][N tiles] of the o_proj
            # and down_proj outputs (N tile >= 64 columns)
            "ss": [torch.empty(T * ((a.hidden + 63) // 64), dtype=torch.float32, device=dev) for _ in range(2)],
        }

    def _buffers(self, T: int, lane=0) -> dict:
        """Activation buffers of a T-row forward, one set per decode lane.
        Lane "graph" is the set the captured decode steps own: allocated at
        a capacity (the largest batch seen) and handed out as [:T] views, so
        every graph keeps pointing at live memory; growing it drops the
        graphs (``_graph_capacity``)."""
        st = self.state
        a = self.arch
        slot = self._bufs.setdefault(lane, {})
        if lane == "graph":
            full = slot["full"]
            tiles = (a.hidden + 63) // 64
            buf = {k: v[:T] for k, v in full.items() if k != "ss"}
            buf["ss"] = [s[: T * tiles] for s in full["ss"]]
        else:
            key = ("buf", T, st.cfg.tp)
            if slot.get("key") != key:
                slot["key"] = key
                slot["buf"] = self._alloc_buffers(T)
            buf = slot["buf"]
        if "ws" not in slot:
            # split-K workspace of this lane's stream (zeroed once; the GEMM
            # leaves its tile counters zero), see ssb_gemm_bf16_ws
            slot["ws"] = torch.zeros(self.GEMM_WS_BYTES, dtype=torch.uint8, device=self.device)
        buf["ws"] = slot["ws"] if self.split_k else None
        return buf

    def _graph_capacity(self, B: int) -> None:
        """Make the graph-owned buffers hold B rows under the current layout;
        a reallocation invalidates every captured step."""
        st = self.state
        slot = self._bufs.setdefault("graph", {})
        key = (st.cfg.tp, st.weights.ffn_local, st.weights.n_q_heads, st.weights.n_kv_heads)
        if slot.get("key") == key and slot.get("cap", 0) >= B:
            return
        self._drop_graphs()
        cap = max(B, slot.get("cap", 0) if slot.get("key") == key else 0)
        full = self._alloc_buffers(cap)
        full["x"] = torch.empty(cap, self.arch.hidden, dtype=torch.bfloat16, device=self.device)
        slot.update(key=key, cap=cap, full=full)

    def _logits_argmax(self, h_last: torch.Tensor, out_tokens: torch.Tensor, ws: torch.Tensor | None = None,
                       rownorm=None) -> None:
        """Vocab-parallel LM head + greedy argmax (fp32 logits).  ``rownorm``:
        h_last is the un-normed x and the final norm is the GEMM's row scale."""
        st = self.state
        n = h_last.shape[0]
        vals = torch.empty(n, dtype=torch.float32, device=self.device)
        idxs = torch.empty(n, dtype=torch.int32, device=self.device)
        ar = self._arena(n) if st.tp_comm.size > 1 and not self.record_logits and self.fuse_argmax else None
        if ar is not None:
            # every rank's argmax keys meet over peer memory: no all-gather
            ops.lm_head_keys(h_last, self.w("head"), st.weights.vocab_begin, ar.keys[:n], workspace=ws,
                             rownorm=rownorm)
            ar.argmax(n, out_tokens)
            return
        if self.record_logits or not self.fuse_argmax:
            logits = ops.gemm(h_last, self.w("head"), out_f32=True, workspace=ws, rownorm=rownorm)
            ops.argmax_rows(logits, st.weights.vocab_begin, vals, idxs)
            if self.record_logits:
                self._record(logits)
        else:
            # argmax in the LM-head GEMM epilogue: no [n, vocab] fp32 logits round trip
            ops.lm_head_argmax(h_last, self.w("head"), st.weights.vocab_begin, vals, idxs, workspace=ws,
                               rownorm=rownorm)
        if st.tp_comm.size == 1:
            out_tokens.copy_(idxs)
            return
        P = st.tp_comm.size
        gv = torch.empty(P * n, dtype=torch.float32, device=self.device)
        gi = torch.empty(P * n, dtype=torch.int32, device=self.device)
        st.tp_comm.all_gather(gv, vals)
        st.tp_comm.all_gather(gi, idxs)
        ops.argmax_combine(gv.view(P, n), gi.view(P, n), out_tokens)

    def _record(self, logits: torch.Tensor) -> None:
        st = self.state
        if st.tp_comm.size > 1:
            P = st.tp_comm.size
            g = torch.empty(P * logits.numel(), dtype=torch.float32, device=self.device)
            st.tp_comm.all_gather(g, logits.contiguous())
            logits = g.view(P, *logits.shape).permute(1, 0, 2).reshape(logits.shape[0], -1)
        self.logit_log.append(logits.detach().float().cpu())

    def prefill(self, tokens: torch.Tensor, cu_seqlens: np.ndarray, tables: np.ndarray,
                first_tokens: torch.Tensor) -> None:
        """Prefill a micro-batch of packed prompts through this GPU's stage.

        tokens: int32 [T] on device (used on stage 0); cu_seqlens: host
        int32 [n+1]; tables: host int32 [n, max_blocks].  Stage s>0 receives
        the activations from s-1, stage s<pp-1 sends to s+1; the last stage
        writes the greedy first token of every prompt into first_tokens[n]."""
        st = self.state
        a = self.arch
        T = int(cu_seqlens[-1])
        n = len(cu_seqlens) - 1
        buf = self._buffers(T)
        ar = self._arena(T)
        h_ready = False
        if ar is not None:
            x = ar.x[:T]
        else:
            x = torch.empty(T, a.hidden, dtype=torch.bfloat16, device=self.device)
        if st.stage == 0:
            if ar is not None:
                ops.embedding(tokens, self.w("embed"), st.weights.vocab_begin, ar.part[:T])
                ar.combine(T, self.w(f"L{st.weights.layer_begin}.attn_norm"), a.rms_eps)
                h_ready = True
            else:
                ops.embedding(tokens, self.w("embed"), st.weights.vocab_begin, x)
                if st.tp_comm.size > 1:
                    st.tp_comm.all_reduce_(x)
        else:
            self.replica_comm.recv(x, st.pp_prev)
        pos = np.concatenate([np.arange(cu_seqlens[i + 1] - cu_seqlens[i], dtype=np.int32) for i in range(n)])
        seq_of = np.repeat(np.arange(n), np.diff(cu_seqlens))
        bs = self.block_size
        slots = tables[seq_of, pos // bs].astype(np.int64) * bs + pos % bs
        pos_d = torch.from_numpy(pos).to(self.device)
        slots_d = torch.from_numpy(slots).to(self.device)
        cu_d = torch.from_numpy(np.asarray(cu_seqlens, dtype=np.int32)).to(self.device)
        max_len = int(np.max(np.diff(cu_seqlens)))
        geo = self.geometry()
        nq, nk = st.weights.n_q_heads, st.weights.n_kv_heads

        def attn(qkv, layer_local):
            return ops.prefill_attention(qkv, nq, nk, a.head_dim, cu_d, max_len, buf["attn"], self.scale)

        for layer in self._layers():
            h_ready = self._block(x, layer, attn, buf, (pos_d, slots_d), ar=ar, h_ready=h_ready)
        if st.stage < st.cfg.pp - 1:
            self.replica_comm.send(x, st.pp_next)
            return
        last = torch.from_numpy(np.asarray(cu_seqlens[1:], dtype=np.int32) - 1).to(self.device)
        h_last = ops.rmsnorm(x, self.w("final_norm"), a.rms_eps, row_idx=last)
        self._logits_argmax(h_last, first_tokens)

    def decode_round(self, tokens: torch.Tensor, ctx_lens: torch.Tensor, tables: torch.Tensor,
                     positions: torch.Tensor, slots: torch.Tensor, out_tokens: torch.Tensor,
                     spans: list[tuple[int, int]]) -> None:
        """One decode round of the batch: every row advances one token.

        pp = 1: one decode step of the whole batch (``spans`` is one span).
        pp > 1 (sim.py:517-535): the rows are split into the micro-batches
        ``spans`` (ceil(n/pp) rows each); every stage runs its layers on each
        micro-batch in turn — stage 0 embeds, the others receive the
        activations from the previous stage, the last stage computes the
        greedy tokens — so micro-batch i+1 enters stage 0 while micro-batch
        i is in stage 1 (the pipeline).  At the end of the round the last
        stage returns the round's tokens to stage 0, which embeds them next
        round (the pipeline drains once per round)."""
        st = self.state
        if st.cfg.pp == 1:
            assert len(spans) == 1 and spans[0] == (0, tokens.numel())
            self.decode_step(tokens, ctx_lens, tables, positions, slots, out_tokens)
            return
        a = self.arch
        geo = self.geometry()
        nq, nk = st.weights.n_q_heads, st.weights.n_kv_heads
        first, last = st.stage == 0, st.stage == st.cfg.pp - 1
        for lane, (b0, b1) in enumerate(spans):
            n = b1 - b0
            buf = self._buffers(n, lane=lane)
            v = dict(tok=tokens[b0:b1], ctx=ctx_lens[b0:b1], tab=tables[b0:b1], pos=positions[b0:b1],
                     slot=slots[b0:b1], out=out_tokens[b0:b1])
            ops.decode_positions(v["ctx"], v["tab"], self.block_size, v["pos"], v["slot"])
            ar = self._arena(n)
            h_ready = False
            if ar is not None:
                x = ar.x[:n]
            else:
                x = buf.get("x")
                if x is None or x.shape[0] != n:
                    x = buf["x"] = torch.empty(n, a.hidden, dtype=torch.bfloat16, device=self.device)
            fold = self._tp_fold(ar)
            if first:
                if ar is not None:
                    ops.embedding(v["tok"], self.w("embed"), st.weights.vocab_begin, ar.part[:n])
                    if fold:
                        ar.combine_ss(n)
                    else:
                        ar.combine(n, self.w(f"L{st.weights.layer_begin}.attn_norm"), a.rms_eps)
                    h_ready = True
                else:
                    ops.embedding(v["tok"], self.w("embed"), st.weights.vocab_begin, x)
                    if st.tp_comm.size > 1:
                        st.tp_comm.all_reduce_(x)
            else:
                self.replica_comm.recv(x, st.pp_prev)

            def attn(qkv, layer_local, v=v, buf=buf):
                return ops.decode_attention(qkv, nq, nk, self.pool, geo.as_tuple(), self.num_blocks,
                                            layer_local, v["tab"], v["ctx"], buf["attn"], self.scale)

            for layer in self._layers():
                h_ready = self._block(x, layer, attn, buf, (v["pos"], v["slot"]), ar=ar, h_ready=h_ready,
                                      final=last, fold=fold)
            if not last:
                self.replica_comm.send(x, st.pp_next)
                continue
            rn = None
            if ar is not None and h_ready and fold:
                h, rn = x, ops.row_norm(ss_in=ar.ss[:n].view(n, 1), ss_in_parts=1, hidden=a.hidden, eps=a.rms_eps)
            elif ar is not None and h_ready:
                h = ar.h[:n]
            elif self.fold_norm and st.tp_comm.size == 1 and h_ready:
                h, rn = x, self._final_rownorm(buf, n, int(h_ready))
            else:
                h = ops.rmsnorm(x, self.w("final_norm"), a.rms_eps, out=buf["h"])
            self._logits_argmax(h, v["out"], buf["ws"], rownorm=rn)
        # the round's tokens back to the stage that embeds them
        src = (st.cfg.pp - 1) * st.cfg.tp + st.rank
        dst = st.rank
        if last:
            self.replica_comm.send(out_tokens, dst)
        elif first:
            self.replica_comm.recv(out_tokens, src)

    def runtime_reserve_bytes(self, cfg_p: ParallelismConfig, cfg_d: ParallelismConfig, max_prefill_tokens: int) -> int:
        """HBM this GPU needs beyond its weights and KV pool at the peak of a
        run (ADVICE: the pool must leave room for it); see :func:`runtime_reserve`."""
        return runtime_reserve(self.arch, self.gpu, cfg_p, cfg_d, max_prefill_tokens, self.block_size,
                               self.GEMM_WS_BYTES, self.RESHARD_CHUNK_BYTES)["total"]

    def check_peer_errors(self) -> None:
        """Raise if a fused TP combine's peer barrier timed out (host sync)."""
        for ar in self._tp_arenas.values():
            if ar.usable:
                ar.check()

    def decode_step(self, tokens: torch.Tensor, ctx_lens: torch.Tensor, tables: torch.Tensor,
                    positions: torch.Tensor, slots: torch.Tensor, out_tokens: torch.Tensor) -> None:
        """One decode step of the resident batch under a pure-TP layout:
        tokens[B] in, next greedy tokens into out_tokens[B]; ctx_lens grows by one.

        With ``decode_lanes == 2`` the batch is split into two halves issued on
        two CUDA streams, layer by layer: one half's paged attention (HBM
        bound) runs while the other half's projections (tensor bound) run on
        the SMs the capped persistent GEMM leaves free."""
        B = tokens.numel()
        lanes = self.decode_lanes if (B >= 2 * self.min_lane_rows and not self.record_logits) else 1
        if lanes == 1:
            if self._graph_ok(B):
                self._decode_step_graph(tokens, ctx_lens, tables, positions, slots, out_tokens)
                return
            self._decode_lanes([(0, B)], tokens, ctx_lens, tables, positions, slots, out_tokens, 0)
            return
        h = B // 2
        self._decode_lanes([(0, h), (h, B)], tokens, ctx_lens, tables, positions, slots, out_tokens,
                           self.lane_gemm_cap)

    # ------------------------------------------------------- CUDA graphs --
    def _graph_ok(self, B: int) -> bool:
        """A decode step is captured in a CUDA graph when nothing in it needs
        the host: one lane, a pure tensor-parallel layout whose collectives
        all run as peer-memory kernels (the fused combine and the peer argmax;
        tp = 1 has none), no logit recording, no per-launch profiling."""
        from . import _lib

        if not self.cuda_graphs or self.device.type != "cuda" or self.record_logits or _lib.STATS.timing:
            return False
        st = self.state
        if st.cfg.pp != 1:
            return False
        from .comm import ThreadComm

        if isinstance(self.world, ThreadComm) and self.world.size > st.tp_comm.size:
            # virtual ranks of OTHER replicas share this device and process and
            # step on their own schedule: their device-wide synchronisations
            # would invalidate this thread's capture (one process per GPU has
            # no such neighbours)
            return False
        if st.tp_comm.size > 1:
            return self.fuse_argmax and self._arena(B) is not None
        return True

    def _decode_step_graph(self, tokens, ctx_lens, tables, positions, slots, out_tokens) -> None:
        """Replay the captured decode step of this batch size: the step's
        inputs are copied into the graph's static buffers, its outputs copied
        back.  A batch size is captured the second time it occurs (the first
        occurrence runs eagerly and warms every lazy allocation); the ~6L+10
        library launches of a step become one graph launch, which removes the
        per-launch host cost that bounds a TP8 step (~2-3 ms of GPU work)."""
        from . import _lib

        B = tokens.numel()
        st = self.state
        ar = self._arena(B) if st.tp_comm.size > 1 else None
        self._graph_capacity(B)
        key = (B, tables.shape[1], st.cfg, self.pool.data_ptr(), st.arena.data_ptr(),
               ar.generation if ar is not None else 0, self.fold_norm, self.tp_fold,
               self.fuse_rope, self.split_k)
        ent = self._graphs.get(key)
        if ent is None:
            ent = self._graphs[key] = {
                "tok": torch.empty_like(tokens), "ctx": torch.empty_like(ctx_lens), "tab": torch.empty_like(tables),
                "pos": torch.empty_like(positions), "slot": torch.empty_like(slots),
                "out": torch.empty_like(out_tokens), "graph": None, "seen": 0, "launches": 0}
        ent["tok"].copy_(tokens)
        ent["ctx"].copy_(ctx_lens)
        ent["tab"].copy_(tables)
        args = (ent["tok"], ent["ctx"], ent["tab"], ent["pos"], ent["slot"], ent["out"])
        if ent["graph"] is not None:
            ent["graph"].replay()
            _lib.STATS.count += ent["launches"]
        else:
            self._decode_lanes([(0, B)], *args, 0, buf_lane="graph")
            ent["seen"] += 1
            if ent["seen"] >= 2:
                self._capture_group(ent, args, B)
        ctx_lens.copy_(ent["ctx"])
        positions.copy_(ent["pos"])
        slots.copy_(ent["slot"])
        out_tokens.copy_(ent["out"])

    def _capture_group(self, ent: dict, args, B: int) -> None:
        """Capture this rank's step.  Virtual ranks (ThreadComm threads on one
        device) capture one at a time between host barriers: torch's capture
        entry synchronizes the whole device and empties the allocator cache,
        which must not happen while a peer thread is capturing, or while a
        peer's combine kernel is still waiting on this rank's next step.  The
        group agrees on the outcome, so no rank replays a graph while another
        runs eagerly-with-a-failed-capture (their kernel sequences would
        still match, but a mixed group is not worth the doubt)."""
        from .comm import ThreadComm

        tp = self.state.tp_comm
        if not isinstance(tp, ThreadComm) or tp.size == 1:
            self._capture(ent, args, B)
            return
        for turn in range(tp.size):
            tp.barrier()
            if turn == tp.rank:
                self._capture(ent, args, B)
        flags = tp._exchange(ent["graph"] is not None)
        tp._done()
        if not all(flags):
            ent["graph"] = None
            self.cuda_graphs = False

    def _capture(self, ent: dict, args, B: int) -> None:
        """Record one decode step on the static buffers into a CUDA graph
        (capture only records; the step that just ran eagerly was the real
        one).  A capture failure disables graphs for this worker."""
        from . import _lib

        if self._graph_pool is None:
            self._graph_pool = torch.cuda.graph_pool_handle()
        g = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream(self.device)
        cap.wait_stream(torch.cuda.current_stream(self.device))
        n0 = _lib.STATS.count
        try:
            with torch.cuda.graph(g, pool=self._graph_pool, stream=cap, capture_error_mode="thread_local"):
                self._decode_lanes([(0, B)], *args, 0, buf_lane="graph")
        except RuntimeError as exc:  # noqa: BLE001 - any capture failure falls back to eager launches
            import warnings

            warnings.warn(f"decode-step CUDA graph capture failed ({exc}); running eagerly", RuntimeWarning,
                          stacklevel=2)
            self.cuda_graphs = False
            _lib.STATS.count = n0
            return
        torch.cuda.current_stream(self.device).wait_stream(cap)
        ent["launches"] = _lib.STATS.count - n0
        _lib.STATS.count = n0
        ent["graph"] = g

    def _drop_graphs(self) -> None:
        """Forget every captured step (weights, pool or peer arena moved)."""
        self._graphs.clear()

    def _decode_lanes(self, spans, tokens, ctx_lens, tables, positions, slots, out_tokens, cap,
                      buf_lane=None) -> None:
        st = self.state
        a = self.arch
        main = torch.cuda.current_stream(self.device)
        if len(spans) > 1:
            if self._side is None:
                self._side = torch.cuda.Stream(self.device)
            self._side.wait_stream(main)
        streams = [main] + [self._side] * (len(spans) - 1)
        geo = self.geometry()
        nq, nk = st.weights.n_q_heads, st.weights.n_kv_heads
        lanes = []
        ar = self._arena(spans[0][1] - spans[0][0]) if len(spans) == 1 else None
        fold = self._tp_fold(ar)
        final = st.stage == st.cfg.pp - 1
        for li, ((b0, b1), s) in enumerate(zip(spans, streams)):
            with torch.cuda.stream(s):
                n = b1 - b0
                buf = self._buffers(n, lane=li if buf_lane is None else buf_lane)
                v = dict(tok=tokens[b0:b1], ctx=ctx_lens[b0:b1], tab=tables[b0:b1], pos=positions[b0:b1],
                         slot=slots[b0:b1], out=out_tokens[b0:b1], h_ready=False)
                ops.decode_positions(v["ctx"], v["tab"], self.block_size, v["pos"], v["slot"])
                if ar is not None:
                    x = ar.x[:n]
                    ops.embedding(v["tok"], self.w("embed"), st.weights.vocab_begin, ar.part[:n])
                    if fold:
                        ar.combine_ss(n)
                    else:
                        ar.combine(n, self.w(f"L{st.weights.layer_begin}.attn_norm"), a.rms_eps)
                    v["h_ready"] = True
                else:
                    x = buf.get("x")
                    if x is None or x.shape[0] != n:
                        x = buf["x"] = torch.empty(n, a.hidden, dtype=torch.bfloat16, device=self.device)
                    ops.embedding(v["tok"], self.w("embed"), st.weights.vocab_begin, x)
                    if st.tp_comm.size > 1:
                        st.tp_comm.all_reduce_(x)

                def attn(qkv, layer_local, v=v, buf=buf):
                    return ops.decode_attention(qkv, nq, nk, self.pool, geo.as_tuple(), self.num_blocks,
                                                layer_local, v["tab"], v["ctx"], buf["attn"], self.scale)

                lanes.append((s, x, attn, buf, v))
        for layer in self._layers():
            for s, x, attn, buf, v in lanes:
                with torch.cuda.stream(s):
                    v["h_ready"] = self._block(x, layer, attn, buf, (v["pos"], v["slot"]), cap, ar=ar,
                                               h_ready=v["h_ready"], final=final, fold=fold)
        for s, x, _, buf, v in lanes:
            with torch.cuda.stream(s):
                rn = None
                n = x.shape[0]
                if ar is not None and v["h_ready"] and fold:
                    h, rn = x, ops.row_norm(ss_in=ar.ss[:n].view(n, 1), ss_in_parts=1, hidden=a.hidden,
                                            eps=a.rms_eps)
                elif ar is not None and v["h_ready"]:
                    h = ar.h[:n]
                elif self.fold_norm and st.tp_comm.size == 1 and v["h_ready"]:
                    h, rn = x, self._final_rownorm(buf, x.shape[0], int(v["h_ready"]))
                else:
                    h = ops.rmsnorm(x, self.w("final_norm"), a.rms_eps, out=buf["h"])
                self._logits_argmax(h, v["out"], buf["ws"], rownorm=rn)
        if len(spans) > 1:
            main.wait_stream(self._side)
