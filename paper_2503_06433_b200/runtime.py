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
        self.stream = torch.cuda.current_stream(device) if device.type == "cuda" else None
        self.record_logits = False
        self.logit_log: list[torch.Tensor] = []
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
        geo = self.geometry()
        # zero-filled once: decode attention multiplies the (masked, p = 0)
        # tail of a sequence's last block by its V rows, and never-written
        # memory may hold NaN bit patterns (0 * NaN = NaN).  Afterwards a block
        # only ever holds finite KV of some sequence.
        self.pool = torch.zeros(num_blocks * geo.block_elems, dtype=torch.bfloat16, device=self.device)

    # ------------------------------------------------------- re-partition --
    def repartition_weights(self, cfg_new: ParallelismConfig) -> int:
        """Weight column/row re-partition over the replica group; returns bytes
        this GPU sent to other GPUs."""
        old = self.state
        new = self.make_layout(cfg_new)
        n = self.per_replica
        old_layouts = [weight_layout(self.arch, old.cfg.tp, old.cfg.pp, g) for g in range(n)]
        new_layouts = [weight_layout(self.arch, cfg_new.tp, cfg_new.pp, g) for g in range(n)]
        send_entries, recv_entries = [], []
        send_splits, recv_splits = [], []
        s_pos = r_pos = 0
        for q in range(n):
            pieces = repartition_pieces(old_layouts[self.gpu], new_layouts[q])
            start = s_pos
            for p in pieces:
                send_entries.append((p.src_off * 2, s_pos * 2, p.src_ld * 2, p.cols * 2, p.rows, p.cols * 2))
                s_pos += p.numel
            send_splits.append(s_pos - start)
            pieces = repartition_pieces(old_layouts[q], new_layouts[self.gpu])
            start = r_pos
            for p in pieces:
                recv_entries.append((r_pos * 2, p.dst_off * 2, p.cols * 2, p.dst_ld * 2, p.rows, p.cols * 2))
                r_pos += p.numel
            recv_splits.append(r_pos - start)
        recv = torch.empty(max(r_pos, 8), dtype=torch.bfloat16, device=self.device)
        rd, rtot = _copy_desc_rows(recv_entries)
        if self.p2p_reshard and self.device.type == "cuda" and n > 1:
            # pack + transfer in one kernel: every piece is stored straight into
            # its owner's receive buffer (IPC peer memory), at the section that
            # follows the sections of the ranks before this one
            addrs = self.replica_comm.peer_addresses(recv)
            p2p_entries = []
            for q in range(n):
                base = sum(pc.numel for p in range(self.gpu)
                           for pc in repartition_pieces(old_layouts[p], new_layouts[q]))
                for pc in repartition_pieces(old_layouts[self.gpu], new_layouts[q]):
                    p2p_entries.append((pc.src_off * 2, addrs[q] + base * 2, pc.src_ld * 2, pc.cols * 2, pc.rows,
                                        pc.cols * 2))
                    base += pc.numel
            pd, ptot = _copy_desc_rows(p2p_entries)
            stream = torch.cuda.current_stream(self.device)
            stream.synchronize()
            self.replica_comm.barrier()  # every receive buffer exists and is idle
            if ptot:
                ops.copy2d_batched(old.arena, None, torch.from_numpy(pd).to(self.device), ptot)
            stream.synchronize()
            self.replica_comm.barrier()  # every piece landed
        else:
            send = torch.empty(max(s_pos, 8), dtype=torch.bfloat16, device=self.device)
            sd, stot = _copy_desc_rows(send_entries)
            if stot:
                ops.copy2d_batched(old.arena, send, torch.from_numpy(sd).to(self.device), stot)
            self.replica_comm.all_to_all(recv, send, recv_splits, send_splits)
        if rtot:
            ops.copy2d_batched(recv, new.arena, torch.from_numpy(rd).to(self.device), rtot)
        self.state = new
        return 2 * (s_pos - send_splits[self.gpu])

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
        if getattr(self, "_comm_stream", None) is None:
            self._comm_stream = torch.cuda.Stream(self.device)
        cs = self._comm_stream
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
        key = (src_cfg, dst_cfg, chunk, recv_cells)
        if getattr(self, "_p2p", None) is None or self._p2p[0] != key:
            recv = torch.empty(chunk * recv_cells * cell + 8, dtype=torch.bfloat16, device=self.device)
            self._p2p = (key, recv, self.replica_comm.peer_addresses(recv))
        _, recv, addrs = self._p2p
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
               h_ready: bool = False, final: bool = False) -> bool:
        """One transformer layer on x (in place); attn_fn(qkv, layer_local) -> attn out.
        ``rope`` = (positions, slots) of the rows: RoPE and the paged K/V
        append run in the QKV GEMM's epilogue (head_dim 128) or as a separate
        kernel.  ``cap`` bounds the GEMMs' persistent grid (decode lane overlap).

        With a peer arena ``ar`` (TP > 1, x = ar.x[:T]) the row-parallel
        projections write their partials to ar.part and each combine also
        produces the NEXT rmsnorm (ar.h): ``h_ready`` says this layer's input
        norm is already in ar.h; returns whether the next one is (the
        combine after the MLP applies the next layer's attn_norm, or
        final_norm on the last layer when ``final``)."""
        if ar is not None:
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

    def _reduce_into(self, x: torch.Tensor) -> None:
        """Row-parallel combine: rank 0 added the residual in its GEMM epilogue,
        the others hold partial sums; the all-reduce yields residual + sum."""
        if self.state.tp_comm.size > 1:
            self.state.tp_comm.all_reduce_(x)

    def _buffers(self, T: int, lane: int = 0) -> dict:
        """Activation buffers of a T-row forward, one set per decode lane."""
        st = self.state
        a = self.arch
        nq, nk = st.weights.n_q_heads, st.weights.n_kv_heads
        key = ("buf", T, st.cfg.tp)
        slot = self._bufs.setdefault(lane, {})
        if slot.get("key") != key:
            dev = self.device
            slot["key"] = key
            slot["buf"] = {
                "h": torch.empty(T, a.hidden, dtype=torch.bfloat16, device=dev),
                "qkv": torch.empty(T, (nq + 2 * nk) * a.head_dim, dtype=torch.bfloat16, device=dev),
                "attn": torch.empty(T, nq * a.head_dim, dtype=torch.bfloat16, device=dev),
                "act": torch.empty(T, st.weights.ffn_local, dtype=torch.bfloat16, device=dev),
                # folded-norm row sums of squares: [T][N tiles] of the o_proj
                # and down_proj outputs (N tile >= 64 columns)
                "ss": [torch.empty(T * ((a.hidden + 63) // 64), dtype=torch.float32, device=dev) for _ in range(2)],
            }
        if "ws" not in slot:
            # split-K workspace of this lane's stream (zeroed once; the GEMM
            # leaves its tile counters zero), see ssb_gemm_bf16_ws
            slot["ws"] = torch.zeros(self.GEMM_WS_BYTES, dtype=torch.uint8, device=self.device)
        slot["buf"]["ws"] = slot["ws"] if self.split_k else None
        return slot["buf"]

    def _logits_argmax(self, h_last: torch.Tensor, out_tokens: torch.Tensor, ws: torch.Tensor | None = None,
                       rownorm=None) -> None:
        """Vocab-parallel LM head + greedy argmax (fp32 logits).  ``rownorm``:
        h_last is the un-normed x and the final norm is the GEMM's row scale."""
        st = self.state
        n = h_last.shape[0]
        vals = torch.empty(n, dtype=torch.float32, device=self.device)
        idxs = torch.empty(n, dtype=torch.int32, device=self.device)
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
            self._decode_lanes([(0, B)], tokens, ctx_lens, tables, positions, slots, out_tokens, 0)
            return
        h = B // 2
        self._decode_lanes([(0, h), (h, B)], tokens, ctx_lens, tables, positions, slots, out_tokens,
                           self.lane_gemm_cap)

    def _decode_lanes(self, spans, tokens, ctx_lens, tables, positions, slots, out_tokens, cap) -> None:
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
        final = st.stage == st.cfg.pp - 1
        for li, ((b0, b1), s) in enumerate(zip(spans, streams)):
            with torch.cuda.stream(s):
                n = b1 - b0
                buf = self._buffers(n, lane=li)
                v = dict(tok=tokens[b0:b1], ctx=ctx_lens[b0:b1], tab=tables[b0:b1], pos=positions[b0:b1],
                         slot=slots[b0:b1], out=out_tokens[b0:b1], h_ready=False)
                ops.decode_positions(v["ctx"], v["tab"], self.block_size, v["pos"], v["slot"])
                if ar is not None:
                    x = ar.x[:n]
                    ops.embedding(v["tok"], self.w("embed"), st.weights.vocab_begin, ar.part[:n])
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
                                               h_ready=v["h_ready"], final=final)
        for s, x, _, buf, v in lanes:
            with torch.cuda.stream(s):
                rn = None
                if ar is not None and v["h_ready"]:
                    h = ar.h[: x.shape[0]]
                elif self.fold_norm and st.tp_comm.size == 1 and v["h_ready"]:
                    h, rn = x, self._final_rownorm(buf, x.shape[0], int(v["h_ready"]))
                else:
                    h = ops.rmsnorm(x, self.w("final_norm"), a.rms_eps, out=buf["h"])
                self._logits_argmax(h, v["out"], buf["ws"], rownorm=rn)
        if len(spans) > 1:
            main.wait_stream(self._side)
