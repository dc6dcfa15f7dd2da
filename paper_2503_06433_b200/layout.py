"""Physical placement of weights and KV-cache on one GPU for a (tp, pp) layout.

Every GPU keeps its weights in one flat bf16 *arena*; each local tensor is a
2-D region of it described by *segments* — rectangles of a LOGICAL tensor
(the unsharded Llama parameter).  A weight re-partition between two layouts is
then the set of pairwise segment intersections (see :func:`repartition_pieces`),
executed as batched strided copies plus an all-to-all.

Placement rules follow the reference's shard map (reshard.py:98-122): stage s
owns layers [s*L/pp, (s+1)*L/pp); tensor rank r owns KV heads
[r*h_kv/tp, ...).  Beyond the reference (which folds all weights into a
per-layer W): Q heads follow their KV group, the FFN and
vocabulary are split evenly by rank, the embedding lives on stage 0 and the
LM head + final norm on the last stage, vocab-parallel across that stage's
ranks.  Column-parallel weights (QKV, gate/up) are row blocks; row-parallel
weights (O, down) are column slices.  Gate and up rows are interleaved in
groups of 32 so one GEMM tile holds matching columns for the fused
SiLU·mul epilogue.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

from .arch import LlamaArch

ALIGN = 64  # elements (128 B) between local tensors in the arena
GATE_UP_GROUP = 32


@dataclass(frozen=True)
class Logical:
    name: str
    tensor_id: int
    rows: int
    cols: int
    scale: float   # std of the N(0, scale^2) init; 0 => constant one (norm gains)


def logical_tensors(arch: LlamaArch) -> dict[str, Logical]:
    """The unsharded parameter set and its init convention."""
    h, d, f, v = arch.hidden, arch.head_dim, arch.ffn, arch.vocab
    hq, hk = arch.num_query_heads, arch.num_kv_heads
    out = {
        "embed": Logical("embed", 1, v, h, 1.0),
        "head": Logical("head", 2, v, h, 1.0 / math.sqrt(h)),
        "final_norm": Logical("final_norm", 3, 1, h, 0.0),
    }
    for layer in range(arch.num_layers):
        b = 1000 + 16 * layer
        p = f"L{layer}."
        out[p + "attn_norm"] = Logical(p + "attn_norm", b + 0, 1, h, 0.0)
        out[p + "wq"] = Logical(p + "wq", b + 1, hq * d, h, 1.0 / math.sqrt(h))
        out[p + "wk"] = Logical(p + "wk", b + 2, hk * d, h, 1.0 / math.sqrt(h))
        out[p + "wv"] = Logical(p + "wv", b + 3, hk * d, h, 1.0 / math.sqrt(h))
        out[p + "wo"] = Logical(p + "wo", b + 4, h, hq * d, 1.0 / math.sqrt(hq * d))
        out[p + "mlp_norm"] = Logical(p + "mlp_norm", b + 5, 1, h, 0.0)
        out[p + "w1"] = Logical(p + "w1", b + 6, f, h, 1.0 / math.sqrt(h))
        out[p + "w3"] = Logical(p + "w3", b + 7, f, h, 1.0 / math.sqrt(h))
        out[p + "w2"] = Logical(p + "w2", b + 8, h, f, 1.0 / math.sqrt(f))
    return out


@dataclass(frozen=True)
class Segment:
    """Logical rectangle [row0, row0+rows) x [col0, col0+cols) of ``logical``
    stored at (dst_row, dst_col) of a local tensor."""

    logical: str
    row0: int
    col0: int
    rows: int
    cols: int
    dst_row: int
    dst_col: int


@dataclass
class LocalTensor:
    key: str
    rows: int
    cols: int
    offset: int = 0               # elements into the arena
    segments: list[Segment] = field(default_factory=list)

    @property
    def numel(self) -> int:
        return self.rows * self.cols


@dataclass
class WeightLayout:
    arch: LlamaArch
    tp: int
    pp: int
    stage: int
    rank: int
    tensors: dict[str, LocalTensor]
    arena_elems: int

    @property
    def layer_begin(self) -> int:
        return self.stage * (self.arch.num_layers // self.pp)

    @property
    def layer_end(self) -> int:
        return (self.stage + 1) * (self.arch.num_layers // self.pp)

    @property
    def first_stage(self) -> bool:
        return self.stage == 0

    @property
    def last_stage(self) -> bool:
        return self.stage == self.pp - 1

    @property
    def n_q_heads(self) -> int:
        return self.arch.num_query_heads // self.tp

    @property
    def n_kv_heads(self) -> int:
        return self.arch.num_kv_heads // self.tp

    @property
    def ffn_local(self) -> int:
        return self.arch.ffn // self.tp

    @property
    def vocab_local(self) -> int:
        return self.arch.vocab // self.tp

    @property
    def vocab_begin(self) -> int:
        return self.rank * self.vocab_local

    def has(self, key: str) -> bool:
        return key in self.tensors


def weight_layout(arch: LlamaArch, tp: int, pp: int, gpu: int) -> WeightLayout:
    """Local tensors of replica-GPU ``gpu`` (= stage*tp + rank) under (tp, pp)."""
    arch.validate_layout(tp, pp)
    stage, rank = divmod(gpu, tp)
    h, d = arch.hidden, arch.head_dim
    nq, nk = arch.num_query_heads // tp, arch.num_kv_heads // tp
    q0, k0 = rank * nq, rank * nk
    fl, f0 = arch.ffn // tp, rank * (arch.ffn // tp)
    vl, v0 = arch.vocab // tp, rank * (arch.vocab // tp)
    lps = arch.num_layers // pp
    tensors: dict[str, LocalTensor] = {}

    def add(key, rows, cols, segs):
        tensors[key] = LocalTensor(key, rows, cols, segments=segs)

    if stage == 0:
        add("embed", vl, h, [Segment("embed", v0, 0, vl, h, 0, 0)])
    for layer in range(stage * lps, (stage + 1) * lps):
        p = f"L{layer}."
        add(p + "attn_norm", 1, h, [Segment(p + "attn_norm", 0, 0, 1, h, 0, 0)])
        add(p + "wqkv", (nq + 2 * nk) * d, h, [
            Segment(p + "wq", q0 * d, 0, nq * d, h, 0, 0),
            Segment(p + "wk", k0 * d, 0, nk * d, h, nq * d, 0),
            Segment(p + "wv", k0 * d, 0, nk * d, h, (nq + nk) * d, 0),
        ])
        add(p + "wo", h, nq * d, [Segment(p + "wo", 0, q0 * d, h, nq * d, 0, 0)])
        add(p + "mlp_norm", 1, h, [Segment(p + "mlp_norm", 0, 0, 1, h, 0, 0)])
        segs = []
        for g in range(fl // GATE_UP_GROUP):
            r = f0 + g * GATE_UP_GROUP
            segs.append(Segment(p + "w1", r, 0, GATE_UP_GROUP, h, 2 * g * GATE_UP_GROUP, 0))
            segs.append(Segment(p + "w3", r, 0, GATE_UP_GROUP, h, (2 * g + 1) * GATE_UP_GROUP, 0))
        add(p + "w13", 2 * fl, h, segs)
        add(p + "w2", h, fl, [Segment(p + "w2", 0, f0, h, fl, 0, 0)])
    if stage == pp - 1:
        add("final_norm", 1, h, [Segment("final_norm", 0, 0, 1, h, 0, 0)])
        add("head", vl, h, [Segment("head", v0, 0, vl, h, 0, 0)])
    off = 0
    for t in tensors.values():
        t.offset = off
        off += -(-t.numel // ALIGN) * ALIGN
    return WeightLayout(arch, tp, pp, stage, rank, tensors, off)


@dataclass(frozen=True)
class Piece:
    """One strided copy of a weight re-partition: ``rows`` x ``cols`` elements
    from the src arena (row stride src_ld) to the dst arena (row stride dst_ld)."""

    src_off: int
    dst_off: int
    src_ld: int
    dst_ld: int
    rows: int
    cols: int

    @property
    def numel(self) -> int:
        return self.rows * self.cols

    def row_slice(self, k: int, parts: int) -> "Piece | None":
        """The k-th of ``parts`` row ranges of this piece (None if empty):
        how a re-partition is streamed in chunks every rank agrees on."""
        a, b = k * self.rows // parts, (k + 1) * self.rows // parts
        if b <= a:
            return None
        return Piece(self.src_off + a * self.src_ld, self.dst_off + a * self.dst_ld, self.src_ld, self.dst_ld,
                     b - a, self.cols)


def repartition_pieces(src: WeightLayout, dst: WeightLayout) -> list[Piece]:
    """Everything GPU ``src`` holds that GPU ``dst`` needs, in a deterministic
    order (dst tensor order, then segment order, then src segment order).

    The norm gains are the only tensors a layout replicates (every tensor
    rank of a stage holds them whole); they are sent by the stage's rank 0
    only, so each element of the new layout has exactly one source."""
    by_logical: dict[str, list[tuple[LocalTensor, Segment]]] = {}
    for t in src.tensors.values():
        for s in t.segments:
            if src.rank != 0 and s.logical.endswith("norm"):
                continue
            by_logical.setdefault(s.logical, []).append((t, s))
    pieces: list[Piece] = []
    for dt in dst.tensors.values():
        for ds in dt.segments:
            for st, ss in by_logical.get(ds.logical, ()):
                r0, r1 = max(ds.row0, ss.row0), min(ds.row0 + ds.rows, ss.row0 + ss.rows)
                c0, c1 = max(ds.col0, ss.col0), min(ds.col0 + ds.cols, ss.col0 + ss.cols)
                if r1 <= r0 or c1 <= c0:
                    continue
                s_off = st.offset + (ss.dst_row + r0 - ss.row0) * st.cols + ss.dst_col + c0 - ss.col0
                d_off = dt.offset + (ds.dst_row + r0 - ds.row0) * dt.cols + ds.dst_col + c0 - ds.col0
                pieces.append(Piece(s_off, d_off, st.cols, dt.cols, r1 - r0, c1 - c0))
    return pieces


@dataclass(frozen=True)
class KVPoolGeometry:
    """[num_blocks][layers][2][heads][block_size][head_dim] bf16 pool of one GPU."""

    num_blocks: int
    n_layers: int
    n_heads: int
    block_size: int
    head_dim: int

    @property
    def block_elems(self) -> int:
        return self.n_layers * 2 * self.n_heads * self.block_size * self.head_dim

    @property
    def layer_stride(self) -> int:          # elements between layers inside a block
        return 2 * self.n_heads * self.block_size * self.head_dim

    def as_tuple(self) -> tuple[int, int, int, int]:
        return (self.n_layers, self.n_heads, self.block_size, self.head_dim)


def kv_geometry(arch: LlamaArch, tp: int, pp: int, num_blocks: int, block_size: int) -> KVPoolGeometry:
    return KVPoolGeometry(num_blocks, arch.num_layers // pp, arch.num_kv_heads // tp, block_size, arch.head_dim)
