"""ORACLE (test infrastructure only) — CPU restatement of the KV-cache and
weight placement of the reference, used to check the CUDA re-shard path.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
import this module; the product package never does.

Placement follows the reference exactly:
  * GPU ids enumerate replica-major, then pipeline stage, then tensor rank
    (/root/reference/pkg/src/shardsim/reshard.py:6-7, :106-121);
  * stage s holds layers [s*L/pp, (s+1)*L/pp) (reshard.py:101, :114-115);
  * tensor rank r holds KV heads [r*h/tp, (r+1)*h/tp) (reshard.py:102, :116-117);
  * a sequence's KV splits into exactly these (layer range x head range)
    blocks under the prefill config on swap-out and under the decode config on
    swap-in (reshard.py:151-188).

The paged pool of one GPU is [block][local layer][K|V][local head][token][dim]
(DESIGN.md §3); the oracle builds the GLOBAL cache [block][L][2][H][BS][D]
from the source pools and slices it again for the target layout — an
independent statement of the same permutation the product computes as
pairwise (layer x head) rectangle intersections.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Placement:
    gpu: int          # index inside the replica (stage * tp + rank)
    layer_begin: int
    layer_end: int
    head_begin: int
    head_end: int


def placements(num_layers: int, num_kv_heads: int, tp: int, pp: int) -> list[Placement]:
    """Per-GPU (layer, head) ranges of one replica — reshard.py:98-122."""
    if num_layers % pp or num_kv_heads % tp:
        raise ValueError("tp must divide heads and pp must divide layers")
    lp, hr = num_layers // pp, num_kv_heads // tp
    out = []
    for stage in range(pp):
        for rank in range(tp):
            out.append(Placement(stage * tp + rank, stage * lp, (stage + 1) * lp, rank * hr, (rank + 1) * hr))
    return out


def gather_global(pools: list[np.ndarray], num_layers: int, num_kv_heads: int, tp: int, pp: int) -> np.ndarray:
    """Reassemble [NB, L, 2, H, BS, D] from the per-GPU pools of one replica."""
    nb, _, two, _, bs, d = pools[0].shape
    full = np.zeros((nb, num_layers, two, num_kv_heads, bs, d), dtype=pools[0].dtype)
    for pl, pool in zip(placements(num_layers, num_kv_heads, tp, pp), pools):
        full[:, pl.layer_begin : pl.layer_end, :, pl.head_begin : pl.head_end] = pool
    return full


def scatter_global(full: np.ndarray, tp: int, pp: int) -> list[np.ndarray]:
    """Per-GPU pools of one replica for layout (tp, pp)."""
    _, num_layers, _, num_kv_heads, _, _ = full.shape
    return [
        np.ascontiguousarray(full[:, pl.layer_begin : pl.layer_end, :, pl.head_begin : pl.head_end])
        for pl in placements(num_layers, num_kv_heads, tp, pp)
    ]


def reshard_pools(
    pools: list[np.ndarray], num_layers: int, num_kv_heads: int, src: tuple[int, int], dst: tuple[int, int],
    blocks: np.ndarray | None = None,
) -> list[np.ndarray]:
    """KV re-shard of the listed blocks (all if None) from layout src=(tp,pp)
    to dst=(tp,pp); blocks not listed keep their bytes (the product re-shards
    in place, block by block)."""
    full = gather_global(pools, num_layers, num_kv_heads, *src)
    new = scatter_global(full, *dst)
    if blocks is None:
        return new
    out = []
    for old, nw in zip(pools, new):
        o = old.copy().reshape(old.shape[0], -1)
        o[blocks] = nw.reshape(nw.shape[0], -1)[blocks]
        out.append(o.reshape(nw.shape))
    return out


def pack_rectangles(pool: np.ndarray, ids: np.ndarray, peers: list[tuple[int, int, int, int]]) -> list[np.ndarray]:
    """Staging content for each peer rectangle (l0, nl, h0, nh): the
    rectangle of every listed block in order, [n_ids][nl][2][nh][BS][D]."""
    return [
        np.ascontiguousarray(pool[ids][:, l0 : l0 + nl, :, h0 : h0 + nh]).reshape(-1)
        for (l0, nl, h0, nh) in peers
    ]


def kv_route_bytes(num_layers: int, num_kv_heads: int, head_dim: int, bytes_per_param: int,
                   src: tuple[int, int], dst: tuple[int, int], tokens: int) -> np.ndarray:
    """Byte matrix [src gpu, dst gpu] of one sequence's KV crossing the
    layout switch: intersection of the swap-out and swap-in descriptors
    (reshard.py:151-188); row sums equal the swap-out descriptor bytes."""
    a = placements(num_layers, num_kv_heads, *src)
    b = placements(num_layers, num_kv_heads, *dst)
    per_cell = 2 * bytes_per_param * head_dim * tokens
    m = np.zeros((len(a), len(b)), dtype=np.int64)
    for x in a:
        for y in b:
            nl = min(x.layer_end, y.layer_end) - max(x.layer_begin, y.layer_begin)
            nh = min(x.head_end, y.head_end) - max(x.head_begin, y.head_begin)
            if nl > 0 and nh > 0:
                m[x.gpu, y.gpu] = nl * nh * per_cell
    return m
