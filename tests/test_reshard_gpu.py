"""KV re-shard pack/unpack kernels: byte-exact against the CPU oracle.

A replica of W GPUs is emulated on one device ("virtual ranks"): every rank
packs its per-peer rectangles, the staging segments are exchanged by plain
device copies (the role NCCL all-to-all plays on real peers) and every rank
unpacks.  The result must equal oracle.kv_layout.reshard_pools bit for bit.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import kv_layout as oracle
from paper_2503_06433_b200 import ops
from paper_2503_06433_b200.reshard import kv_exchange
from paper_2503_06433_b200.specs import ModelSpec, ParallelismConfig

pytestmark = pytest.mark.gpu


def _offsets(rects, n_ids, cell_bytes):
    offs, acc = [], 0
    for r in rects:
        offs.append(acc)
        acc += n_ids * r.cells * cell_bytes
    return offs, acc


@pytest.mark.parametrize(
    "L,H,src,dst",
    [
        (8, 8, (1, 4), (4, 1)),   # PP4 -> TP4
        (8, 8, (4, 1), (1, 4)),   # TP4 -> PP4 (the D -> P direction)
        (8, 8, (2, 2), (4, 1)),   # mixed
        (4, 4, (1, 2), (2, 1)),   # tiny-config shape
        (32, 8, (1, 8), (8, 1)),  # Llama-3-8B PP8 -> TP8 geometry
    ],
)
def test_kv_reshard_virtual_world(cuda, L, H, src, dst):
    model = ModelSpec(num_layers=L, params_per_layer=1024, num_query_heads=2 * H, num_kv_heads=H, head_dim=64)
    tp_s, pp_s = src
    tp_d, pp_d = dst
    W = tp_s * pp_s
    NB, BS, D = 10, 16, 64
    gen = np.random.default_rng(L * 100 + W)
    pools_np = [
        gen.integers(-30000, 30000, size=(NB, L // pp_s, 2, H // tp_s, BS, D), dtype=np.int16) for _ in range(W)
    ]
    ids_np = np.array([7, 2, 9, 0, 4], dtype=np.int32)
    expect = oracle.reshard_pools(pools_np, L, H, src, dst, blocks=ids_np)

    cfg_s = ParallelismConfig(tp_s, pp_s, 1)
    cfg_d = ParallelismConfig(tp_d, pp_d, 1)
    pools = [torch.from_numpy(p).to(cuda) for p in pools_np]
    ids = torch.from_numpy(ids_np).to(cuda)
    cell = 2 * BS * D * 2  # K+V bytes of one (layer, head) of one block
    ex = [kv_exchange(model, cfg_s, cfg_d, g) for g in range(W)]
    send_bufs, send_offs = [], []
    for g in range(W):
        offs, total = _offsets(ex[g].send, len(ids_np), cell)
        buf = torch.empty(total // 2 + 8, dtype=torch.int16, device=cuda)
        peers = [(r.l0, r.nl, r.h0, r.nh, o) for r, o in zip(ex[g].send, offs)]
        geo = (L // pp_s, H // tp_s, BS, D)
        ops.kv_reshard_pack(pools[g], geo, ids, peers, buf)
        send_bufs.append(buf)
        send_offs.append(offs)
        # pack alone must match the oracle's rectangle packing
        exp_rects = oracle.pack_rectangles(pools_np[g], ids_np, [(r.l0, r.nl, r.h0, r.nh) for r in ex[g].send])
        got = buf.cpu().numpy().view(np.int16)
        for r, o, e in zip(ex[g].send, offs, exp_rects):
            np.testing.assert_array_equal(got[o // 2 : o // 2 + e.size], e)
    torch.cuda.synchronize()
    # "all-to-all": segment for g from q = send_bufs[q][send_offs[q][g] : ...]
    for g in range(W):
        offs, total = _offsets(ex[g].recv, len(ids_np), cell)
        recv = torch.empty(total // 2 + 8, dtype=torch.int16, device=cuda)
        for q in range(W):
            n = len(ids_np) * ex[g].recv[q].cells * cell // 2
            assert n == len(ids_np) * ex[q].send[g].cells * cell // 2
            if n:
                recv[offs[q] // 2 : offs[q] // 2 + n].copy_(send_bufs[q][send_offs[q][g] // 2 : send_offs[q][g] // 2 + n])
        peers = [(r.l0, r.nl, r.h0, r.nh, o) for r, o in zip(ex[g].recv, offs)]
        # the dst pool is the same allocation reinterpreted (in-place re-shard)
        dst_view = pools[g].view(NB, L // pp_d, 2, H // tp_d, BS, D)
        ops.kv_reshard_unpack(dst_view, (L // pp_d, H // tp_d, BS, D), ids, peers, recv)
    torch.cuda.synchronize()
    for g in range(W):
        got = pools[g].view(NB, L // pp_d, 2, H // tp_d, BS, D).cpu().numpy()
        np.testing.assert_array_equal(got, expect[g])
