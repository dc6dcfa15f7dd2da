"""Multi-process (world_size 2, gloo, CPU) run of the re-shard engine's rank
logic: Worker.reshard_kv and Worker.repartition_weights with the real
torch.distributed all-to-all between two processes.

The CUDA kernels are replaced by byte-exact CPU emulations defined HERE (test
infrastructure), so what is exercised is the SPMD host logic: peer
rectangles, staging offsets, split sizes, the all-to-all and the in-place
re-interpretation of the pool.  Results must equal the oracle bit for bit.
"""

from __future__ import annotations

import os
import socket
import struct
import tempfile

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from oracle import kv_layout as kvo
from oracle import llama as lo

TP_P, PP_P, TP_D, PP_D = 1, 2, 2, 1
NB = 6
BLOCKS = np.array([4, 1, 3], dtype=np.int32)


def _emulate_ops(ops):
    """Patch paper_2503_06433_b200.ops with CPU byte-exact stand-ins."""

    def init_weights(arena, segs, total, seed):
        a = arena.view(torch.int16).numpy()
        for row in segs.numpy():
            dst_off, ld, row0, col0, full_cols, _, rc, ts = (int(x) for x in row)
            rows, cols = rc & 0xFFFFFFFF, (rc >> 32) & 0xFFFFFFFF
            tid = ts & 0xFFFFFFFF
            scale = struct.unpack("<f", struct.pack("<I", (ts >> 32) & 0xFFFFFFFF))[0]
            idx = (np.arange(row0, row0 + rows)[:, None] * full_cols + np.arange(col0, col0 + cols)[None, :])
            v = lo.init_values(seed, tid, idx, scale)
            bits = (v.view(np.uint32) >> 16).astype(np.uint16).view(np.int16)
            for r in range(rows):
                a[dst_off + r * ld : dst_off + r * ld + cols] = bits[r]

    def kv_pack(pool, geo, ids, peers, staging):
        L, H, BS, D = geo
        p = pool.view(torch.int16).numpy().reshape(-1, L, 2, H, BS, D)
        s = staging.view(torch.int16).numpy()
        for l0, nl, h0, nh, off in peers:
            r = np.ascontiguousarray(p[ids.numpy()][:, l0 : l0 + nl, :, h0 : h0 + nh]).reshape(-1)
            s[off // 2 : off // 2 + r.size] = r

    def kv_unpack(pool, geo, ids, peers, staging):
        L, H, BS, D = geo
        p = pool.view(torch.int16).numpy().reshape(-1, L, 2, H, BS, D)
        s = staging.view(torch.int16).numpy()
        idn = ids.numpy()
        for l0, nl, h0, nh, off in peers:
            n = idn.size * nl * 2 * nh * BS * D
            if n:
                p[idn, l0 : l0 + nl, :, h0 : h0 + nh] = s[off // 2 : off // 2 + n].reshape(idn.size, nl, 2, nh, BS, D)

    def copy2d(src, dst, descs, total):
        sb = src.view(torch.uint8).numpy()
        db = dst.view(torch.uint8).numpy()
        for so, do, ss, ds, cum, rr in descs.numpy():
            rows, rb = int(rr) & 0xFFFFFFFF, (int(rr) >> 32) & 0xFFFFFFFF
            for r in range(rows):
                db[do + r * ds : do + r * ds + rb] = sb[so + r * ss : so + r * ss + rb]

    ops.init_weights = init_weights
    ops.kv_reshard_pack = kv_pack
    ops.kv_reshard_unpack = kv_unpack
    ops.copy2d_batched = copy2d


def _rank(rank, port, outdir):
    import torch.distributed as dist

    from paper_2503_06433_b200 import PRESETS, ParallelismConfig
    from paper_2503_06433_b200 import runtime
    from paper_2503_06433_b200.comm import TorchComm

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=2)
    _emulate_ops(runtime.ops)
    arch = PRESETS["tiny"]
    w = runtime.Worker(arch, TorchComm(), 1, torch.device("cpu"), seed=0, max_pos=64)
    # stream the weight re-partition in many chunks (the 8B/70B regime)
    w.RESHARD_CHUNK_BYTES = 200_000
    w.init_weights(ParallelismConfig(TP_P, PP_P, 1))
    np.save(f"{outdir}/arena_p_{rank}.npy", w.state.arena.view(torch.int16).numpy().copy())
    w.alloc_pool(NB)
    rng = np.random.default_rng(100 + rank)
    w.pool.view(torch.int16).copy_(torch.from_numpy(rng.integers(-3000, 3000, w.pool.numel(), dtype=np.int16)))
    np.save(f"{outdir}/pool_before_{rank}.npy", w.pool.view(torch.int16).numpy().copy())
    sent_kv = w.reshard_kv(ParallelismConfig(TP_D, PP_D, 1), BLOCKS, chunk_blocks=2)
    sent_w = w.repartition_weights(ParallelismConfig(TP_D, PP_D, 1))
    np.save(f"{outdir}/pool_after_{rank}.npy", w.pool.view(torch.int16).numpy().copy())
    np.save(f"{outdir}/arena_{rank}.npy", w.state.arena.view(torch.int16).numpy().copy())
    chunks = w._weight_plan(ParallelismConfig(TP_P, PP_P, 1), ParallelismConfig(TP_D, PP_D, 1))[1]
    # and back: TP2 -> PP2 (the norm gains are replicated on both TP ranks;
    # only rank 0 of a stage sends them)
    sent_back = w.repartition_weights(ParallelismConfig(TP_P, PP_P, 1))
    np.save(f"{outdir}/arena_back_{rank}.npy", w.state.arena.view(torch.int16).numpy().copy())
    with open(f"{outdir}/sent_{rank}.txt", "w") as fh:
        fh.write(f"{sent_kv} {sent_w} {sent_back} {chunks}")
    dist.destroy_process_group()


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture(scope="module")
def gloo_run():
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_rank, args=(_free_port(), d), nprocs=2, join=True)
        out = {k: [np.load(f"{d}/{k}_{r}.npy") for r in range(2)]
               for k in ("pool_before", "pool_after", "arena", "arena_p", "arena_back")}
        out["sent"] = [tuple(map(int, open(f"{d}/sent_{r}.txt").read().split())) for r in range(2)]
    return out


def test_kv_reshard_two_processes_bit_exact(gloo_run):
    from paper_2503_06433_b200 import PRESETS

    a = PRESETS["tiny"]
    L, H, BS, D = a.num_layers, a.num_kv_heads, 64, a.head_dim
    before = [p.reshape(NB, L // PP_P, 2, H // TP_P, BS, D) for p in gloo_run["pool_before"]]
    exp = kvo.reshard_pools(before, L, H, (TP_P, PP_P), (TP_D, PP_D), blocks=BLOCKS)
    for r in range(2):
        got = gloo_run["pool_after"][r].reshape(exp[r].shape)
        np.testing.assert_array_equal(got, exp[r])
    # bytes leaving each GPU = (tp-1)/tp of its resident KV
    cell = 2 * BS * D * 2
    per_gpu = BLOCKS.size * (L // PP_P) * (H // TP_P) * cell
    assert all(s[0] == per_gpu // 2 for s in gloo_run["sent"])


def test_weight_repartition_two_processes_bit_exact(gloo_run):
    from paper_2503_06433_b200 import PRESETS
    from paper_2503_06433_b200.layout import weight_layout

    a = PRESETS["tiny"]
    oa = lo.Arch(a.num_layers, a.hidden, a.num_query_heads, a.num_kv_heads, a.head_dim, a.ffn, a.vocab, a.rope_theta)
    specs = lo.tensor_specs(oa)
    for r in range(2):
        wl = weight_layout(a, TP_D, PP_D, r)
        arena = gloo_run["arena"][r]
        for t in wl.tensors.values():
            loc = arena[t.offset : t.offset + t.numel].reshape(t.rows, t.cols)
            for s in t.segments:
                full = lo.init_tensor(0, specs[s.logical])
                bits = (full.view(np.uint32) >> 16).astype(np.uint16).view(np.int16)
                np.testing.assert_array_equal(loc[s.dst_row : s.dst_row + s.rows, s.dst_col : s.dst_col + s.cols],
                                              bits[s.row0 : s.row0 + s.rows, s.col0 : s.col0 + s.cols])


def test_weight_repartition_streams_in_chunks_and_round_trips(gloo_run):
    """The P->D re-partition ran in many chunks; D->P restores the prefill
    arenas bit for bit, and each element crossed once (the replicated norm
    gains are sent by tensor rank 0 only)."""
    from paper_2503_06433_b200 import PRESETS

    a = PRESETS["tiny"]
    for r in range(2):
        np.testing.assert_array_equal(gloo_run["arena_back"][r], gloo_run["arena_p"][r])
    sent_kv, sent_w, sent_back, chunks = zip(*gloo_run["sent"])
    assert min(chunks) > 4
    # TP2 -> PP2 on the 2-layer model: GPU 0 (TP rank 0) sends stage 1 its
    # half of layer 1's matrices and of the LM head, plus layer 1's two norm
    # gains and the final norm (it is its stage's rank 0); GPU 1 sends
    # stage 0 its half of layer 0's matrices and of the embedding, no gains
    h, f, v = a.hidden, a.ffn, a.vocab
    matrices = h * a.qkv_dim + a.num_query_heads * a.head_dim * h + 3 * h * f
    half = matrices // 2 + v * h // 2
    assert sent_back == (2 * (half + 3 * h), 2 * half)
