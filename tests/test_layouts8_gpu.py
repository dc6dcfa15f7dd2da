"""The headline 8-GPU layouts end to end on EIGHT ranks (ThreadComm threads
sharing cuda:0 — the only way to execute them on the single-GPU test box):

* PP8 -> TP8 (BASELINE.json configs[1]'s layout);
* PP4 -> TP4 x DP2 (configs[2] at 8 GPUs: two independent replicas,
  requests assigned round robin, reference sim.py:241-243, :267;
  "routing is within one replica", reshard.py:180-182).

On a head_dim-128 GQA model (8 layers, 8 KV heads, so every tcgen05 path
runs: fused RoPE/K-V append, pair prefill attention, TMA decode attention),
each run is checked against the CPU oracle:

* the event log of every rank passes replay_check, one transition;
* every rank's re-partitioned weight arena is bit-exact with the oracle init;
* every replica's re-sharded KV pool is bit-exact with the oracle's
  re-layout of the pre-transition pools (oracle/kv_layout.py), block by block;
* bytes sent per GPU equal the placement-rule volumes (SURVEY.md A.3 rules);
* greedy tokens of every replica are identical to the bf16-faithful oracle.

The full Llama-3-8B shape at PP8 -> TP8 runs too: bytes per GPU must equal
SURVEY A.3 (14,336 B of KV per token and 1.757 GB of weights on average) and
the KV pool must be bit-exact.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from engine_helpers import (
    check_greedy,
    step_logits,
    expected_kv_bytes_per_token_sent,
    expected_weight_bytes_sent,
    oracle_arch,
    run_threads,
    tiny_hw,
)
from oracle import kv_layout as kvo
from oracle import llama as lo
from paper_2503_06433_b200 import PRESETS, LlamaArch, execute, replay_check
from paper_2503_06433_b200.comm import ThreadComm
from paper_2503_06433_b200.engine import synthetic_prompts
from paper_2503_06433_b200.report import SchedulingPolicy
from paper_2503_06433_b200.runtime import Worker
from paper_2503_06433_b200.specs import ParallelismConfig, Request

pytestmark = pytest.mark.gpu

# head_dim 128, GQA group 2, one KV head per rank at TP8
L8 = LlamaArch("l8-d128", 8, 512, 16, 8, 128, 1024, 2048, rope_theta=500000.0)
BS = 64


def _run(arch, cfg_p, cfg_d, reqs, prompts, gpu_memory=4e9, fused_tp=False, snap_weights=None, record_logits=False):
    """``snap_weights``: ranks whose post-transition arena is copied to the
    host (None: all)."""
    W = cfg_p.num_gpus
    comms = ThreadComm.create(W)
    model = arch.model_spec()
    hw = tiny_hw(W, gpu_memory=gpu_memory)
    snaps: dict = {}

    def body(r):
        dev = torch.device("cuda", 0)
        # the fused TP combine's device barrier needs the ranks' kernels to
        # run concurrently: one stream per virtual rank
        with torch.cuda.stream(torch.cuda.Stream(dev) if fused_tp else torch.cuda.current_stream(dev)):
            wk = Worker(arch, comms[r], cfg_p.dp, dev, seed=0, max_pos=512)
            wk.fused_tp = fused_tp
            wk.tp_fold = False  # the fused combine's bit-identity with the all-reduce path

            def before(w, blocks, cfg_to):
                snaps[(r, "pool_before")] = (w.pool.detach().cpu().clone(), blocks.copy())

            def after(w, blocks, cfg_to):
                snaps[(r, "pool_after")] = w.pool.detach().cpu().clone()
                if snap_weights is None or r in snap_weights:
                    snaps[(r, "arena_after")] = (w.state.arena.detach().cpu().clone(), w.state.weights)

            wk.hooks = {"before_reshard": before, "after_reshard": after}
            rep = execute(model, hw, reqs, SchedulingPolicy.TRANSITION_MINIMIZING, cfg_p, cfg_d, arch=arch,
                          prompts=prompts, comm=comms[r], device=dev, worker=wk, record_logits=record_logits)
            torch.cuda.current_stream(dev).synchronize()
            if fused_tp:
                assert wk._tp_arenas and all(a.usable for a in wk._tp_arenas.values())
            return rep, wk.replica, wk.gpu, (step_logits(wk) if record_logits else None)

    return run_threads(W, body), snaps


def _bf16_bits(x: np.ndarray) -> np.ndarray:
    """bf16 bit patterns (int16) of bf16-representable float32 values."""
    return (np.ascontiguousarray(x, dtype=np.float32).view(np.uint32) >> 16).astype(np.uint16).view(np.int16)


def _check_weights(arch, snaps, ranks, full_rows: bool = True):
    """Every segment of every rank's arena equals, bit for bit, the oracle's
    init of that logical rectangle (three sampled rows per segment when
    ``full_rows`` is False: the 8B shape's tensors take minutes in numpy)."""
    specs = lo.tensor_specs(oracle_arch(arch))
    full: dict = {}
    for r in ranks:
        arena, wl = snaps[(r, "arena_after")]
        bits = arena.view(torch.int16).numpy()
        for t in wl.tensors.values():
            local = bits[t.offset : t.offset + t.numel].reshape(t.rows, t.cols)
            for s in t.segments:
                if full_rows:
                    if s.logical not in full:
                        full[s.logical] = _bf16_bits(lo.init_tensor(0, specs[s.logical]))
                    exp = full[s.logical][s.row0 : s.row0 + s.rows, s.col0 : s.col0 + s.cols]
                    got = local[s.dst_row : s.dst_row + s.rows, s.dst_col : s.dst_col + s.cols]
                    np.testing.assert_array_equal(got, exp, err_msg=f"rank {r} {t.key} {s.logical}")
                    continue
                for i in sorted({0, s.rows // 2, s.rows - 1}):
                    row = lo.init_tensor(0, specs[s.logical], rows=slice(s.row0 + i, s.row0 + i + 1))[0]
                    exp = _bf16_bits(row[s.col0 : s.col0 + s.cols])
                    got = local[s.dst_row + i, s.dst_col : s.dst_col + s.cols]
                    np.testing.assert_array_equal(got, exp, err_msg=f"rank {r} {t.key} {s.logical} row {i}")


def _check_pools(arch, snaps, ranks, cfg_p, cfg_d):
    """The replica's pools after the transition equal the oracle's re-layout
    of its pools before it, on every re-sharded block."""
    L, H, D = arch.num_layers, arch.num_kv_heads, arch.head_dim
    before = [snaps[(r, "pool_before")] for r in ranks]
    blocks = before[0][1]
    assert all(np.array_equal(b[1], blocks) for b in before), "ranks of a replica re-shard the same blocks"
    pools = [b[0].view(torch.int16).numpy().reshape(-1, L // cfg_p.pp, 2, H // cfg_p.tp, BS, D) for b in before]
    expect = kvo.reshard_pools(pools, L, H, (cfg_p.tp, cfg_p.pp), (cfg_d.tp, cfg_d.pp), blocks=blocks)
    for g, r in enumerate(ranks):
        got = snaps[(r, "pool_after")].view(torch.int16).numpy().reshape(expect[g].shape)
        np.testing.assert_array_equal(got[blocks], expect[g][blocks], err_msg=f"rank {r}")
    return blocks


def _check_bytes(arch, rep, gpu, cfg_p, cfg_d, n_blocks):
    src, dst = (cfg_p.tp, cfg_p.pp), (cfg_d.tp, cfg_d.pp)
    kv = expected_kv_bytes_per_token_sent(arch, src, dst, gpu) * BS * n_blocks
    w = expected_weight_bytes_sent(arch, src, dst, gpu)
    assert rep.measured["kv_bytes_sent"] == kv, (gpu, rep.measured["kv_bytes_sent"], kv)
    assert rep.measured["weight_bytes_sent"] == w, (gpu, rep.measured["weight_bytes_sent"], w)
    assert rep.measured["reshard_bytes_sent"] == kv + w


LENS = [(64, 8), (100, 5), (17, 12), (128, 3), (1, 6), (65, 9), (33, 7), (90, 4)]


@pytest.fixture(scope="module")
def pp8_tp8(cuda):
    reqs = [Request(i, a, b) for i, (a, b) in enumerate(LENS)]
    prompts = synthetic_prompts(reqs, L8.vocab)
    cfg_p, cfg_d = ParallelismConfig(1, 8, 1), ParallelismConfig(8, 1, 1)
    res, snaps = _run(L8, cfg_p, cfg_d, reqs, prompts, record_logits=True)
    return reqs, prompts, cfg_p, cfg_d, res, snaps


def test_pp8_tp8_replay_and_schedule(pp8_tp8):
    reqs, _, _, _, res, _ = pp8_tp8
    for rep, replica, _, _ in res:
        assert replica == 0
        assert replay_check(rep), replay_check(rep).violation
        assert rep.transitions == 1
        assert rep.config["cfg_p"] == "tp1.pp8.dp1" and rep.config["cfg_d"] == "tp8.pp1.dp1"
    # every rank saw the same schedule (SPMD) and the same tokens
    logs = [[(e.kind, e.seq_id) for e in rep.event_log] for rep, _, _, _ in res]
    assert all(lg == logs[0] for lg in logs)
    assert all(rep.outputs == res[0][0].outputs for rep, _, _, _ in res)


def test_pp8_tp8_weights_bit_exact(pp8_tp8):
    _check_weights(L8, pp8_tp8[5], range(8))


def test_pp8_tp8_kv_bit_exact_and_bytes(pp8_tp8):
    reqs, _, cfg_p, cfg_d, res, snaps = pp8_tp8
    blocks = _check_pools(L8, snaps, range(8), cfg_p, cfg_d)
    assert blocks.size == sum(-(-(a + b) // BS) for a, b in LENS)
    for rep, _, gpu, _ in res:
        _check_bytes(L8, rep, gpu, cfg_p, cfg_d, blocks.size)


def test_pp8_tp8_greedy_tokens(pp8_tp8):
    reqs, prompts, _, _, res, _ = pp8_tp8
    check_greedy(L8, reqs, prompts, res[0][0].outputs, 1, 8, max_pos=512, pp_prefill=8, gpu_logits=res[7][3])


@pytest.fixture(scope="module")
def pp4_tp4_dp2(cuda):
    lens = LENS + [(50, 6), (77, 2)]
    reqs = [Request(i, a, b) for i, (a, b) in enumerate(lens)]
    prompts = synthetic_prompts(reqs, L8.vocab)
    cfg_p, cfg_d = ParallelismConfig(1, 4, 2), ParallelismConfig(4, 1, 2)
    res, snaps = _run(L8, cfg_p, cfg_d, reqs, prompts, record_logits=True)
    return reqs, prompts, cfg_p, cfg_d, res, snaps


def test_dp2_replicas_split_round_robin(pp4_tp4_dp2):
    reqs, _, _, _, res, _ = pp4_tp4_dp2
    for rank, (rep, replica, gpu, _) in enumerate(res):
        assert (replica, gpu) == divmod(rank, 4)
        assert replay_check(rep), replay_check(rep).violation
        assert rep.transitions == 1
        # each replica decodes exactly its round-robin share (sim.py:267)
        assert set(rep.outputs) == {r.id for i, r in enumerate(reqs) if i % 2 == replica}
        # the event log covers every replica (gpu_id = replica index, sim.py:101)
        gpus = {e.gpu_id for e in rep.event_log if e.kind == "prefill_complete"}
        assert gpus == {0, 1}
    logs = [[(e.kind, e.seq_id, e.gpu_id) for e in rep.event_log] for rep, _, _, _ in res]
    assert all(lg == logs[0] for lg in logs)


def test_dp2_weights_and_kv_bit_exact(pp4_tp4_dp2):
    _, _, cfg_p, cfg_d, res, snaps = pp4_tp4_dp2
    _check_weights(L8, snaps, range(8))
    for replica in range(2):
        ranks = range(4 * replica, 4 * replica + 4)
        blocks = _check_pools(L8, snaps, ranks, cfg_p, cfg_d)
        for r in ranks:
            rep, _, gpu, _ = res[r]
            _check_bytes(L8, rep, gpu, cfg_p, cfg_d, blocks.size)


def test_dp2_greedy_tokens(pp4_tp4_dp2):
    reqs, prompts, _, _, res, _ = pp4_tp4_dp2
    for replica in range(2):
        mine = [(r, p) for i, (r, p) in enumerate(zip(reqs, prompts)) if i % 2 == replica]
        out = res[4 * replica][0].outputs
        check_greedy(L8, [r for r, _ in mine], [p for _, p in mine], out, 1, 4, max_pos=512, pp_prefill=4,
                     gpu_logits=res[4 * replica + 3][3])


def test_pp8_tp8_fused_combine_same_tokens(pp8_tp8):
    """TP8 decode with the fused peer-memory combine (8 virtual ranks, one
    stream each) produces the same tokens as the all-reduce path."""
    reqs, prompts, cfg_p, cfg_d, res, _ = pp8_tp8
    fused, _ = _run(L8, cfg_p, cfg_d, reqs, prompts, fused_tp=True, snap_weights=())
    assert fused[0][0].outputs == res[0][0].outputs
    assert replay_check(fused[0][0])


def test_llama3_8b_pp8_tp8_volumes(cuda):
    """Full Llama-3-8B shape, PP8 -> TP8 on 8 virtual ranks: the bytes every
    GPU sends equal SURVEY.md A.3 (KV 14,336 B per token; weights 2.447 GB
    from the first and last stage, 1.527 GB from the others, 1.757 GB on
    average), the KV pool is bit-exact with the oracle re-layout, and the
    weights are bit-exact on sampled rows of every segment."""
    arch = PRESETS["llama3-8b"]
    reqs = [Request(i, 64, 4) for i in range(4)]
    prompts = synthetic_prompts(reqs, arch.vocab)
    cfg_p, cfg_d = ParallelismConfig(1, 8, 1), ParallelismConfig(8, 1, 1)
    res, snaps = _run(arch, cfg_p, cfg_d, reqs, prompts, gpu_memory=8e9, snap_weights=(0, 3, 7))
    assert all(replay_check(rep) for rep, _, _, _ in res)
    blocks = _check_pools(arch, snaps, range(8), cfg_p, cfg_d)
    per_tok = [expected_kv_bytes_per_token_sent(arch, (1, 8), (8, 1), g) for g in range(8)]
    assert per_tok == [14336] * 8
    w = [res[g][0].measured["weight_bytes_sent"] for g in range(8)]
    assert abs(sum(w) / 8 - 1.757e9) < 1e6
    for rep, _, gpu, _ in res:
        _check_bytes(arch, rep, gpu, cfg_p, cfg_d, blocks.size)
    _check_weights(arch, snaps, [0, 3, 7], full_rows=False)
