"""Shared helpers of the engine tests (not a test module).

* ``run_threads``: SPMD ranks as threads of one process on cuda:0 (ThreadComm).
* ``check_greedy``: greedy token identity against the bf16-faithful oracle.
* ``expected_weight_bytes_sent`` / ``expected_kv_bytes_per_token_sent``: the
  bytes a GPU must send in a P->D transition, computed independently of the
  product's layout code from the placement rules (oracle/kv_layout.py,
  reference reshard.py:98-122, :151-188) — SURVEY.md Appendix A.3.
"""

from __future__ import annotations

import threading

import numpy as np
import torch

from oracle import kv_layout as kvo
from oracle import llama as lo
from paper_2503_06433_b200.specs import HardwareSpec, RingAllReduce


def tiny_hw(n: int, gpu_memory: float = 2e9, host_memory_per_gpu: float = 2e9) -> HardwareSpec:
    return HardwareSpec(num_gpus=n, hbm_bandwidth=8e12, peak_flops=2.25e15, gpu_memory=gpu_memory,
                        host_memory_per_gpu=host_memory_per_gpu, host_link_bandwidth=64e9,
                        allreduce=RingAllReduce(9e11))


def oracle_arch(a) -> lo.Arch:
    return lo.Arch(a.num_layers, a.hidden, a.num_query_heads, a.num_kv_heads, a.head_dim, a.ffn, a.vocab,
                   a.rope_theta, a.rms_eps)


def run_threads(n, fn, timeout=900):
    """Run fn(rank) on n threads; the first failure is re-raised (the other
    ranks' ThreadComm waits time out instead of hanging)."""
    out, errs = [None] * n, []

    def body(r):
        try:
            torch.cuda.set_device(0)
            out[r] = fn(r)
        except BaseException as e:  # noqa: BLE001
            errs.append(e)
            raise

    ts = [threading.Thread(target=body, args=(r,)) for r in range(n)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=timeout)
    if errs:
        raise errs[0]
    if any(t.is_alive() for t in ts):
        raise TimeoutError(f"rank threads still running after {timeout} s")
    return out


def step_logits(worker) -> dict:
    """{(request id, step): fp32 logits} of a run with record_logits: step 0
    is the prefill's last position, step k the k-th decode step's input
    position (the engine logs each recorded forward's row ids)."""
    out, count = {}, {}
    assert len(worker.logit_rows) == len(worker.logit_log)
    for rec, ids in zip(worker.logit_log, worker.logit_rows):
        assert rec.shape[0] == len(ids)
        for j, sid in enumerate(ids):
            k = count.get(sid, 0)
            count[sid] = k + 1
            out[(sid, k)] = rec[j]
    return out


def greedy_margins(arch, reqs, prompts, outputs, tp_prefill, tp_decode, max_pos=256, pp_prefill=1,
                   fold_norm=True, weights=None, gpu_logits=None, pp_decode=1, tp_fold=False):
    """Teacher-forced comparison with the bf16-faithful oracle: per step
    (seq, step, gpu token, oracle token, oracle top-1/top-2 margin, measured
    max |gpu - oracle| logit deviation or None).  ``fold_norm`` mirrors the
    engine default (SSB_FOLD_NORM=1) on the tensor-parallel-1 phases;
    ``pp_prefill`` places the stage boundaries."""
    oracle = lo.LlamaOracle(oracle_arch(arch), seed=0, bf16_faithful=True, max_pos=max_pos,
                            tp_prefill=tp_prefill, tp_decode=tp_decode, fold_norm=fold_norm, pp_prefill=pp_prefill,
                            weights=weights, pp_decode=pp_decode, tp_fold=tp_fold)
    rows = []
    for r, p in zip(reqs, prompts):
        got = outputs[r.id]
        assert len(got) == r.output_len
        exp, logs = oracle.generate(p, r.output_len, forced=got)
        for k, (g, e, lg) in enumerate(zip(got, exp, logs)):
            top2 = torch.topk(lg, 2).values
            dev = None if gpu_logits is None else (gpu_logits[(r.id, k)] - lg).abs().max().item()
            rows.append((r.id, k, g, e, float(top2[0] - top2[1]), dev))
    return rows


# Greedy identity.  The GPU and the bf16-faithful oracle round to bf16 at the
# same points but accumulate in fp32 in different orders (tensor-core MMA vs
# einsum), which flips a few bf16 roundings per step and moves the logits by
# ~0.02 (measured: median 0.018 on configs[0]).  Two tokens whose oracle
# logits are closer than the GPU's deviation on that step are a tie at the
# computation's precision.  A substitution is therefore accepted only when
# the oracle's top-1/top-2 margin is below the GPU-vs-oracle logit deviation
# MEASURED on that very step (tests that record the GPU's logits), else
# below TIE_EPS; every substitution is counted and reported, and at most 1 %
# of the steps may have one.
TIE_EPS = 0.02


def check_greedy(arch, reqs, prompts, outputs, tp_prefill, tp_decode, max_pos=256, pp_prefill=1,
                 fold_norm=True, gpu_logits=None, max_subs=None, weights=None, pp_decode=1, tp_fold=False):
    """Greedy identity against the bf16-faithful oracle (teacher forced).
    ``gpu_logits``: step_logits() of the run.  Returns {"steps",
    "substitutions": [(seq, step, gpu, oracle, margin, deviation)],
    "min_margin", "deviations"}."""
    rows = greedy_margins(arch, reqs, prompts, outputs, tp_prefill, tp_decode, max_pos, pp_prefill, fold_norm,
                          weights, gpu_logits, pp_decode, tp_fold)
    subs = [r for r in rows if r[2] != r[3]]
    for sid, k, g, e, margin, dev in subs:
        bound = TIE_EPS if dev is None else dev
        assert margin <= bound, (f"seq {sid} step {k}: gpu {g} != oracle {e} with oracle margin {margin:.5f} "
                                 f"> {bound:.5f}")
    limit = max(1, len(rows) // 100) if max_subs is None else max_subs
    assert len(subs) <= limit, f"{len(subs)} near-tie substitutions in {len(rows)} steps: {subs}"
    margins = np.array([r[4] for r in rows])
    devs = np.array([r[5] for r in rows if r[5] is not None])
    return {"steps": len(rows), "substitutions": subs, "min_margin": float(margins.min()), "deviations": devs}


def _owned(arch, tp: int, pp: int, gpu: int) -> dict[str, tuple[int, int, int, int]]:
    """Logical rectangles (r0, r1, c0, c1) GPU ``gpu`` of a (tp, pp) replica
    holds: stage layers; Q heads following the rank's KV heads; FFN and
    vocabulary split evenly by rank; norms whole; embedding on stage 0 and
    LM head + final norm on the last stage."""
    stage, rank = divmod(gpu, tp)
    L, h, d, f, v = arch.num_layers, arch.hidden, arch.head_dim, arch.ffn, arch.vocab
    hq, hk = arch.num_query_heads, arch.num_kv_heads
    q0, q1 = rank * hq // tp * d, (rank + 1) * hq // tp * d
    k0, k1 = rank * hk // tp * d, (rank + 1) * hk // tp * d
    f0, f1 = rank * f // tp, (rank + 1) * f // tp
    v0, v1 = rank * v // tp, (rank + 1) * v // tp
    out = {}
    for l in range(stage * L // pp, (stage + 1) * L // pp):
        p = f"L{l}."
        out[p + "attn_norm"] = (0, 1, 0, h)
        out[p + "mlp_norm"] = (0, 1, 0, h)
        out[p + "wq"] = (q0, q1, 0, h)
        out[p + "wk"] = (k0, k1, 0, h)
        out[p + "wv"] = (k0, k1, 0, h)
        out[p + "wo"] = (0, h, q0, q1)
        out[p + "w1"] = (f0, f1, 0, h)
        out[p + "w3"] = (f0, f1, 0, h)
        out[p + "w2"] = (0, h, f0, f1)
    if stage == 0:
        out["embed"] = (v0, v1, 0, h)
    if stage == pp - 1:
        out["head"] = (v0, v1, 0, h)
        out["final_norm"] = (0, 1, 0, h)
    return out


def expected_weight_bytes_sent(arch, src: tuple[int, int], dst: tuple[int, int], gpu: int) -> int:
    """Bytes of weights GPU ``gpu`` sends to the other GPUs of its replica in
    a src=(tp,pp) -> dst=(tp,pp) re-partition whose source holds every
    element once (tp_src = 1: the prefill layouts)."""
    assert src[0] == 1, "unique source ownership only"
    mine = _owned(arch, *src, gpu)
    n = src[0] * src[1]
    total = 0
    for q in range(n):
        if q == gpu:
            continue
        for key, (r0, r1, c0, c1) in _owned(arch, *dst, q).items():
            if key in mine:
                a0, a1, b0, b1 = mine[key]
                total += max(0, min(r1, a1) - max(r0, a0)) * max(0, min(c1, b1) - max(c0, b0))
    return 2 * total


def expected_kv_bytes_per_token_sent(arch, src: tuple[int, int], dst: tuple[int, int], gpu: int) -> int:
    """KV bytes per token position GPU ``gpu`` sends to other GPUs
    (oracle.kv_layout.kv_route_bytes off the diagonal)."""
    m = kvo.kv_route_bytes(arch.num_layers, arch.num_kv_heads, arch.head_dim, 2, src, dst, 1)
    return int(m[gpu].sum() - m[gpu, gpu])


def oracle_weights_from_worker(w, arch, sample_check: bool = True) -> dict:
    """The oracle's logical tensors read back from a single-GPU (tp1.pp1)
    Worker's arena — for shapes whose numpy init would take minutes (the
    8B head and embedding are 525 M elements each).  With ``sample_check``
    three rows of every tensor are first compared bit for bit with the
    oracle's own init (oracle/llama.py init_tensor), so the read-back weights
    ARE the oracle's weights.  Returned as fp32 tensors."""
    names = list(lo.tensor_specs(oracle_arch(arch)).keys())
    specs = lo.tensor_specs(oracle_arch(arch))
    h, d = arch.hidden, arch.head_dim
    nq, nk = arch.num_query_heads, arch.num_kv_heads
    out = {}
    for name in names:
        if name.startswith("L"):
            layer, key = name.split(".", 1)
            p = layer + "."
            if key in ("wq", "wk", "wv"):
                t = w.w(p + "wqkv")
                r0 = {"wq": 0, "wk": nq * d, "wv": (nq + nk) * d}[key]
                r1 = r0 + (nq * d if key == "wq" else nk * d)
                out[name] = t[r0:r1].cpu()
            elif key in ("w1", "w3"):
                t = w.w(p + "w13").view(-1, 2, 32, h)
                out[name] = t[:, 0 if key == "w1" else 1].reshape(-1, h).cpu()
            else:
                out[name] = w.w(p + key).cpu().clone()
        else:
            out[name] = w.w(name).cpu().clone()
        if sample_check:
            t = out[name]
            for i in sorted({0, t.shape[0] // 2, t.shape[0] - 1}):
                exp = lo.init_tensor(0, specs[name], rows=slice(i, i + 1))[0]
                np.testing.assert_array_equal(t[i].float().numpy(), exp, err_msg=f"{name} row {i}")
    return {k: v.float() for k, v in out.items()}
