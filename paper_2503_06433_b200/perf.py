"""The reference's analytic cost model, kept as the PREDICTION the real
kernels are compared against.

Restates /root/reference/pkg/src/shardsim/perf.py: the five per-layer terms
(weight traffic :59-65, attention traffic :68-89, linear/attention compute
:92-111 with the reference's unconventional d^2 attention factor :9-11,
all-reduce :114-122), roofline/additive composition :125-137,
layer_time / layer_time_batch :140-184, stage_quantum / stage_time
:187-218 and throughput_inverse :221-236.  The engine reports
``predicted`` phase times from it beside the measured ones.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

from .report import Mode
from .specs import HardwareSpec, ModelSpec, ParallelismConfig

from enum import Enum


class Phase(Enum):
    PREFILL = "prefill"
    DECODE = "decode"


@dataclass(frozen=True)
class CostBreakdown:
    t_dm_linear: float
    t_dm_attn: float
    t_comp_linear: float
    t_comp_attn: float
    t_comm: float
    layer_time: float
    mode: Mode

    def as_dict(self) -> dict:
        return {"t_dm_linear": self.t_dm_linear, "t_dm_attn": self.t_dm_attn, "t_comp_linear": self.t_comp_linear,
                "t_comp_attn": self.t_comp_attn, "t_comm": self.t_comm, "layer_time": self.layer_time,
                "mode": self.mode.value}


def linear_dm_time(model: ModelSpec, hw: HardwareSpec, cfg: ParallelismConfig) -> float:
    """Per-layer weight bytes over HBM, sharded only by tp."""
    return model.bytes_per_param * model.params_per_layer / (hw.hbm_bandwidth * cfg.tp)


def attn_dm_time(model: ModelSpec, hw: HardwareSpec, cfg: ParallelismConfig, batch: float, seq_len: float,
                 phase: Phase) -> float:
    if batch <= 0:
        return 0.0
    per_token_heads = (model.num_query_heads + 2 * model.num_kv_heads) if phase is Phase.PREFILL \
        else 2 * model.num_kv_heads
    return model.bytes_per_param * batch * seq_len * per_token_heads * model.head_dim / (hw.hbm_bandwidth * cfg.tp)


def compute_time(model: ModelSpec, hw: HardwareSpec, cfg: ParallelismConfig, batch: float, seq_len: float,
                 phase: Phase) -> tuple[float, float]:
    if batch <= 0:
        return 0.0, 0.0
    dd = model.head_dim * model.head_dim
    rate = hw.peak_flops * cfg.tp
    if phase is Phase.PREFILL:
        return (2.0 * model.params_per_layer * batch * seq_len / rate,
                batch * model.num_query_heads * seq_len * seq_len * dd / rate)
    return 2.0 * model.params_per_layer * batch / rate, 2.0 * batch * model.num_query_heads * seq_len * dd / rate


def allreduce_time(model: ModelSpec, hw: HardwareSpec, cfg: ParallelismConfig, tokens: float) -> float:
    if cfg.tp == 1 or tokens <= 0:
        return 0.0
    return tokens * model.activation_bytes_per_token * model.allreduces_per_layer / hw.allreduce_bandwidth(cfg.tp)


def _compose(dml, dma, cl, ca, comm, mode: Mode) -> CostBreakdown:
    total = (max(dml, cl) + max(dma, ca) + comm) if mode is Mode.ROOFLINE else (dml + cl + dma + ca + comm)
    return CostBreakdown(dml, dma, cl, ca, comm, total, mode)


def layer_time(model, hw, cfg, batch, seq_len, phase, mode=Mode.ROOFLINE) -> CostBreakdown:
    cl, ca = compute_time(model, hw, cfg, batch, seq_len, phase)
    tokens = batch * seq_len if phase is Phase.PREFILL else batch
    return _compose(linear_dm_time(model, hw, cfg), attn_dm_time(model, hw, cfg, batch, seq_len, phase), cl, ca,
                    allreduce_time(model, hw, cfg, tokens), mode)


def layer_time_batch(model, hw, cfg, seq_lens: Sequence[int], phase, mode=Mode.ROOFLINE) -> CostBreakdown:
    dma = cl = ca = tokens = 0.0
    for s in seq_lens:
        dma += attn_dm_time(model, hw, cfg, 1, s, phase)
        a, b = compute_time(model, hw, cfg, 1, s, phase)
        cl += a
        ca += b
        tokens += s if phase is Phase.PREFILL else 1
    return _compose(linear_dm_time(model, hw, cfg), dma, cl, ca, allreduce_time(model, hw, cfg, tokens), mode)


def stage_quantum(model, hw, cfg, micro_batch, seq_len, phase, mode=Mode.ROOFLINE) -> float:
    return model.num_layers / cfg.pp * layer_time(model, hw, cfg, micro_batch, seq_len, phase, mode).layer_time


def stage_time(model, hw, cfg, global_batch, seq_len, phase, mode=Mode.ROOFLINE) -> float:
    if global_batch < 0:
        raise ValueError("global_batch must be non-negative")
    return stage_quantum(model, hw, cfg, global_batch / (cfg.pp * cfg.dp), seq_len, phase, mode)


def throughput_inverse(model, hw, cfg, global_batch, seq_len, phase, mode=Mode.ROOFLINE) -> float:
    if global_batch <= 0:
        raise ValueError("global_batch must be >= 1")
    return stage_time(model, hw, cfg, global_batch, seq_len, phase, mode) / (global_batch / cfg.pp)


def predict_phases(model: ModelSpec, hw: HardwareSpec, cfg_p: ParallelismConfig, cfg_d: ParallelismConfig,
                   input_len: int, output_len: int, prompts: int, mode: Mode = Mode.ROOFLINE) -> dict:
    """Reference-model prediction of one offline batch that fits the GPU tier:
    prefill one sequence per micro-batch (sim.py:371-381), decode rounds of
    ceil(n/pp) with ctx = max in chunk (sim.py:525-535)."""
    per_replica = -(-prompts // cfg_p.dp)
    if cfg_p.pp > 1:
        q = model.num_layers / cfg_p.pp * layer_time_batch(model, hw, cfg_p, [input_len], Phase.PREFILL, mode).layer_time
        prefill = per_replica * q + (cfg_p.pp - 1) * q
    else:
        prefill = model.num_layers * layer_time_batch(model, hw, cfg_p, [input_len] * per_replica, Phase.PREFILL,
                                                       mode).layer_time
    decode = 0.0
    chunk = -(-per_replica // cfg_d.pp)
    for k in range(output_len):
        ctx = input_len + k + 1
        q = model.num_layers / cfg_d.pp * layer_time_batch(model, hw, cfg_d, [ctx] * chunk, Phase.DECODE,
                                                           mode).layer_time
        decode += q * (cfg_d.pp if k == 0 else -(-per_replica // chunk))
    return {"prefill_s": prefill, "decode_s": decode}
