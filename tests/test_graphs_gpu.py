"""Decode steps replayed from CUDA graphs (runtime.Worker._decode_step_graph)
produce exactly the tokens of the eagerly launched steps: single GPU (tiny
and the 8B shape's kernels on 2 layers) and TP2 on two virtual ranks whose
collectives are all peer-memory kernels (fused combine + peer argmax, device
epochs: the only way a TP step can live in a graph).  The graphs must really
have been captured and replayed."""

from __future__ import annotations

import dataclasses

import pytest
import torch

from engine_helpers import run_threads, tiny_hw
from paper_2503_06433_b200 import PRESETS, execute, replay_check
from paper_2503_06433_b200.comm import SoloComm, ThreadComm
from paper_2503_06433_b200.engine import synthetic_prompts
from paper_2503_06433_b200.report import SchedulingPolicy
from paper_2503_06433_b200.runtime import Worker
from paper_2503_06433_b200.specs import ParallelismConfig, Request

pytestmark = pytest.mark.gpu


def _run(arch, cfg_p, cfg_d, reqs, graphs: bool, fused: bool = False, gpu_memory=40e9):
    W = cfg_p.num_gpus
    comms = ThreadComm.create(W) if W > 1 else [SoloComm()]
    prompts = synthetic_prompts(reqs, arch.vocab)

    def body(r):
        dev = torch.device("cuda", 0)
        with torch.cuda.stream(torch.cuda.Stream(dev) if fused else torch.cuda.current_stream(dev)):
            wk = Worker(arch, comms[r], 1, dev, seed=0, max_pos=512)
            wk.cuda_graphs = graphs
            wk.fused_tp = fused
            rep = execute(arch.model_spec(), tiny_hw(W, gpu_memory=gpu_memory), reqs,
                          SchedulingPolicy.TRANSITION_MINIMIZING, cfg_p, cfg_d, arch=arch, prompts=prompts,
                          comm=comms[r], device=dev, worker=wk)
            torch.cuda.current_stream(dev).synchronize()
            replayed = sum(1 for e in wk._graphs.values() if e["graph"] is not None)
            return rep, replayed

    return run_threads(W, body)


@pytest.mark.parametrize("name", ["tiny", "llama3-8b-2l"])
def test_single_gpu_graphs_match_eager(cuda, name):
    arch = PRESETS["tiny"] if name == "tiny" else dataclasses.replace(PRESETS["llama3-8b"], num_layers=2, name=name)
    reqs = [Request(i, 96, 12) for i in range(6)] + [Request(6, 40, 5)]
    cfg = ParallelismConfig(1, 1, 1)
    eager = _run(arch, cfg, cfg, reqs, graphs=False)[0]
    graph = _run(arch, cfg, cfg, reqs, graphs=True)[0]
    assert eager[1] == 0 and graph[1] >= 1, "graphs must have been captured"
    assert replay_check(graph[0])
    assert graph[0].outputs == eager[0].outputs


def test_tp2_fused_graphs_match_eager(cuda):
    arch = PRESETS["tiny"]
    reqs = [Request(i, 64, 12) for i in range(8)]
    cfg_p, cfg_d = ParallelismConfig(1, 2, 1), ParallelismConfig(2, 1, 1)
    eager = _run(arch, cfg_p, cfg_d, reqs, graphs=False, fused=True, gpu_memory=2e9)
    graph = _run(arch, cfg_p, cfg_d, reqs, graphs=True, fused=True, gpu_memory=2e9)
    for r in range(2):
        assert graph[r][1] >= 1, "TP2 decode steps must have been captured"
        assert graph[r][0].outputs == eager[0][0].outputs
