"""Record every op output of a 1-GPU tiny prefill (one prompt) for offline
comparison with the oracle's intermediates."""

from __future__ import annotations

import pickle
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2503_06433_b200 import PRESETS, ops  # noqa: E402
from paper_2503_06433_b200 import runtime as rt  # noqa: E402
from paper_2503_06433_b200.comm import SoloComm  # noqa: E402
from paper_2503_06433_b200.specs import ParallelismConfig  # noqa: E402

rec = []


def wrap(name):
    fn = getattr(ops, name)

    def inner(*a, **k):
        out = fn(*a, **k)
        torch.cuda.synchronize()
        if name == "rope_kv_append":
            rec.append((name, a[0].detach().float().cpu().clone()))
        elif out is not None:
            rec.append((name, out.detach().float().cpu().clone()))
        return out

    return inner


for n in ["gemm", "rmsnorm", "rope_kv_append", "prefill_attention", "embedding"]:
    setattr(rt.ops, n, wrap(n))

arch = PRESETS["tiny"]
dev = torch.device("cuda", 0)
w = rt.Worker(arch, SoloComm(), 1, dev, seed=0, max_pos=256)
w.init_weights(ParallelismConfig(1, 1, 1))
w.alloc_pool(4)
prompt = (np.arange(64) * 37 + 11) % arch.vocab
toks = torch.tensor(prompt, dtype=torch.int32, device=dev)
first = torch.zeros(1, dtype=torch.int32, device=dev)
tables = np.array([[0, 1]], dtype=np.int32)
w.prefill(toks, np.array([0, 64], dtype=np.int32), tables, first)
torch.cuda.synchronize()
Path("gpurun_out").mkdir(exist_ok=True)
pickle.dump({"prompt": prompt, "rec": rec, "first": int(first.item())}, open("gpurun_out/debug_layers.pkl", "wb"))
print("recorded", [r[0] for r in rec])
