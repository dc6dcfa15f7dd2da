import sys
sys.path.insert(0, "tests")
import torch
from paper_2503_06433_b200 import ParallelismConfig
import test_engine_gpu as T

cfg = ParallelismConfig(1, 1, 1)
runs = {}
for name, fold in (("base", False), ("base2", False), ("fold", True)):
    _, reqs, _, res = T._run_ragged("tiny", cfg, cfg, T.RAGGED, gpu_memory=2e9, record_logits=True, fold_norm=fold)
    runs[name] = res[0]
for name in ("base2", "fold"):
    lb, lf = runs["base"][1], runs[name][1]
    print(name, "records", len(lb), len(lf))
    for i, (a, b) in enumerate(zip(lb, lf)):
        d = (a - b).abs().max().item()
        if d > 1e-3 or i < 3:
            print("  rec", i, tuple(a.shape), "maxdiff", d, "scale", a.abs().max().item())
            if d > 0.5:
                rows = (a - b).abs().amax(1)
                print("   bad rows", (rows > 0.5).nonzero().flatten().tolist()[:20], "of", a.shape[0])
                break
