"""Run the tiny config end to end on one GPU (ThreadComm ranks) and dump the
generated tokens and recorded logits for offline analysis against the oracle."""

from __future__ import annotations

import pickle
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent.parent / "tests"))

from test_engine_gpu import _run_tiny  # noqa: E402

from paper_2503_06433_b200 import ParallelismConfig  # noqa: E402

if __name__ == "__main__":
    name = sys.argv[1] if len(sys.argv) > 1 else "tiny"
    p = ParallelismConfig(*map(int, (sys.argv[2] if len(sys.argv) > 2 else "1,2").split(",")))
    d = ParallelismConfig(*map(int, (sys.argv[3] if len(sys.argv) > 3 else "2,1").split(",")))
    torch.cuda.set_device(0)
    arch, reqs, prompts, res, snaps = _run_tiny(name, p, d)
    out = {"arch": name, "p": (p.tp, p.pp), "d": (d.tp, d.pp), "outputs": res[0][0].outputs,
           "prompts": prompts, "logits": [wk.logit_log for _, wk in res]}
    Path("gpurun_out").mkdir(exist_ok=True)
    with open(f"gpurun_out/dump_{name}_{p.tp}{p.pp}_{d.tp}{d.pp}.pkl", "wb") as fh:
        pickle.dump(out, fh)
    print("ok", {k: v[:6] for k, v in list(res[0][0].outputs.items())[:2]})
