"""Timeline of CTA 0 of the prefill attention pair kernel (debug trace,
ssb_debug_attn_trace): runs one launch at 16 x 1024 causal (32 q / 8 kv heads,
d 128) -- or the lengths given -- and prints per-item and per-tile timings of
the producer, MMA issuer and both softmax warpgroups, as JSON lines.

    python tools/attn_trace.py [--lens 1024x16]
"""
from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2503_06433_b200 import _lib, ops  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--lens", default="1024x16")
args = ap.parse_args()
L, n = (int(x) for x in args.lens.split("x"))
lens = [L] * n
nq, nk, d = 32, 8, 128
T = sum(lens)
qkv = torch.randn(T, (nq + 2 * nk) * d, device="cuda").to(torch.bfloat16)
cu = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int32, device="cuda")
out = torch.empty(T, nq * d, dtype=torch.bfloat16, device="cuda")
for _ in range(3):
    ops.prefill_attention(qkv, nq, nk, d, cu, max(lens), out, d ** -0.5)
torch.cuda.synchronize()
cap = 4096
buf = torch.zeros(5 * cap, dtype=torch.int64, device="cuda")
lib = _lib.load()
lib.ssb_debug_attn_trace(buf.data_ptr())
ops.prefill_attention(qkv, nq, nk, d, cu, max(lens), out, d ** -0.5)
torch.cuda.synchronize()
lib.ssb_debug_attn_trace(None)
raw = buf.cpu().numpy().astype(np.uint64).reshape(5, cap)
names = {1: "q_issue", 2: "kv_issue", 3: "q_landed", 4: "k_landed", 10: "pv_issue_A", 11: "pv_issue_B",
         20: "sm_wait_S", 21: "S_ready", 22: "P_written", 23: "O_final", 24: "epi_done"}
ev = []
for role in range(5):
    for x in raw[role]:
        x = int(x)
        if x == 0:
            continue
        ev.append({"role": role, "t": x >> 24, "ev": names.get((x >> 16) & 0xFF, (x >> 16) & 0xFF),
                   "item": (x >> 8) & 0xFF, "j": x & 0xFF})
t0 = min(e["t"] for e in ev)
for e in ev:
    e["t"] = (e["t"] - t0) / 1e3  # us
ev.sort(key=lambda e: e["t"])
# per softmax role: time per tile (S_ready -> P_written), wait for S, per-item boundary gaps
summary = {}
for role, head in ((3, "A"), (4, "B")):
    es = [e for e in ev if e["role"] == role]
    sm, wait, epi, gap = [], [], [], []
    last_p = None
    for a, b in zip(es, es[1:]):
        if a["ev"] == "S_ready" and b["ev"] == "P_written":
            sm.append(b["t"] - a["t"])
        if a["ev"] == "sm_wait_S" and b["ev"] == "S_ready":
            wait.append((b["t"] - a["t"], a["j"]))
        if a["ev"] == "O_final" and b["ev"] == "epi_done":
            epi.append(b["t"] - a["t"])
    ends = [e for e in es if e["ev"] == "epi_done"]
    summary[head] = {"tiles": len(sm), "softmax_us_mean": float(np.mean(sm)), "wait_S_us_first_tile":
                     float(np.mean([w for w, j in wait if j == 0])), "wait_S_us_other": float(np.mean([w for w, j in wait if j > 0] or [0])),
                     "epilogue_us_mean": float(np.mean(epi)), "o_wait_us_mean": float(np.mean(
                         [b["t"] - a["t"] for a, b in zip(es, es[1:]) if a["ev"] == "P_written" and b["ev"] == "O_final"] or [0])),
                     "items": len(ends), "span_us": es[-1]["t"] - es[0]["t"]}
print(json.dumps({"lens": args.lens, "summary": summary}))
for e in ev[:400]:
    print(json.dumps(e))
