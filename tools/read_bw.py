"""Pure-read HBM bandwidth on this GPU (the ceiling decode attention streams
against): torch.sum over an 8 GiB bf16 tensor and amax over an fp32 view,
CUDA events, best of 10.  Prints one JSON line."""
import json

import torch

x = torch.empty(4 << 30, dtype=torch.bfloat16, device="cuda").uniform_()
res = {}
for name, fn in (("sum_bf16", lambda: x.sum(dtype=torch.float32)), ("amax_f32view", lambda: x.view(torch.float32).amax())):
    for _ in range(3):
        fn()
    best = 1e9
    for _ in range(10):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e))
    res[name] = round(x.numel() * 2 / best / 1e6, 1)
print(json.dumps({"read_gbs": res, "bytes": x.numel() * 2}))
