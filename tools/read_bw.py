"""Pure-read HBM bandwidth on this GPU (the ceiling decode attention streams
against): torch.sum over an 8 GiB bf16 tensor and amax over an fp32 view,
and the library's bulk-copy read stream (ssb_debug_read_stream) over a sweep
of CTAs per SM / chunk / ring depth; CUDA events, best of 10.  Prints one
JSON line."""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2503_06433_b200 import _lib  # noqa: E402

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
lib = _lib.load()
stream = torch.cuda.current_stream().cuda_stream
for ctas, chunk, stages in ((1, 32768, 6), (2, 32768, 3), (2, 16384, 6), (3, 16384, 4), (4, 16384, 3), (2, 65536, 3),
                            (1, 65536, 3), (4, 8192, 6)):
    def fn():
        rc = lib.ssb_debug_read_stream(x.data_ptr(), x.numel() * 2, ctas, chunk, stages, stream)
        assert rc == 0, lib.ssb_last_error()
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
    res[f"bulk_c{ctas}_k{chunk // 1024}_s{stages}"] = round(x.numel() * 2 / best / 1e6, 1)
print(json.dumps({"read_gbs": res, "bytes": x.numel() * 2}))
