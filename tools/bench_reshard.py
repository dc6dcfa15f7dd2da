"""Re-shard pack/unpack microbenchmark alone (bench.py's reshard_micro)."""
import json
import sys
from pathlib import Path
from types import SimpleNamespace

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import bench  # noqa: E402
from paper_2503_06433_b200 import PRESETS  # noqa: E402

args = SimpleNamespace(prompts=512, input_len=1024, output_len=256)
w = SimpleNamespace(pool=None, device=torch.device("cuda", 0))
r = bench.reshard_microbench(w, PRESETS["llama3-8b"], args, bench._peaks())
for row in r["sweep"]:
    print(json.dumps({k: row[k] for k in ("gpus", "kv_pack_hbm_gbs", "kv_unpack_hbm_gbs", "w_pack_hbm_gbs",
                                          "w_unpack_hbm_gbs", "pack_unpack_s_vs_nvlink_floor")}))
