SSB_RESHARD_BULK=1 timeout 600 python -m pytest tests/test_reshard_gpu.py -q -x 2>&1 | tail -1
timeout 300 python tools/bench_reshard.py
SSB_RESHARD_BULK=1 timeout 300 python tools/bench_reshard.py
