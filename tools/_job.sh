timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "decode" 2>&1 | tail -2
timeout 600 python -m pytest tests/test_engine_gpu.py tests/test_shapes_gpu.py -q -x 2>&1 | tail -2
SSB_DECODE_ATTN_VARIANT=1 timeout 600 python tools/ab_bench.py --configs base --tag decode_v1_per_item_ctas
timeout 600 python tools/ab_bench.py --configs base --tag decode_v0_persistent
SSB_DECODE_ATTN_VARIANT=1 timeout 600 python tools/ab_bench.py --configs base --tag decode_v1_per_item_ctas
