timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_engine_gpu.py -q -x 2>&1 | tail -1
SSB_GEMM_NO_TABLE=1 timeout 600 python tools/ab_bench.py --configs base --tag model_only
timeout 600 python tools/ab_bench.py --configs base --tag with_measured_table
SSB_GEMM_NO_TABLE=1 timeout 600 python tools/ab_bench.py --configs base --tag model_only
