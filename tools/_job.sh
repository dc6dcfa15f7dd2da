timeout 600 python -m pytest tests/test_gemm_gpu.py tests/test_kernels_gpu.py -q -x 2>&1 | tail -3
timeout 900 python tools/bench_kernels.py --what splitk > gpurun_out/kb_splitk4.log 2>&1; tail -2 gpurun_out/kb_splitk4.log | cut -c1-300
