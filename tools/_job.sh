timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench6.log 2>&1; tail -1 gpurun_out/bench6.log | cut -c1-300
