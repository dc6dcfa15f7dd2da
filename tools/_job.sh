timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -3
bash tools/profile.sh launches
ls -la gpurun_out/prof/
