timeout 1500 python tools/bench_tier.py --arch llama2-13b --prompts 256 --kv-gb 110 --host-gb 110 > gpurun_out/tier13.log 2>&1; grep -v "Warning\|^\[W" gpurun_out/tier13.log | tail -30 | cut -c1-300
