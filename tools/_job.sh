timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
SSB_PDL=0 timeout 600 python tools/ab_bench.py --configs base --tag pdl_off
timeout 600 python tools/ab_bench.py --configs base --tag pdl_on
SSB_PDL=0 timeout 600 python tools/ab_bench.py --configs base --tag pdl_off
