timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
SSB_PREFILL_ATTN_SINGLE=1 timeout 600 python tools/ab_bench.py --configs base --tag attn_single_head
timeout 600 python tools/ab_bench.py --configs base --tag attn_pair_heads
