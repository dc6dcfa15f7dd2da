timeout 300 python tools/debug_split.py 2>&1 | grep -c "err=0.0[0-9]"
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -4
