# GPU tests (short) + C5 timing
timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -3
timeout 120 python tools/quick_c5.py C5 2>&1 | grep status
