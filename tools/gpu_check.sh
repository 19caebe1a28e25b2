# GPU tests (short) + C5 timing + C5 per-CTA phase trace
timeout 600 python -m pytest tests -q -m gpu -x 2>&1 | tail -4
timeout 120 python tools/quick_c5.py C5 2>&1
bash tools/march_trace.sh 2>&1 | head -5
