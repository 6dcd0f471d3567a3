python tools/probe_timing.py
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 -x 2>&1 | tail -30
