python tools/probe_timing.py
ADMM_PERSIST_GRID=1 python tools/probe_timing.py
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 2>&1 | tail -15
