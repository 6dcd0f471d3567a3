timeout 400 python -m pytest tests/test_gpu_admm.py -q -x --timeout 60 -k "cluster" 2>&1 | tail -1
for f in 0.05 0.1 0.2 0.4 0.6 1.0; do echo "frac $f"; ADMM_TILE0_FRAC=$f timeout 120 python tools/probe_engines.py 2>&1 | grep "persist grid=0"; done
ADMM_TILE0_FRAC=0.1 ADMM_SO=$PWD/tools/libadmm_prof.so timeout 120 python tools/probe_phase.py
