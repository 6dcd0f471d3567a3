for f in 0.03 0.06 0.1 0.2 0.3 0.6; do echo "frac $f"; ADMM_TILE0_FRAC=$f timeout 120 python tools/probe_engines.py 2>&1 | grep "persist grid=0" | grep -v horizon; done
ADMM_TILE0_FRAC=0.06 ADMM_SO=$PWD/tools/libadmm_prof.so timeout 120 python tools/probe_phase.py
