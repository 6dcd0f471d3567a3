"""Compare GPU engines with the oracle on PHEV q=50 (fixed iterations): per-array errors and history diffs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_gpu_admm import gpu_run, orc_run, scales, STATE_KEYS
import oracle, synth
q = int(os.environ.get("Q", "50")); iters = int(os.environ.get("IT", "200"))
P = synth.phev_problem(1000, q)
prm = oracle.default_params(r_bar=1e-6 * P["c"][1])
So, _, ho = orc_run(P, prm, iters)
for eng in ("stream", "cluster"):
    Sg, _, hg = gpu_run(P, prm, iters, engine=eng)
    sc = scales(P, So)
    print(eng, {k: f"{np.abs(np.asarray(Sg[k]) - np.asarray(So[k])).max() / sc[k]:.1e}" for k in STATE_KEYS})
    d = np.abs(ho - hg)
    for r in range(len(ho)):
        bad = [(c, ho[r, c], hg[r, c]) for c in range(1, 14) if d[r, c] > 1e-9 * (abs(ho[r, c]) + 1e-12)]
        if bad:
            print("  check", int(ho[r, 0]), [(c, f"{a:.8g}", f"{b:.8g}") for c, a, b in bad][:6])
