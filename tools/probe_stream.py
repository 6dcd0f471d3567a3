"""Streaming engine smoke: toy + PHEV q=50 via exec_mode=1, prints dev/iter."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_10041_b200 as L, synth
for name, P, m, n, q in [("toy", synth.toy_problem(), 2, 10, 1), ("phev q50", synth.phev_problem(1000, 50), 2, 1000, 50)]:
    s = L.AdmmSolver(m, n, q, r_bar=1e-6 * P["c"][-1], exec_mode=1)
    s.set_problem(P)
    try:
        s.iterate(20)
        print(name, "dev/iter us", s.timing()[0] * 1e3, flush=True)
    except Exception as e:
        print(name, "ERR", e, flush=True)
    s.close()
