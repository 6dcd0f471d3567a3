"""ncu target: PHEV q=50, persistent engine, 200 fixed iterations."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_10041_b200 as L, synth
q = int(os.environ.get("Q", "50")); it = int(os.environ.get("IT", "200"))
P = synth.phev_problem(1000, q)
s = L.AdmmSolver(2, 1000, q, r_bar=1e-6 * P["c"][1], exec_mode=int(os.environ.get("ENG", "2")))
s.set_problem(P)
s.iterate(it)
s.reset()
s.iterate(it)
print("dev/iter us", s.timing()[0] * 1e3)
