"""ncu target: toy config (one CTA), persistent engine, IT fixed iterations."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1903_10041_b200 as L, synth
P = synth.toy_problem(); it = int(os.environ.get("IT", "200"))
s = L.AdmmSolver(2, 10, 1, r_bar=1e-6 * P["c"][1], exec_mode=2)
s.set_problem(P)
s.iterate(it)
s.reset()
s.iterate(it)
print("dev/iter us", s.timing()[0] * 1e3)
