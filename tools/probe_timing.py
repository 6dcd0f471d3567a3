"""Per-iteration timing probe for the PHEV workload (graph vs plain launches)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1903_10041_b200 as L, synth

q = int(os.environ.get("Q", "50")); n = int(os.environ.get("N", "1000"))
P = synth.phev_problem(n, q)
s = L.AdmmSolver(2, n, q, r_bar=1e-6 * P["c"][1])
s.set_problem(P)
for rep in range(3):
    s.reset()
    t = time.perf_counter()
    info = s.solve(1e-6 * P["c"][1], 1e-2, 20000)
    dt = time.perf_counter() - t
    print(f"graph={os.environ.get('ADMM_NO_GRAPH','0')!='1'} solve: {info['iterations']} it, wall {dt*1e3:.2f} ms, "
          f"dev/iter {s.timing()[0]*1e3:.2f} us, call {s.timing()[1]:.2f} ms")
s.reset()
s.iterate(1000)
print(f"iterate(1000): dev/iter {s.timing()[0]*1e3:.2f} us")
