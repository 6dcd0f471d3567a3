"""VERDICT r01 'untested configurations' (a): solve PHEV q=200 (n=1000) to the paper's
thresholds with the CPU oracle (OpenMP build, bitwise equal to the serial one) and
record its iteration count, objective and rho / residual history; tests/ compare the
GPU against the committed record (profiles/r02_q200/oracle_q200.json)."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import oracle, synth

q = int(sys.argv[1]) if len(sys.argv) > 1 else 200
oracle.set_threads(os.cpu_count())
P = synth.phev_problem(1000, q)
dE = P["c"][1]
o = oracle.Oracle(P, oracle.default_params(r_bar=1e-6 * dE), omp=True)
t0 = time.time()
info, hist = o.run(200000, stop_on_converge=True, hist_cap=20001)
dt = time.time() - t0
out = dict(q=q, n=1000, iterations=info["iterations"], status=info["status"], objective=info["objective"],
           rho=info["rho"], seconds=dt, threads=os.cpu_count(),
           hist_cols="iter r sigma rho1..4 r1..r4 s1..s3 conv fac",
           hist=hist.tolist())
json.dump(out, open(os.path.join(ROOT, "profiles", "r02_q200", f"oracle_q{q}.json"), "w"))
print(q, info["iterations"], info["status"], info["objective"], dt)
