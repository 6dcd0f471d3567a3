"""Per-phase cycles of the barrier cluster kernel (persist_cluster_kernel, selected with
ADMM_CLUSTER_V=1; dev build with -DADMM_PHASE_PROF, ADMM_SO=...).  The message-passing engine
has its own probe, tools/probe_phase2.py."""
import ctypes as C, os, sys
os.environ["ADMM_CLUSTER_V"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch  # noqa: F401  (load torch's NCCL first)
import paper_1903_10041_b200 as L, synth
from paper_1903_10041_b200 import _lib

names = ["cells(rest)", "warp-red", "cons:poll+6h", "cons:k0cell+pub", "cluster.sync", "row-update", "check", "tail-sync"]
for name, P, m, n, q in [("toy", synth.toy_problem(), 2, 10, 1), ("phev q50", synth.phev_problem(1000, 50), 2, 1000, 50),
                         ("phev q5", synth.phev_problem(1000, 5), 2, 1000, 5)]:
    s = L.AdmmSolver(m, n, q, r_bar=1e-6 * P["c"][-1], exec_mode=2)
    print(name, "engine", s.engine() if False else "")
    s.set_problem(P)
    s.iterate(500)
    out = np.zeros(24, dtype=np.uint64)
    _lib._lib.admm_debug_phase(out.ctypes.data_as(C.POINTER(C.c_ulonglong)))
    print(f"{name}: dev/iter {s.timing()[0]*1e3:.2f} us")
    for who in range(3):
        row = out[who * 8:(who + 1) * 8].astype(float) / 500
        print("  ", ["tile0 t0", "cons l0", "tile1 t0"][who], " ".join(f"{nm}={v:.0f}" for nm, v in zip(names, row)), f"sum={row.sum():.0f}")
    s.close()
