"""Per-phase cycles of the cluster kernel (dev build with -DADMM_PHASE_PROF, ADMM_SO=...)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch  # noqa: F401  (load torch's NCCL first)
import paper_1903_10041_b200 as L, synth
from paper_1903_10041_b200 import _lib

names = ["cells", "warp-red", "syncthreads", "cta-red+dsmem", "cluster.sync", "row-update", "check", "tail-sync"]
for name, P, m, n, q in [("toy", synth.toy_problem(), 2, 10, 1), ("phev q50", synth.phev_problem(1000, 50), 2, 1000, 50),
                         ("phev q5", synth.phev_problem(1000, 5), 2, 1000, 5)]:
    s = L.AdmmSolver(m, n, q, r_bar=1e-6 * P["c"][-1], exec_mode=2)
    s.set_problem(P)
    s.iterate(500)
    out = np.zeros(16, dtype=np.uint64)
    _lib._lib.admm_debug_phase(out.ctypes.data_as(C.POINTER(C.c_ulonglong)))
    print(f"{name}: dev/iter {s.timing()[0]*1e3:.2f} us")
    for who in range(2):
        row = out[who * 8:(who + 1) * 8].astype(float) / 500
        print("  ", ["bulk t0", "cons l0"][who], " ".join(f"{nm}={v:.0f}" for nm, v in zip(names, row)), f"sum={row.sum():.0f}")
    s.close()
