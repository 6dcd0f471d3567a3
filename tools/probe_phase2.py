"""Per-phase cycles of the message-passing cluster kernel (admm_onchip2.cuh).
Dev build: python -c "from paper_1903_10041_b200 import build; build.build(out='paper_1903_10041_b200/libadmm_prof.so', defines=['ADMM_PHASE_PROF'])"
run: ADMM_SO=paper_1903_10041_b200/libadmm_prof.so python tools/probe_phase2.py"""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch  # noqa: F401  (load torch's NCCL first)
import paper_1903_10041_b200 as L, synth
from paper_1903_10041_b200 import _lib

names = ["cons:poll+6h", "cons:k0cell", "cells/pub+tail", "red+send", "row:mbar-wait", "row:update",
         "-", "syncthreads", "row:sums", "row:check"]
cnames = ["pre+publish", "poll", "reduce", "decide", "write"]
who = ["tile0 row", "cons l0", "tile1 row", "tile1 w1"]
cases = [("toy", synth.toy_problem(), 2, 10, 1), ("phev q50", synth.phev_problem(1000, 50), 2, 1000, 50),
         ("phev q5", synth.phev_problem(1000, 5), 2, 1000, 5)]
for name, P, m, n, q in cases:
    s = L.AdmmSolver(m, n, q, r_bar=1e-6 * P["c"][-1], exec_mode=2)
    s.set_problem(P)
    _lib._lib.admm_debug_phase2c(np.zeros(12, dtype=np.uint64).ctypes.data_as(C.POINTER(C.c_ulonglong)))
    s.iterate(500)
    out = np.zeros(40, dtype=np.uint64)
    _lib._lib.admm_debug_phase2(out.ctypes.data_as(C.POINTER(C.c_ulonglong)))
    oc = np.zeros(12, dtype=np.uint64)
    _lib._lib.admm_debug_phase2c(oc.ctypes.data_as(C.POINTER(C.c_ulonglong)))
    print(f"{name}: dev/iter {s.timing()[0]*1e3:.2f} us")
    for b in range(2):
        print(f"   check CTA{b} per check:", " ".join(f"{nm}={v:.0f}" for nm, v in zip(cnames, oc[b * 6:b * 6 + 5].astype(float) / 50)))
    for w in range(4):
        row = out[w * 10:(w + 1) * 10].astype(float) / 500
        print(f"   {who[w]:10s}", " ".join(f"{nm}={v:.0f}" for nm, v in zip(names, row)), f"sum={row.sum():.0f}")
    allp = np.zeros(1024 * 2 * 11, dtype=np.uint64)
    _lib._lib.admm_debug_phase2all(allp.ctypes.data_as(C.POINTER(C.c_ulonglong)))
    allp = allp.reshape(1024, 2, 11)
    plan_T = {"toy": 1, "phev q50": 5, "phev q5": 3}[name]
    G = q * plan_T
    cons = allp[0:G:plan_T, 1, :10].astype(float) / 500   # consensus lanes of the tile-0 CTAs
    order = np.argsort(cons[:, 0])
    print("   rows by consensus poll wait (cycles/iter): min", cons[order[0], 0].round(), "median", np.median(cons[:, 0]).round(), "max", cons[order[-1], 0].round())
    for r in list(order[:3]) + list(order[-2:]):
        b = r * plan_T
        sms = [int(allp[b + t, 0, 10]) for t in range(plan_T)]
        print(f"   row {r:3d} sms {sms} cons:", " ".join(f"{nm}={v:.0f}" for nm, v in zip(names, cons[r]) if v > 0),
              "| row0:", " ".join(f"{nm}={v:.0f}" for nm, v in zip(names, allp[b, 0, :10].astype(float) / 500) if v > 0))
    smids = allp[:G, 0, 10]
    u, c = np.unique(smids, return_counts=True)
    print("   CTAs per SM histogram:", dict(zip(*np.unique(c, return_counts=True))))
    s.close()
