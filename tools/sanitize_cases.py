"""Small runs of every engine for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1903_10041_b200 as L, synth

cases = [("toy", synth.toy_problem()), ("phev q3 n200", synth.phev_problem(200, 3)),
         ("random m3 n37 q3", synth.random_problem(3, 37, 3, seed=5)),
         ("random m2 n1025 q2", synth.random_problem(2, 1025, 2, seed=6)),
         # more rows than CTAs and rows of several chunks/tiles: every CTA walks several units
         # (the row loop's and the TMA sweep's slot reuse)
         ("phev q1200 n300", synth.phev_problem(300, 1200)),
         # message-passing cluster engine: several rows of several CTAs, checks every 10
         ("phev q8 n300", synth.phev_problem(300, 8))]
engines = [("stream", 1, {}), ("cluster", 2, {}), ("grid", 2, {"ADMM_PERSIST_GRID": "1"}),
           ("cluster_v1", 2, {"ADMM_CLUSTER_V": "1"}),
           ("cluster_t3w2", 2, {"ADMM_CLUSTER_T": "3", "ADMM_CLUSTER_WARPS": "2"}),
           ("stream_l1", 1, {"ADMM_S2_L": "1"}), ("stream_l2", 1, {"ADMM_S2_L": "2"}),
           ("stream_f32", 1, {}),
           ("stream_legacy", 1, {"ADMM_SWEEP2": "0"}),
           ("stream_fx", 1, {"ADMM_SWEEP_FX": "1", "ADMM_SWEEP2": "0"}),
           ("stream_rl", 1, {"ADMM_SWEEP_RL": "1", "ADMM_SWEEP2": "0"}),
           ("stream_u4", 1, {"ADMM_SWEEP_CPT": "4", "ADMM_SWEEP2": "0"}),
           ("stream_pf", 1, {"ADMM_SWEEP_PF": "1", "ADMM_SWEEP2": "0"}),
           ("stream_rl_f32", 1, {"ADMM_SWEEP_RL": "1", "ADMM_SWEEP2": "0"})]
KEYS = ("ADMM_PERSIST_GRID", "ADMM_CLUSTER_V", "ADMM_CLUSTER_T", "ADMM_CLUSTER_WARPS", "ADMM_SWEEP_FX", "ADMM_SWEEP2", "ADMM_S2_L", "ADMM_SWEEP_RL",
        "ADMM_SWEEP_CPT", "ADMM_SWEEP_PF")
only = os.environ.get("ENGINES")
for name, P in cases:
    for en, mode, env in engines:
        if only and en not in only.split(","):
            continue
        for k in KEYS:
            os.environ.pop(k, None)
        os.environ.update(env)
        s = L.AdmmSolver(P["m"], P["n"], P["q"], r_bar=1e-6 * max(1.0, float(np.nanmax(np.where(np.isfinite(P["c"]), P["c"], 0)))), exec_mode=mode, coeff_bits=32 if en.endswith("_f32") else 64)
        s.set_problem(P)
        try:
            s.iterate(25)
        except Exception as e:  # e.g. the on-chip engine refusing a problem too large for it
            print(name, en, "refused:", str(e)[:80], flush=True)
            s.close()
            continue
        S = s.state()
        print(name, en, L._lib.ENGINE_NAMES[s.engine()[0]], "x finite", bool(np.isfinite(S["x"]).all()), flush=True)
        s.close()
x = L.quartic_minimize_batch(*[__import__("torch").rand(1000, dtype=__import__("torch").float64, device="cuda") + 0.1 for _ in range(4)])
print("quartic ok", bool(__import__("torch").isfinite(x).all()))
