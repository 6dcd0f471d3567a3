"""Per-iteration device time of each execution engine on the small configs."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if len(sys.argv) == 1:
    for grid in ("0", "1"):
        env = dict(os.environ, ADMM_PERSIST_GRID=grid)
        subprocess.run([sys.executable, __file__, "child"], env=env)
    sys.exit(0)

import paper_1903_10041_b200 as L, synth  # noqa: E402

cases = [("toy", synth.toy_problem(), 2, 10, 1), ("phev q50", synth.phev_problem(1000, 50), 2, 1000, 50),
         ("phev q5", synth.phev_problem(1000, 5), 2, 1000, 5),
         ("horizon 1e4", synth.horizon_problem(10000), 4, 10000, 1)]
for name, P, m, n, q in cases:
    for eng in (1, 2):
        if eng == 1 and os.environ.get("ADMM_PERSIST_GRID") == "1":
            continue
        try:
            s = L.AdmmSolver(m, n, q, r_bar=1e-6 * P["c"][-1], exec_mode=eng)
            s.set_problem(P)
            s.iterate(200)
            s.reset()
            s.iterate(500)
            print(f"{name:12s} engine={'stream' if eng == 1 else 'persist'} grid={os.environ.get('ADMM_PERSIST_GRID')} "
                  f"last={s.last_engine() if hasattr(s, 'last_engine') else '?'} dev/iter {s.timing()[0] * 1e3:8.2f} us", flush=True)
            s.close()
        except Exception as e:  # noqa: BLE001
            print(name, eng, "ERR", e, flush=True)
