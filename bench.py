#!/usr/bin/env python
"""bench.py -- throughput of the ADMM hot path (arXiv 1903.10041) on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--workload sweep|phev|toy|horizon|microbench|crossover|qsweep] [--q Q] [--n N]

Default workload = BASELINE.json configs[3], the largest single-GPU config and the
one the north star's ">= 60 % of the HBM roofline" target applies to: the scenario
sweep, PHEV-shaped (m = 2 engine + battery, n = 1000), q = 1e5 scenarios, sharded by
scenario over the ranks (strong scaling: q_total = 1e5 for every N).  One step =
admm_reset + admm_iterate(100): every ADMM iteration runs all §8(a) rows (quartic
build, Algorithm 1, box, demand and capacity couplings, consensus, duals; residuals,
termination test and rho adaptation every 10th iteration).
Metric = element-updates/s = m n q_total x iterations / s (BASELINE.json "metric"),
iterations/s alongside; roofline = algorithmic bytes per iteration (DESIGN.md "Byte
model") / the measured time per launch, against MEASURED_PEAKS.json hbm_gbs.

At N = 1 the line also carries `secondary` measurements of the other configs:
PHEV q = 50 solved to tolerance (configs[1], on-chip engine: latency/sync bound),
horizon n = 1e6 (configs[2]), the 1e8-quartic microbench (configs[4]) and the toy
(configs[0]); plus `cpu_baseline` (the CPU oracle, 1 thread) and
`cpu_baseline_allcore` (its OpenMP build on every affinity core) on a bounded
sample of the headline workload.

Multi-GPU (torchrun, one rank per GPU, NCCL): each rank owns a contiguous scenario
shard; per iteration the library all-gathers 32 doubles (consensus sums, residual
maxima) inside its CUDA graph.  Timing: W warm-up steps; L2 flushed (512 MiB write)
before every timed step; each step bracketed by CUDA events on the solver's
stream; barrier + synchronize around the timed loop; max over ranks.

--impl reference: this tier's reference arm is the CPU oracle (oracle/), timed as
it stands on the host cores (OpenMP build, all affinity cores) on a bounded sample
of the same workload; it imports nothing from paper_1903_10041_b200.
"""

from __future__ import annotations

import argparse
import importlib.util
import json
import os
import platform
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

L2_FLUSH_BYTES = 512 << 20
SWEEP_ITERS = 100  # ADMM iterations per step of the scenario sweep


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="sweep",
                    choices=["sweep", "phev", "toy", "horizon", "microbench", "crossover", "qsweep"])
    ap.add_argument("--q", type=int, default=None,
                    help="scenarios: sweep = q_total (default 1e5), phev = per GPU (default 50)")
    ap.add_argument("--n", type=int, default=None, help="horizon (horizon workload)")
    ap.add_argument("--family", default="C",
                    help="microbench quartic family: C = convex (BASELINE.json configs[4]) or R")
    ap.add_argument("--coeff-bits", type=int, default=64, choices=[64, 32],
                    help="F2: storage precision of a2,a1,b2,b1 (32 = fp32 coefficients, fp64 math)")
    ap.add_argument("--exec", type=int, default=0, choices=[0, 1, 2],
                    help="admm_exec_mode: 0 auto (default), 1 streaming, 2 persistent")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-secondary", action="store_true",
                    help="skip the other configs' lines added to the default N=1 run")
    return ap.parse_args()


def _dist_module():
    """paper_1903_10041_b200/dist.py loaded by path: the reference arm must not import
    the product package (its __init__ loads the CUDA library)."""
    spec = importlib.util.spec_from_file_location(
        "_admm_dist", os.path.join(ROOT, "paper_1903_10041_b200", "dist.py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def _shard_range():
    return _dist_module().shard_range


def _horizon_slice(P, k0, k1):
    """Steps [k0, k1) of every array of a problem (horizon blocks)."""
    import numpy as np

    Q = dict(P)
    for k in ("a2", "a1", "a0", "b2", "b1", "b0"):
        Q[k] = np.ascontiguousarray(P[k][:, :, k0:k1])
    for k in ("lo", "hi", "y"):
        Q[k] = np.ascontiguousarray(P[k][:, k0:k1])
    Q["n"] = k1 - k0
    return Q


# ------------------------------------------------------------------ workloads
def workload(args, rank, world):
    """Per-rank description of the workload: a dict with the shard [j0, j1), the
    problem generator make(j0, q) (synthetic, seeded: scenario j depends on (seed, j)
    only) and the step kind."""
    import synth

    shard_range = _shard_range()
    w = args.workload
    if w == "microbench":
        return dict(kind="quartic", N=100_000_000, family=args.family, cfg="configs[4]",
                    name=f"quartic-minimiser microbench: 1e8 random quartics (family "
                         f"{args.family}), box bounds, fp64 (BASELINE.json configs[4])")
    if w == "sweep":
        q_total = args.q or 100_000
        j0, j1 = shard_range(q_total, rank, world)
        dE = synth.DELTA_E
        return dict(kind="iterate", m=2, n=1000, q_total=q_total, j0=j0, j1=j1, iters=SWEEP_ITERS,
                    make=lambda a, q: synth.phev_problem(1000, q, j0=a), r_bar=1e-6 * dE,
                    sigma_bar=1e-2, cfg="configs[3]", scaling="strong",
                    name=f"scenario sweep PHEV m=2 n=1000 q={q_total} (BASELINE.json configs[3]), "
                         f"{SWEEP_ITERS} fixed ADMM iterations per step")
    if w == "phev":
        qg = args.q or 50
        q_total = qg * world
        j0, j1 = shard_range(q_total, rank, world)
        dE = synth.DELTA_E
        return dict(kind="solve", m=2, n=1000, q_total=q_total, j0=j0, j1=j1,
                    make=lambda a, q: synth.phev_problem(1000, q, j0=a), r_bar=1e-6 * dE,
                    sigma_bar=1e-2, max_iter=20000, cfg="configs[1]", scaling="weak",
                    name=f"PHEV robust energy management m=2 n=1000 q={qg}/GPU, solve to "
                         f"r<1e-6 dE, sigma<1e-2 (BASELINE.json configs[1])")
    if w == "toy":
        P = synth.toy_problem()
        return dict(kind="iterate", m=2, n=10, q_total=1, j0=0, j1=1, iters=200,
                    make=lambda a, q: P, r_bar=1e-6 * P["c"][1], sigma_bar=1e-2,
                    cfg="configs[0]", scaling="weak",
                    name="nominal toy n=10 m=2 q=1, 200 fixed iterations (BASELINE.json configs[0])")
    if w == "horizon":
        # N > 1: horizon blocks (rank r owns a balanced range of the n steps; strong scaling)
        n = args.n or 1_000_000
        P = synth.horizon_problem(n)
        k0, k1 = _dist_module().horizon_range(n, rank, world) if world > 1 else (0, n)
        make = (lambda a, q: P) if world == 1 else (lambda a, q: _horizon_slice(P, k0, k1))
        return dict(kind="solve", m=4, n=n, q_total=1, j0=0, j1=1, make=make, k0=k0, k1=k1,
                    r_bar=1e-6 * P["c"][2], sigma_bar=1e-2, max_iter=20000, cfg="configs[2]",
                    scaling="strong" if world > 1 else "weak", horizon_blocks=world > 1,
                    name=f"horizon sweep m=4 q=1 n={n}, solve to tol (BASELINE.json configs[2])"
                         + (f", horizon blocks over {world} GPUs" if world > 1 else ""))
    raise ValueError(w)


def alg_bytes_per_iter(m, n, q, coeff_bits=64):
    """Algorithmic bytes one sweep must move (SURVEY.md
    §8(d)): per element a2,a1,b2,b1 + x read/write; per cell y + v read/write;
    per (i,k) lo,hi; per row lam,zeta,h,p read+write, sum b0, nu read/write.
    F2 (coeff_bits=32): the four coefficients are 4 bytes each."""
    cb = 4 * (coeff_bits // 8)
    return cb * m * q * n + 8 * (2 * m * q * n + 3 * q * n + 2 * m * n + 11 * m * q)


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def ncu_record(key, kernel):
    """The committed ncu --set full numbers of `kernel` on workload `key`
    (profiles/ncu_metrics.json): dram bytes per launch, fp64-pipe %, source."""
    try:
        d = json.load(open(os.path.join(ROOT, "profiles", "ncu_metrics.json")))
        return d.get(key, {}).get(kernel)
    except Exception:
        return None


def host_info():
    model = platform.processor() or ""
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                model = ln.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    try:
        aff = len(os.sched_getaffinity(0))
    except Exception:
        aff = os.cpu_count()
    return {"cpu_model": model, "cpu_count": os.cpu_count(), "affinity": aff}


class ClockSampler:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, path):
        self.path = path
        self.p = None

    def __enter__(self):
        try:
            self.f = open(self.path, "w")
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        if self.p is not None:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                self.p.kill()
            self.f.close()

    def summary(self, device):
        try:
            rows = [r.split(", ") for r in open(self.path).read().strip().splitlines()]
        except Exception:
            rows = []
        if not any(len(r) >= 9 and r[0].strip() == str(device) for r in rows):
            # timed region shorter than the 100 ms sampling period: one sample right after
            try:
                out = subprocess.run(["nvidia-smi", f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"],
                                     capture_output=True, text=True, timeout=20).stdout
                rows = [r.split(", ") for r in out.strip().splitlines()]
            except Exception:
                return None
        rows = [r for r in rows if len(r) >= 9 and r[0].strip() == str(device)]
        if not rows:
            return None
        sm = sorted(float(r[1]) for r in rows)
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in rows:
            for nm, v in zip(names, r[5:9]):
                if v.strip() == "Active":
                    reasons.add(nm)
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": float(rows[0][2]),
                "samples": len(rows), "reasons": sorted(reasons)}


def _clock_path(rank, tag):
    d = os.path.join(ROOT, "gpurun_out")
    return os.path.join(d if os.path.isdir(d) else "/tmp", f"clocks_{tag}_rank{rank}.csv")


# ---------------------------------------------------------------- our arm
def _pinned_problem(W):
    """This rank's problem in the boundary layout, packed into pinned host tensors
    (f = [a2,a1,a0], g = [b2,b1,b0] as [3][m][q][n]; lo, hi, y, c)."""
    import numpy as np
    import torch

    P = W["make"](W["j0"], W["j1"] - W["j0"])
    m, q, n = P["m"], P["q"], P["n"]
    f = torch.empty((3, m, q, n), dtype=torch.float64).pin_memory()
    g = torch.empty((3, m, q, n), dtype=torch.float64).pin_memory()
    for t, keys in ((f, ("a2", "a1", "a0")), (g, ("b2", "b1", "b0"))):
        for r, k in enumerate(keys):
            t[r].copy_(torch.from_numpy(np.ascontiguousarray(P[k])))
            del P[k]
    pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
    return dict(f=f, g=g, lo=pin(P["lo"]), hi=pin(P["hi"]), y=pin(P["y"]), c=pin(P["c"]), q=q)


def run_ours(args, W, rank, world, local_rank, dist=None, steps=None, warmup=None, e2e=True):
    import numpy as np
    import torch

    import paper_1903_10041_b200 as L

    steps = args.steps if steps is None else steps
    warmup = args.warmup if warmup is None else warmup
    dev = torch.device("cuda", local_rank)
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    if W["kind"] == "quartic":
        return run_quartic(args, W, dev, flush, steps, warmup, e2e)

    m, n, q_total = W["m"], W["n"], W["q_total"]
    H = _pinned_problem(W)
    q_loc = H["q"]
    n_loc = W.get("k1", n) - W.get("k0", 0)
    s = L.AdmmSolver(m, n, q_total, device=local_rank, dist=dist, r_bar=W["r_bar"],
                     sigma_bar=W["sigma_bar"], coeff_bits=args.coeff_bits, exec_mode=args.exec)
    s.set_problem_packed(H["f"], H["g"], H["lo"], H["hi"], H["y"], H["c"])

    def step():
        s.reset()
        if W["kind"] == "solve":
            info = s.solve(W["r_bar"], W["sigma_bar"], W["max_iter"])
            return info["iterations"]
        s.iterate(W["iters"])
        return W["iters"]

    for _ in range(warmup):
        step()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(steps)]
    iters, sweep_ms, call_ms = [], [], []
    clk = ClockSampler(_clock_path(rank, W["cfg"].replace("[", "").replace("]", "")))
    launches0 = s.engine()[1]
    with clk:
        for k in range(steps):
            flush.zero_()
            ev[k][0].record(stream)
            iters.append(step())
            ev[k][1].record(stream)
            tm = s.timing()
            sweep_ms.append(tm[0])
            call_ms.append(tm[1])
        torch.cuda.synchronize()
    engine, launches1 = s.engine()
    if world > 1:
        torch.distributed.barrier()
    step_ms = [a.elapsed_time(b) for a, b in ev]
    t_ms = torch.tensor([sum(step_ms)], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(t_ms, op=torch.distributed.ReduceOp.MAX)
    T = float(t_ms.item()) / 1e3
    tot_iters = int(sum(iters))
    elem = m * n * q_total
    from paper_1903_10041_b200._lib import ENGINE_NAMES

    kname = ENGINE_NAMES.get(engine, str(engine))
    res = dict(value=elem * tot_iters / T, it_per_s=tot_iters / T, T=T, iters=iters,
               step_ms=step_ms, clocks=clk.summary(local_rank), engine=kname,
               gpu_launches=int(launches1 - launches0))
    res["roof"] = roofline(args, W, q_loc, engine, kname, iters, sweep_ms, call_ms, n_loc)
    if e2e and not args.no_e2e:
        res["e2e"] = run_e2e(s, W, H, dev, flush, world, steps, warmup)
    s.close()
    del H
    return res


def roofline(args, W, q_loc, engine, kname, iters, sweep_ms, call_ms, n_loc=None):
    """Dominant kernel's roofline.  Streaming engines (1, 4): one launch = one ADMM
    iteration, HBM-bound: achieved = algorithmic bytes per iteration / measured time
    per launch.  On-chip engines (2, 3, 5): one launch = the whole call with the state
    in shared memory -- latency/sync bound, reported as time per iteration and the
    fp64-pipe utilisation of the committed ncu capture."""
    import numpy as np

    m, n = W["m"], W["n"]
    ab = alg_bytes_per_iter(m, n if n_loc is None else n_loc, q_loc, args.coeff_bits)
    peaks = measured_peaks()
    hbm = peaks.get("hbm_gbs")
    peak = hbm if hbm else 6650.0
    src = "MEASURED_PEAKS.json hbm_gbs (measured)" if hbm else "fallback 6.65 TB/s"
    key = {"configs[3]": f"sweep_q{q_loc}", "configs[1]": "phev", "configs[2]": f"horizon_n{n}",
           "configs[0]": "toy"}.get(W["cfg"], W["cfg"])
    rec = ncu_record(key, kname)
    if engine in (2, 3, 5):
        per_it_us = float(np.mean(call_ms)) * 1e3 / float(np.mean(iters))
        return {"bound": "latency/sync", "kernel": kname, "us_per_iteration": per_it_us,
                "fp64_pipe_pct": rec.get("fp64_pipe_pct") if rec else None,
                "hbm_equivalent_frac": ab / (per_it_us * 1e-6) / 1e9 / peak,
                "traffic": rec.get("dram_bytes") if rec else None,
                "ncu": rec.get("source") if rec else None,
                "note": "one launch runs every iteration of the call with the state in shared "
                        "memory (DRAM traffic ~ the state once per launch): not an HBM roofline; "
                        "hbm_equivalent_frac = algorithmic bytes per iteration / time per iteration "
                        "/ HBM peak, for context only"}
    avg_launch_ms = float(np.mean(sweep_ms))
    achieved = ab / (avg_launch_ms * 1e-3) / 1e9
    return {"bound": "hbm", "kernel": kname, "achieved": achieved, "peak": peak, "unit": "GB/s",
            "peak_source": src, "frac": achieved / peak,
            "traffic": rec.get("dram_bytes") if rec else None,
            "ncu": rec.get("source") if rec else None,
            "alg_bytes_per_launch": ab, "avg_launch_ms": avg_launch_ms,
            "note": "one launch = one ADMM iteration; time per launch = the library's CUDA-event "
                    "time of its sweep graph / iterations (includes the graph's condition node and "
                    "launch gaps: an upper bound on the kernel time)"}


def run_e2e(s, W, H, dev, flush, world, steps, warmup):
    """Same metric through the public API with pinned HOST buffers: per step
    set_problem_packed (H2D of every input) -> iterate/solve -> solution (D2H)."""
    import torch

    x = torch.empty((W["m"], H["q"], W.get("k1", W["n"]) - W.get("k0", 0)), dtype=torch.float64).pin_memory()
    x1 = torch.empty(W["m"], dtype=torch.float64).pin_memory()
    stream = torch.cuda.current_stream(dev)

    def step():
        s.set_problem_packed(H["f"], H["g"], H["lo"], H["hi"], H["y"], H["c"])
        if W["kind"] == "solve":
            it = s.solve(W["r_bar"], W["sigma_bar"], W["max_iter"])["iterations"]
        else:
            s.iterate(W["iters"])
            it = W["iters"]
        s.solution(x, x1)
        return it

    for _ in range(max(1, min(warmup, 2))):
        step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    tot, its = 0.0, 0
    for _ in range(steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        its += step()
        b.record(stream)
        b.synchronize()
        tot += a.elapsed_time(b)
    t = torch.tensor([tot], dtype=torch.float64, device=dev)
    if world > 1:
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    T = float(t.item()) / 1e3
    h2d = sum(int(H[k].numel() * 8) for k in ("f", "g", "lo", "hi", "y", "c"))
    d2h = int(x.numel() * 8 + x1.numel() * 8)
    return {"value": W["m"] * W["n"] * W["q_total"] * its / T, "unit": "element-updates/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "iterations_per_s": its / T,
            "path": "AdmmSolver.set_problem_packed(pinned host) -> iterate/solve -> "
                    "solution(pinned host)"}


def run_quartic(args, W, dev, flush, steps, warmup, e2e):
    import torch

    import paper_1903_10041_b200 as L
    import synth

    N = W["N"]
    A, B, C, D, lo, hi = synth.quartic_family(W["family"], N, device=dev)
    x = torch.empty_like(A)
    stream = torch.cuda.current_stream(dev)
    for _ in range(warmup):
        L.quartic_minimize_batch(A, B, C, D, lo, hi, out=x)
    torch.cuda.synchronize()
    ms = []
    with ClockSampler(_clock_path(0, "configs4")) as clk:
        for _ in range(steps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            L.quartic_minimize_batch(A, B, C, D, lo, hi, out=x)
            b.record(stream)
            b.synchronize()
            ms.append(a.elapsed_time(b))
    T = sum(ms) / 1e3
    peaks = measured_peaks()
    hbm = peaks.get("hbm_gbs", 6650.0)
    avg = T / steps
    achieved = 56 * N / avg / 1e9
    # the library samples the batch on the device (quartic_sample_kernel, one CTA) and runs
    # the per-lane kernel (one branch dominates: family C) or the warp-compacted one (both
    # branches common: family R) -- both are launched, the other returns at once;
    # ADMM_QB_WC=0/1 forces one.  Launches per call: 3 (1 forced).
    forced = os.environ.get("ADMM_QB_WC") in ("0", "1")
    wc = os.environ.get("ADMM_QB_WC") == "1" if forced else W["family"] == "R"
    kname = "quartic_batch_wc_kernel" if wc else "quartic_batch_vec_kernel"
    rec = ncu_record("microbench_" + W["family"], kname)
    res = dict(value=N * steps / T, T=T, iters=[1] * steps, step_ms=ms,
               clocks=clk.summary(dev.index), gpu_launches=steps * (1 if forced else 3), engine=kname,
               roof={"bound": "hbm", "kernel": kname, "achieved": achieved,
                     "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                     "traffic": rec.get("dram_bytes") if rec else None,
                     "ncu": rec.get("source") if rec else None,
                     "alg_bytes_per_launch": 56 * N, "avg_launch_ms": avg * 1e3})
    del A, B, C, D, lo, hi
    if e2e and not args.no_e2e:
        # e2e: host (pinned) coefficients -> device -> minimise -> host
        n_e = 20_000_000
        hs = [t.cpu().pin_memory() for t in synth.quartic_family(W["family"], n_e, device="cpu")]
        xo = torch.empty(n_e, dtype=torch.float64).pin_memory()
        tot = 0.0
        for _ in range(steps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            ds = [h.to(dev, non_blocking=True) for h in hs]
            xd = L.quartic_minimize_batch(*ds)
            xo.copy_(xd, non_blocking=True)
            b.record(stream)
            b.synchronize()
            tot += a.elapsed_time(b)
        res["e2e"] = {"value": n_e * steps / (tot / 1e3), "unit": "quartics/s",
                      "h2d_bytes_per_step": 48 * n_e, "d2h_bytes_per_step": 8 * n_e,
                      "sample": f"{n_e:.0e} quartics per step"}
    return res


# ------------------------------------------------------------ oracle (CPU)
def oracle_rate(W, budget_s=10.0, threads=1):
    """The CPU oracle as it stands on a bounded sample of the same workload: returns
    (value, sample description, seconds, threads).  threads > 1: the OpenMP build."""
    import numpy as np

    import oracle

    omp = threads > 1
    if omp:
        threads = oracle.set_threads(threads)
    if W["kind"] == "quartic":
        import synth

        Ns = int(min(W["N"], max(1e5, budget_s / 1.2e-7 * threads)))
        A, B, C, D, lo, hi = (t.numpy() for t in synth.quartic_family(W["family"], Ns))
        t0 = time.perf_counter()
        oracle.quartic_batch(A, B, C, D, lo, hi, 0, omp=omp)
        dt = time.perf_counter() - t0
        return Ns / dt, f"{Ns:.2e} quartics of family {W['family']}", dt, threads
    m, n = W["m"], W["n"]
    per = 1.9e-7 / threads  # ~190 ns per element-update per thread
    if W["kind"] == "iterate" and W["q_total"] > 64:
        # scenario sweep: the first K iterations on a sample of qs scenario rows (q_total
        # weights, so every row's arithmetic is the full problem's)
        iters = W["iters"]
        qs = int(max(4, min(W["q_total"], budget_s / (per * m * n * iters))))
        P = W["make"](0, qs)
        o = oracle.Oracle(P, oracle.default_params(r_bar=W["r_bar"], sigma_bar=W["sigma_bar"]),
                          q_total=W["q_total"], omp=omp)
        sample = (f"first {iters} ADMM iterations of scenario rows 0..{qs - 1} of the same "
                  f"workload (q_total = {W['q_total']}), {threads} thread(s)")
        elem = m * n * qs
    else:
        P = W["make"](W["j0"], W["j1"] - W["j0"])
        o = oracle.Oracle(P, oracle.default_params(r_bar=W["r_bar"], sigma_bar=W["sigma_bar"]),
                          omp=omp)
        elem = m * n * P["q"]
        iters = max(1, int(budget_s / (elem * per)))
        if W["kind"] == "iterate":
            iters = min(iters, W["iters"])
        sample = (f"first {iters} ADMM iterations of the same workload from the initial state "
                  f"({elem} element-updates each), {threads} thread(s)")
    t0 = time.perf_counter()
    o.run(iters)
    dt = time.perf_counter() - t0
    return elem * iters / dt, sample, dt, threads


def cpu_baselines(W, unit):
    hi = host_info()
    v1, s1, d1, _ = oracle_rate(W, budget_s=10.0, threads=1)
    out = {"cpu_baseline": {"value": v1, "unit": unit, "cores": 1, "kind": "oracle", "sample": s1,
                            "seconds": d1, **hi}}
    nt = hi["affinity"] or 1
    if nt > 1:
        v, s, d, used = oracle_rate(W, budget_s=10.0, threads=nt)
        out["cpu_baseline_allcore"] = {"value": v, "unit": unit, "cores": used,
                                       "kind": "oracle (OpenMP build, liboracle_omp.so)",
                                       "sample": s, "seconds": d, **hi}
    return out


# ------------------------------------------------ F4: paper-faithful protocols
def run_crossover(args):
    """Fig. 1 analogue: N random quartics, CPU (oracle, 1 thread)
    vs GPU with the host<->device copies inside T1..T2 (steps 3a-3c), >= 10
    repetitions averaged; reports the CPU/GPU crossover N."""
    import torch

    import oracle
    import paper_1903_10041_b200 as L
    import synth

    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream(dev)
    reps = max(10, args.steps)
    rows = []
    cpu_rate = None
    for e in range(2, 9):
        N = 10 ** e
        hs = [t.numpy() for t in synth.quartic_family(args.family, N, device="cpu")]
        pin = [torch.from_numpy(h).pin_memory() for h in hs]
        xo = torch.empty(N, dtype=torch.float64).pin_memory()
        ds = [torch.empty(N, dtype=torch.float64, device=dev) for _ in range(6)]
        xd = torch.empty(N, dtype=torch.float64, device=dev)

        def gpu_once():
            for d, h in zip(ds, pin):
                d.copy_(h, non_blocking=True)
            L.quartic_minimize_batch(*ds, out=xd)
            xo.copy_(xd, non_blocking=True)

        for _ in range(3):
            gpu_once()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            gpu_once()
        stream.synchronize()
        gpu_s = (time.perf_counter() - t0) / reps
        if N <= 10 ** 6:
            t0 = time.perf_counter()
            oracle.quartic_batch(*hs, 0)
            cpu_s = time.perf_counter() - t0
            cpu_rate = N / cpu_s
            kind = "measured"
        else:
            cpu_s = N / cpu_rate
            kind = "extrapolated from N = 1e6"
        rows.append({"N": N, "gpu_s": gpu_s, "cpu_s": cpu_s, "speedup": cpu_s / gpu_s,
                     "cpu": kind})
        del ds, xd, pin
    cross = next((r["N"] for r in rows if r["speedup"] >= 1.0), None)
    return rows, cross


def run_qsweep(args):
    """Fig. 3 analogue: PHEV (m=2, n=1000) solved to r_bar =
    1e-6 dE, sigma_bar = 1e-2 for q = 5..500 on the GPU (copy-inclusive: problem
    H2D, solve, solution D2H); CPU = the oracle's measured per-iteration rate on a
    bounded sample x the iterations of the same solve."""
    import numpy as np
    import torch

    import oracle
    import paper_1903_10041_b200 as L
    import synth

    rows = []
    for q in (5, 10, 20, 50, 100, 200, 500):
        P = synth.phev_problem(1000, q)
        r_bar = 1e-6 * P["c"][1]
        s = L.AdmmSolver(2, 1000, q, device=0, r_bar=r_bar)
        pin = lambda a: torch.from_numpy(np.ascontiguousarray(a)).pin_memory()  # noqa: E731
        f = pin(np.stack([P["a2"], P["a1"], P["a0"]]))
        g = pin(np.stack([P["b2"], P["b1"], P["b0"]]))
        lo, hi, y, c = pin(P["lo"]), pin(P["hi"]), pin(P["y"]), pin(P["c"])
        x = torch.empty((2, q, 1000), dtype=torch.float64).pin_memory()
        x1 = torch.empty(2, dtype=torch.float64).pin_memory()
        ts, its, conv = [], 0, None
        for rep in range(max(3, args.steps) + 1):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            s.set_problem_packed(f, g, lo, hi, y, c)
            info = s.solve(r_bar, 1e-2, 50000)
            s.solution(x, x1)
            torch.cuda.synchronize()
            if rep:
                ts.append(time.perf_counter() - t0)
            its = info["iterations"]
            conv = info["status"] == 0
        eng = L._lib.ENGINE_NAMES.get(s.engine()[0])
        s.close()
        o = oracle.Oracle(P, oracle.default_params(r_bar=r_bar))
        k = max(10, min(its, int(2e6 / (2 * 1000 * q))))
        t0 = time.perf_counter()
        o.run(k)
        cpu_it = (time.perf_counter() - t0) / k
        gpu_s = float(np.mean(ts))
        rows.append({"q": q, "iterations": its, "converged": bool(conv), "gpu_s": gpu_s,
                     "engine": eng, "cpu_s_est": cpu_it * its, "cpu_sample_iterations": k,
                     "speedup": cpu_it * its / gpu_s})
    return rows


def main_f4(args):
    if args.workload == "crossover":
        rows, cross = run_crossover(args)
        last = rows[-1]
        line = {"metric": "quartic minimisations/s incl. host<->device copies (Fig. 1 protocol)",
                "value": last["N"] / last["gpu_s"], "unit": "quartics/s", "n_gpus": 1,
                "steps": max(10, args.steps), "warmup": 3, "ms_per_step": last["gpu_s"] * 1e3,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
                "data": f"synthetic random quartics (family {args.family})",
                "config": {"workload": "F4 crossover N = 1e2..1e8 (PAPER.md:206-237)"},
                "table": rows, "crossover_N": cross,
                "paper_context": "GTX 1060 fp32 vs i5-7300HQ: CPU faster for N < 1e3, 30x (4 cores) / "
                                 "210x (1 core /Od) for N > 1e6 (PAPER.md:237)"}
    else:
        rows = run_qsweep(args)
        last = rows[-1]
        line = {"metric": "PHEV solve-to-tolerance time vs q incl. copies (Fig. 3 protocol)",
                "value": last["gpu_s"], "unit": "s per solve (q = 500)", "n_gpus": 1,
                "steps": max(3, args.steps), "warmup": 1, "ms_per_step": last["gpu_s"] * 1e3,
                "higher_is_better": False, "scaling": "weak", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic (seeded PHEV-shaped generator, synth/)",
                "config": {"workload": "F4 q sweep 5..500, n = 1000 (PAPER.md:328-361)"},
                "table": rows,
                "paper_context": "GTX 1060 fp32 vs 4-core i5 /Ox: 10-20x faster (PAPER.md:350)"}
    print(json.dumps(line))


# ------------------------------------------------------------------ lines
def metric_of(W):
    if W["kind"] == "quartic":
        return "quartic minimisations/s (Algorithm 1 + box, fp64)", "quartics/s"
    return ("ADMM element-updates/s (m*n*q x iterations/s; iterations/s alongside)",
            "element-updates/s")


def config_of(args, W, world):
    cfg = {"workload": W["name"], "baseline_config": W["cfg"],
           "l2": "flushed (512 MiB write) before each timed step; inputs > L2",
           "coeff_bits": args.coeff_bits,
           "parallelism": (f"horizon blocks x{world}" if W.get("horizon_blocks") else
                           f"scenario-sharded dp{world}") if world > 1 else "1 GPU"}
    if W["kind"] != "quartic":
        cfg.update(m=W["m"], n=W["n"], q_total=W["q_total"])
    return cfg


def secondary_lines(args, local_rank):
    """The other BASELINE.json configs, measured the same way on this GPU."""
    import argparse as _ap

    out = []
    for wl, extra in (("phev", {}), ("horizon", {"n": 1_000_000}), ("microbench", {"family": "C"}),
                      ("toy", {})):
        a2 = _ap.Namespace(**vars(args))
        a2.workload, a2.q, a2.n = wl, None, extra.get("n")
        a2.family = extra.get("family", args.family)
        W2 = workload(a2, 0, 1)
        r2 = run_ours(a2, W2, 0, 1, local_rank, steps=5 if wl != "microbench" else 10, warmup=3,
                      e2e=False)
        ln = {"workload": W2["name"], "baseline_config": W2["cfg"], "value": r2["value"],
              "unit": metric_of(W2)[1], "ms_per_step": r2["T"] * 1e3 / len(r2["step_ms"]),
              "engine": r2["engine"], "roofline": r2["roof"], "gpu_launches": r2["gpu_launches"],
              "clocks": r2.get("clocks")}
        if W2["kind"] != "quartic":
            ln["iterations_per_s"] = r2["it_per_s"]
            ln["iterations_per_step"] = r2["iters"]
        out.append(ln)
    return out


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        return main_reference(args, rank, world)
    if args.workload in ("crossover", "qsweep"):
        return main_f4(args)

    import torch

    dist = None
    if world > 1:
        torch.cuda.set_device(local_rank)
        torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    torch.cuda.set_device(local_rank)
    W = workload(args, rank, world)
    if world > 1 and W["kind"] != "quartic":
        import paper_1903_10041_b200 as L

        dist = L.make_dist(W["q_total"], horizon=W["n"] if W.get("horizon_blocks") else None)
    res = run_ours(args, W, rank, world, local_rank, dist=dist)
    metric, unit = metric_of(W)
    line = {
        "metric": metric, "value": res["value"], "unit": unit, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": res["T"] * 1e3 / args.steps,
        "higher_is_better": True, "scaling": W.get("scaling", "weak"), "vs_baseline": None,
        "dtype": "f64" if args.coeff_bits == 64 else "f64 (a2,a1,b2,b1 stored f32: F2)",
        "data": "synthetic (seeded PHEV-shaped generator, synth/)",
        "config": config_of(args, W, world),
        "gpu_launches": res["gpu_launches"], "roofline": res["roof"],
    }
    # config is the workload only (identical in the reference arm's line); what ran and how
    # many iterations each step took are reported beside it
    line["engine"] = res["engine"]
    if W["kind"] != "quartic":
        line["iterations_per_step"] = res["iters"]
        line["iterations_per_s"] = res["it_per_s"]
    if "e2e" in res:
        line["e2e"] = res["e2e"]
    if res.get("clocks"):
        line["clocks"] = res["clocks"]
    if world == 1 and args.workload == "sweep" and not args.no_secondary:
        line["secondary"] = secondary_lines(args, local_rank)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line.update(cpu_baselines(W, unit))
    if rank == 0:
        print(json.dumps(line))
    if world > 1:
        torch.distributed.destroy_process_group()


def main_reference(args, rank, world):
    """--impl reference: the CPU oracle (this tier's reference arm), timed as it stands
    on the host cores (OpenMP build on every affinity core); rank 0 only, each step a
    bounded sample of the workload.  Imports nothing from paper_1903_10041_b200."""
    if rank != 0:
        return
    W = workload(args, 0, world)
    metric, unit = metric_of(W)
    nt = host_info()["affinity"] or 1
    for _ in range(args.warmup):
        oracle_rate(W, budget_s=1.0, threads=nt)
    vals, tot = [], 0.0
    sample, used = "", nt
    for _ in range(args.steps):
        v, sample, dt, used = oracle_rate(W, budget_s=3.0, threads=nt)
        vals.append(v)
        tot += dt
    value = sum(vals) / len(vals)
    line = {"impl": "reference", "metric": metric, "value": value, "unit": unit, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": tot * 1e3 / args.steps,
            "higher_is_better": True, "scaling": W.get("scaling", "weak"), "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (seeded PHEV-shaped generator, synth/)",
            "config": config_of(args, W, world),
            "cpu_baseline": {"value": value, "unit": unit, "cores": used,
                             "kind": "oracle (OpenMP build)", "sample": sample, **host_info()},
            "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))


if __name__ == "__main__":
    main()
