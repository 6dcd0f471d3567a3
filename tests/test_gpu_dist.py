"""The multi-GPU code path of the library on one GPU.

A non-NULL admm_dist always runs the collective path -- at world = 1 a one-rank
NCCL communicator -- so these tests execute, against the CPU oracle, exactly the
device code the N > 1 runs use:
  * scenario sharding (ADMM_SHARD_SCENARIOS): the sweep writes its per-rank
    aggregates, ncclAllGather inside the CUDA graph, finalize_kernel reduces them
    in rank order (consensus (6c), residuals, rho), the host polls once per body;
  * horizon blocks (ADMM_SHARD_HORIZON): the sweep leaves its exact fixed-point
    row sums and dg extrema, ncclAllReduce (u64 sum / max) + ncclAllGather, and
    hz_rows_kernel finalises every row ((6b), (6g), (6d), (6i)) and the check.
The two-rank algebra of both partitions is pinned on the CPU by
tests/test_dist_gloo.py (oracle on gloo)."""

import numpy as np
import pytest

import oracle
import synth
from test_gpu_admm import check_hist, compare_states

pytestmark = pytest.mark.gpu


def _lib():
    import paper_1903_10041_b200 as L

    return L


def dist_run(P, params, iters, horizon=False, mode="iterate", r_bar=None, sigma_bar=None,
             max_iter=None):
    L = _lib()
    uid = L._lib.admm_nccl_unique_id()
    d = L.dist_for(0, 1, P["q"], uid, horizon=P["n"] if horizon else None)
    s = L.AdmmSolver(P["m"], P["n"], P["q"], dist=d, rho=params["rho0"], tau=params["tau"],
                     hi_ratio=params["hi_ratio"], lo_ratio=params["lo_ratio"],
                     r_bar=params["r_bar"], sigma_bar=params["sigma_bar"],
                     check_every=params["check_every"], adapt_rho=params["adapt_rho"],
                     rescale_duals=params["rescale_duals"], box_mode=params["box_mode"])
    s.set_problem(P)
    info = None
    if mode == "iterate":
        s.iterate(iters)
    else:
        info = s.solve(r_bar, sigma_bar, max_iter)
    S = s.state()
    x, x1, sol = s.solution()
    hist = s.history()
    eng = L._lib.ENGINE_NAMES.get(s.engine()[0])
    s.close()
    return S, (sol if info is None else {**sol, **info}), hist, eng


def orc(P, params, iters, solve=False):
    o = oracle.Oracle(P, params)
    info, hist = o.run(iters, stop_on_converge=solve)
    return o.state(), info, hist


CASES = [
    ("toy", lambda: synth.toy_problem(), 200),
    ("phev_q50", lambda: synth.phev_problem(1000, 50), 200),
    ("random_2_300_7", lambda: synth.random_problem(2, 300, 7, seed=41), 60),
    ("random_3_1025_2", lambda: synth.random_problem(3, 1025, 2, seed=42), 60),
    ("random_1_37_5", lambda: synth.random_problem(1, 37, 5, seed=43), 60),
]


def _params(name, P):
    if name.startswith("random"):
        return oracle.default_params(r_bar=1e-9, sigma_bar=1e-9, rho0=(1.0, 0.5, 1.0, 1.0))
    return oracle.default_params(r_bar=1e-6 * P["c"][1])


@pytest.mark.parametrize("horizon", [False, True], ids=["scenarios", "horizon"])
@pytest.mark.parametrize("name,make,iters", CASES, ids=[c[0] for c in CASES])
def test_world1_collective_path_matches_oracle(name, make, iters, horizon):
    P = make()
    prm = _params(name, P)
    So, io, ho = orc(P, prm, iters)
    Sg, ig, hg, eng = dist_run(P, prm, iters, horizon=horizon)
    compare_states(P, So, Sg)
    check_hist(ho, hg, P, So)
    assert eng in ("sweep2_kernel", "sweep_kernel")


@pytest.mark.parametrize("horizon", [False, True], ids=["scenarios", "horizon"])
def test_world1_collective_path_horizon_m4(horizon):
    """BASELINE.json configs[2] shape (m = 4, q = 1), multi-segment rows."""
    P = synth.horizon_problem(20000)
    prm = oracle.default_params(r_bar=1e-6 * P["c"][2])
    So, io, ho = orc(P, prm, 100)
    Sg, ig, hg, eng = dist_run(P, prm, 100, horizon=horizon)
    compare_states(P, So, Sg)
    check_hist(ho, hg, P, So)


@pytest.mark.parametrize("horizon", [False, True], ids=["scenarios", "horizon"])
def test_world1_collective_path_solves_to_tolerance(horizon):
    """PHEV q = 20 to the paper's thresholds through the collective path: same
    iteration count (within one check period) and objective as the oracle."""
    P = synth.phev_problem(1000, 20)
    dE = P["c"][1]
    prm = oracle.default_params(r_bar=1e-6 * dE)
    So, io, ho = orc(P, prm, 20000, solve=True)
    Sg, ig, hg, eng = dist_run(P, prm, 0, horizon=horizon, mode="solve", r_bar=1e-6 * dE,
                               sigma_bar=1e-2, max_iter=20000)
    assert io["status"] == 0 and ig["converged"]
    assert abs(ig["iterations"] - io["iterations"]) <= prm["check_every"]
    assert abs(ig["objective"] - io["objective"]) <= 1e-6 * abs(io["objective"])


def test_horizon_mode_rejects_a_partial_scenario_range():
    L = _lib()
    uid = L._lib.admm_nccl_unique_id()
    d = L.dist_for(0, 1, 4, uid, horizon=100)
    d.j_end = 3  # horizon blocks own every scenario
    with pytest.raises(L.AdmmError):
        L.AdmmSolver(2, 100, 4, dist=d)
