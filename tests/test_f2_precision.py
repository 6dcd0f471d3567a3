"""F2: mixed precision -- the per-element coefficients a2, a1,
b2, b1 stored in fp32 (the paper ran in fp32), every operation and
every state array in fp64 (include/admm.h admm_set_coeff_precision).

Reading F2-a: with fp32 storage the library solves, exactly as
in fp64, the problem whose a2, a1, b2, b1 are the fp32-rounded inputs.  So
  * parity: the CUDA path in fp32 mode must match the oracle run on the rounded
    problem (rounding done here with numpy, not by the CUDA path) to the same
    1e-9 as the fp64 path;
  * convergence study (CPU, oracle only): how far the rounded problem's optimum
    moves from the fp64 one.  The envelope theorem fixes the first-order change
    of the optimal value of Eq. (2) under a perturbation of
    f and g at a KKT point: d obj = (1/q) sum (da2 x^2 + da1 x)
    + sum_ij kappa_ij sum_k (db2 x^2 + db1 x), kappa = -rho1 lam the capacity
    multiplier (identity I3).  The measured change must equal that prediction
    up to second-order terms."""

import numpy as np
import pytest

import oracle
import synth

UNIT = dict(rho0=(1.0, 1.0, 1.0, 1.0))
COEF = ("a2", "a1", "b2", "b1")


def round32(P):
    Q = dict(P)
    for k in COEF:
        Q[k] = np.asarray(P[k], dtype=np.float64).astype(np.float32).astype(np.float64)
    return Q


def envelope_prediction(P, Q, o):
    """First-order change of the optimal value from P to Q at o's KKT point."""
    rho, x, q = o.rho, o.x, P["q"]
    kap = -rho[0] * o.lam[:, :, 0]
    d = {k: Q[k] - P[k] for k in COEF}
    df = (d["a2"] * x * x + d["a1"] * x).sum() / q
    dg = (kap[:, :, None] * (d["b2"] * x * x + d["b1"] * x)).sum()
    return df + dg


def test_round32_changes_only_the_four_coefficient_arrays():
    P = synth.random_problem(2, 7, 3, seed=5)
    Q = round32(P)
    for k in COEF:
        assert not np.array_equal(P[k], Q[k])
        assert np.all(np.abs(Q[k] - P[k]) <= 2.0 ** -24 * np.abs(P[k]))
    for k in ("a0", "b0", "lo", "hi", "y", "c"):
        assert Q[k] is P[k]


@pytest.mark.parametrize("seed", range(4))
@pytest.mark.parametrize("mode", [oracle.BOX_PROJECT, oracle.BOX_EXACT])
def test_fp32_coefficients_move_the_optimum_by_the_envelope_prediction(seed, mode):
    P = synth.random_problem(2, 4, 2, seed=seed)
    Q = round32(P)
    objs = []
    o64 = None
    for X in (P, Q):
        o = oracle.Oracle(X, oracle.default_params(r_bar=1e-12, sigma_bar=1e-12, box_mode=mode,
                                                   **UNIT))
        info, _ = o.solve(2_000_000)
        assert info["status"] == 0
        objs.append(info["objective"])
        o64 = o if o64 is None else o64
    act = objs[1] - objs[0]
    pred = envelope_prediction(P, Q, o64)
    # the change itself is O(2^-24) relative; its second-order remainder O(2^-48), the
    # solves to r = sigma = 1e-12 add ~1e-12 relative (EXACT mode, seed 1)
    assert abs(pred) > 1e-10 * abs(objs[0])
    assert abs(act - pred) <= 1e-12 * abs(objs[0]) + 1e-4 * abs(pred), (act, pred)


def test_fp32_toy_study_paper_tolerance():
    """The PHEV toy (BASELINE configs[0], paper rho0 and units) solved to the
    paper's tolerance: the rounded problem's objective and first control action
    stay within the relative size of the rounding (plus the tolerance's own
    effect, bounded by the fp64 solve's distance to a tight solve)."""
    P = synth.toy_problem()
    dE = P["c"][1]
    res = {}
    for tag, X in (("f64", P), ("f32", round32(P))):
        for tol in (1e-6, 1e-10):
            o = oracle.Oracle(X, oracle.default_params(r_bar=tol * dE))
            info, _ = o.solve(400_000)
            assert info["status"] == 0
            res[tag, tol] = (info["objective"], o.x1.copy())
    o_t, x1_t = res["f64", 1e-10]
    tol_eff = abs(res["f64", 1e-6][0] - o_t) + 1e-12 * abs(o_t)
    assert abs(res["f32", 1e-10][0] - o_t) <= 1e-6 * abs(o_t)
    assert abs(res["f32", 1e-6][0] - o_t) <= tol_eff + 1e-6 * abs(o_t)
    assert np.abs(res["f32", 1e-10][1] - x1_t).max() <= 1e-4 * max(1.0, np.abs(x1_t).max())


# ----------------------------------------------------------------- GPU parity
def _gpu(P, prm, iters, engine, bits=32):
    import os

    import paper_1903_10041_b200 as L

    env = {"grid": {"ADMM_PERSIST_GRID": "1"},
           "stream_fx": {"ADMM_SWEEP_FX": "1", "ADMM_SWEEP2": "0"},
           "stream_legacy": {"ADMM_SWEEP2": "0"}}
    exec_mode = {"stream": 1, "stream_fx": 1, "stream_legacy": 1, "cluster": 2, "grid": 2}[engine]
    s = L.AdmmSolver(P["m"], P["n"], P["q"], rho=prm["rho0"], tau=prm["tau"],
                     r_bar=prm["r_bar"], sigma_bar=prm["sigma_bar"], box_mode=prm["box_mode"],
                     check_every=prm["check_every"], exec_mode=exec_mode, coeff_bits=bits)
    for k in ("ADMM_PERSIST_GRID", "ADMM_SWEEP_FX", "ADMM_SWEEP2"):
        os.environ.pop(k, None)
    os.environ.update(env.get(engine, {}))
    try:
        assert s.coeff_bits == bits
        s.set_problem(P)
        s.iterate(iters)
        S = s.state()
        x, x1, sol = s.solution()
        hist = s.history()
        eng = s.engine()[0]
    finally:
        s.close()
        for k in ("ADMM_PERSIST_GRID", "ADMM_SWEEP_FX", "ADMM_SWEEP2"):
            os.environ.pop(k, None)
    return S, sol, hist, eng


@pytest.mark.gpu
@pytest.mark.parametrize("iters", [10, 200])
@pytest.mark.parametrize("engine", ["stream", "stream_legacy", "stream_fx", "cluster", "grid"])
def test_gpu_fp32_coefficients_phev_q50(iters, engine):
    from test_gpu_admm import check_hist, compare_states

    P = synth.phev_problem(1000, 50)
    prm = oracle.default_params(r_bar=1e-6 * P["c"][1])
    Q = round32(P)
    o = oracle.Oracle(Q, prm)
    io, ho = o.run(iters)
    Sg, sol, hg, eng = _gpu(P, prm, iters, engine)
    assert eng == {"stream": 4, "stream_legacy": 1, "stream_fx": 1, "cluster": 5, "grid": 2}[engine]
    compare_states(Q, o.state(), Sg)
    check_hist(ho, hg, Q, o.state())
    assert abs(sol["objective"] - io["objective"]) <= 1e-9 * abs(io["objective"])


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,q", [(1, 5, 3), (2, 37, 3), (3, 1001, 2), (2, 2500, 2),
                                   (4, 3001, 1)])
@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("engine", ["stream", "stream_legacy", "stream_fx", "cluster"])
def test_gpu_fp32_coefficients_random(m, n, q, mode, engine):
    """Ragged tails, multi-tile rows, every m, both box modes."""
    from test_gpu_admm import check_hist, compare_states

    P = synth.random_problem(m, n, q, seed=77 * m + n + q)
    prm = oracle.default_params(r_bar=1e-9, sigma_bar=1e-9, box_mode=mode,
                                rho0=(1.0, 0.5, 1.0, 1.0))
    Q = round32(P)
    o = oracle.Oracle(Q, prm)
    io, ho = o.run(60)
    Sg, sol, hg, _ = _gpu(P, prm, 60, engine)
    compare_states(Q, o.state(), Sg)
    check_hist(ho, hg, Q, o.state())


@pytest.mark.gpu
def test_gpu_fp32_sweep_full_size_sampled():
    """BASELINE configs[3] at q = 1e4 in the bench's launch configuration
    (streaming engine, fp32 coefficients): q/50 copies of the q = 50 PHEV
    problem, 100 iterations, every copy bitwise identical and equal to the
    oracle of the rounded q = 50 problem replicated."""
    import torch

    import paper_1903_10041_b200 as L
    from test_gpu_admm import _replicated_oracle

    q = 10000
    base = synth.phev_problem(1000, 50)
    reps = q // 50
    P = {}
    for k, v in base.items():
        if k in ("a2", "a1", "a0", "b2", "b1", "b0"):
            P[k] = torch.from_numpy(v).cuda().repeat(1, reps, 1)
        elif k == "y":
            P[k] = torch.from_numpy(v).cuda().repeat(reps, 1)
        elif isinstance(v, np.ndarray):
            P[k] = torch.from_numpy(v).cuda()
        else:
            P[k] = v
    P["q"] = q
    prm = oracle.default_params(r_bar=1e-6 * base["c"][1])
    s = L.AdmmSolver(2, 1000, q, r_bar=prm["r_bar"], coeff_bits=32)
    s.set_problem(P)
    s.iterate(100)
    x, x1, sol = s.solution()
    eng = s.engine()[0]
    s.close()
    del P
    assert eng == 4  # the TMA sweep reads the fp32 coefficient copies
    xs = x.reshape(2, reps, 50, 1000)
    assert np.array_equal(xs.min(axis=1), xs.max(axis=1)), "copies diverged"
    o = _replicated_oracle(round32(base), reps, prm)
    o.run(100)
    assert np.abs(xs[:, 0] - o.x).max() / 1e5 <= 1e-9
    assert np.abs(x1 - o.x1).max() / 1e5 <= 1e-9


@pytest.mark.gpu
def test_gpu_precision_switch_semantics():
    import paper_1903_10041_b200 as L
    from paper_1903_10041_b200 import _lib

    P = synth.toy_problem()
    s = L.AdmmSolver(P["m"], P["n"], P["q"])
    try:
        assert s.coeff_bits == 64
        s.set_problem(P)
        s.iterate(10)
        with pytest.raises(L.AdmmError) as e:
            s.set_coeff_precision(16)
        assert e.value.status == _lib.ADMM_ERR_INVALID
        s.set_coeff_precision(32)  # discards the fp64 problem
        with pytest.raises(L.AdmmError) as e:
            s.iterate(1)
        assert e.value.status == _lib.ADMM_ERR_STATE
        s.set_problem(P)
        s.iterate(10)
        S32 = s.state()
        s.set_coeff_precision(32)  # unchanged precision keeps the problem
        s.iterate(1)
    finally:
        s.close()
    o = oracle.Oracle(round32(P), oracle.default_params(r_bar=1e-6 * P["c"][1]))
    o.run(10)
    assert np.abs(S32["x"] - o.x).max() / 1e5 <= 1e-9
