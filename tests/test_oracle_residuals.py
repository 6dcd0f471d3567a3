"""Pins for the parts of the oracle that decide WHEN the ADMM stops and HOW rho
moves: the residuals r and sigma, the initial state
(reading G19) and the convergence behaviour the north star names
("objective monotone in residual at convergence").  Each pin is independent of
oracle/oracle.c:

  * r and sigma recomputed in numpy from the paper's printed definitions on the
    literal state before and after one iteration (check_every = 1), so any
    dropped or mis-scaled term of the oracle's history shows;
  * the first-order identity behind the dual residual (Boyd §3.3, cited at
    PAPER.md:325): after (6a)-(6i) the stationarity of the x-block written with
    the NEW multipliers is off by exactly rho1 g'(x) (z - z~) + rho3 ((s - s~)
    - sum_{l>i} (x_l - x~_l)) + delta_{k,1} rho4 (x1 - x1~) -- the quantities
    sigma measures;
  * a hand-worked initial state (tests/golden/init_example.json);
  * the objective error against a tight solve shrinks as r-bar is tightened;
  * the SURVEY.md §8(d) iteration count of an independent prototype (PHEV
    n = 1000, q = 5: 660 iterations).
No GPU."""

import json
import os

import numpy as np
import pytest

import oracle
import synth

HERE = os.path.dirname(__file__)
INIT = json.load(open(os.path.join(HERE, "golden", "init_example.json")))


def g_of(P, x):
    return (P["b2"] * x + P["b1"]) * x + P["b0"]


def paper_r_sigma(P, S0, S1, rho):
    """r and sigma exactly as printed at PAPER.md:464-479 (readings E6/E7: max
    over every present index, tilde = value at the start of the iteration)."""
    x, z, s, h, x1 = S1["x"], S1["z"], S1["s"], S1["h"], S1["x1"]
    r_terms = [
        np.abs(s - x.sum(axis=0) + P["y"]).max(),           # max_j ||s - sum_i x + y||
        np.abs(z - g_of(P, x)).max(),                       # max_ij ||z - g(x)||
        np.abs(h - z.sum(axis=2)).max(),                    # max_ij |h - 1'z|
        np.abs(x[:, :, 0] - x1[:, None]).max(),             # max_ij |x_1^(i,j) - x1^(i)|
    ]
    s_terms = [
        rho[0] * np.abs(z - S0["z"]).max(),                 # rho1 max ||z - z~||
        rho[1] * np.abs(h - S0["h"]).max(),                 # rho2 max |h - h~|
        rho[2] * np.abs((s - S0["s"]) - (x - S0["x"]).sum(axis=0)).max(),
    ]
    return r_terms, s_terms


def _cases():
    yield "random_m2", synth.random_problem(2, 5, 3, seed=11), dict(rho0=(0.7, 0.3, 0.9, 0.5))
    yield "random_m3", synth.random_problem(3, 4, 2, seed=12), dict(rho0=(1.0, 0.2, 0.6, 1.3))
    P = synth.phev_problem(40, 3)
    yield "phev", P, dict(r_bar=1e-6 * P["c"][1])


@pytest.mark.parametrize("name,P,kw", list(_cases()), ids=lambda v: v if isinstance(v, str) else "")
def test_history_equals_paper_residuals(name, P, kw):
    """Every residual column of the oracle's history equals r and sigma
    recomputed from PAPER.md:464-479, iteration by iteration, through rho
    changes (check_every = 1 so every iteration is a check)."""
    o = oracle.Oracle(P, oracle.default_params(check_every=1, **kw))
    changed = 0
    for it in range(25):
        S0 = o.state()
        rho = o.rho.copy()
        info, hist = o.run(1)
        S1 = o.state()
        rt, st = paper_r_sigma(P, S0, S1, rho)
        row = hist[0]
        sc_r = 1.0 + max(rt)
        sc_s = 1e-300 + max(st)
        assert np.allclose(row[3:7], rho, rtol=1e-15, atol=0)
        for c, want in zip(row[7:11], rt):
            assert abs(c - want) <= 1e-12 * sc_r, (name, it, row[7:11], rt)
        for c, want in zip(row[11:14], st):
            assert abs(c - want) <= 1e-12 * sc_s, (name, it, row[11:14], st)
        assert abs(row[1] - max(rt)) <= 1e-12 * sc_r
        assert abs(row[2] - max(st)) <= 1e-12 * sc_s
        changed += int(row[15] != 1.0)
    # the cases exercise each term: every sigma term and the r z-term nonzero
    assert min(st) > 0 and rt[1] > 0, (st, rt)


def test_dual_residual_identity():
    """First-order identity behind sigma (PAPER.md:421-450 + Boyd §3.3): in
    EXACT mode an interior x-update satisfies J'(x) = 0 for the (6a) objective
    built from the OLD state.  Rewriting J' with the NEW duals (6f)-(6h) gives
      (1/q) f'(x) - rho1 g'(x) lam - rho3 mu - d rho4 nu
        = -[rho1 g'(x) (z - z~) + rho3 ((s - s~) - sum_{l>i}(x_l - x~_l)) + d rho4 (x1 - x1~)],
    with d = delta_{k,1} (Gauss-Seidel: sources l > i entered (6a) with their
    old values).  Adaptation is off so no dual rescale intervenes."""
    for seed in range(3):
        P = synth.random_problem(2, 6, 3, seed=30 + seed)
        prm = oracle.default_params(rho0=(0.8, 0.4, 1.1, 0.6), adapt_rho=0,
                                    box_mode=oracle.BOX_EXACT)
        o = oracle.Oracle(P, prm)
        o.run(3)
        S0 = o.state()
        rho = o.rho
        o.run(1)
        S1 = o.state()
        x, q = S1["x"], P["q"]
        fp = (2 * P["a2"] * x + P["a1"]) / q
        gp = 2 * P["b2"] * x + P["b1"]
        lhs = fp - rho[0] * gp * S1["lam"] - rho[2] * S1["mu"][None]
        lhs[:, :, 0] -= rho[3] * S1["nu"]
        dx = x - S0["x"]
        later = np.zeros_like(x)  # sum_{l > i} (x_l - x~_l)
        for i in range(P["m"]):
            later[i] = dx[i + 1:].sum(axis=0)
        rhs = rho[0] * gp * (S1["z"] - S0["z"]) + rho[2] * ((S1["s"] - S0["s"])[None] - later)
        rhs[:, :, 0] += rho[3] * (S1["x1"] - S0["x1"])[:, None]
        lo, hi = P["lo"][:, None, :], P["hi"][:, None, :]
        interior = (x > lo + 1e-9) & (x < hi - 1e-9)
        assert interior.sum() >= 6
        scale = 1 + np.abs(fp).max() + np.abs(rho[0] * gp * S1["lam"]).max()
        err = np.abs(lhs + rhs)[interior].max() / scale
        assert err < 1e-11, err
        # at an active bound J' points out of the box (x = lo: J' >= 0, x = hi: J' <= 0)
        J1 = lhs + rhs
        assert np.all(J1[x <= lo] >= -1e-11 * scale)
        assert np.all(J1[x >= hi] <= 1e-11 * scale)


def test_initial_state_hand_worked():
    """G19 on a hand-worked instance: every array of the state
    right after initialisation equals the values computed by hand."""
    c = INIT
    P = {k: np.array(v, dtype=float) for k, v in c["problem"].items()}
    P.update(m=c["m"], n=c["n"], q=c["q"])
    o = oracle.Oracle(P, oracle.default_params())
    S = o.state()
    for k, want in c["state"].items():
        got = S[k]
        assert np.array_equal(np.asarray(got, dtype=float), np.array(want, dtype=float)), (k, got, want)


def test_objective_converges_as_rbar_tightens():
    """North-star invariant 'objective monotone in residual at convergence':
    on a PHEV-shaped instance with the capacity binding, the distance of the
    objective from a tight solve shrinks monotonically, and the Eq. (2)
    violations stay within what r < r-bar allows, as r-bar goes 1e-3 -> 1e-6 dE at the paper's sigma-bar
    (PAPER.md:317)."""
    P = synth.phev_problem(600, 2)
    dE = P["c"][1]
    tight = oracle.Oracle(P, oracle.default_params(r_bar=1e-9 * dE, sigma_bar=1e-6))
    info_t, _ = tight.solve(400000)
    assert info_t["status"] == 0
    ot = info_t["objective"]
    errs, viol = [], []
    for rb in (1e-3, 1e-4, 1e-5, 1e-6):
        o = oracle.Oracle(P, oracle.default_params(r_bar=rb * dE, sigma_bar=1e-2))
        info, _ = o.solve(400000)
        assert info["status"] == 0
        errs.append(abs(info["objective"] - ot) / abs(ot))
        G = g_of(P, o.x).sum(axis=2)
        short = max(0.0, (P["y"] - o.x.sum(axis=0)).max())
        excess = max(0.0, (G[1] - dE).max())
        viol.append(max(short, excess / P["n"]))
        # demand shortfall <= r1 and capacity excess <= n r2 + r3 (both terms < r-bar)
        assert viol[-1] <= (1 + 1.0 / P["n"]) * rb * dE, (rb, viol)
    assert all(a > b for a, b in zip(errs, errs[1:])), errs
    assert errs[-1] < 1e-4


def test_phev_q5_iteration_count_matches_survey():
    """SURVEY.md §8(d) generator-feasibility table: an independent numpy
    prototype of the literal algorithm on the PHEV generator (n = 1000, q = 5,
    paper rho0 / tau / thresholds, check every 10, dual rescale on, PROJECT)
    converged in 660 iterations.  Any change to r, sigma, the rho rule or the
    init shifts the check at which both thresholds are first met."""
    P = synth.phev_problem(1000, 5)
    o = oracle.Oracle(P, oracle.default_params(r_bar=1e-6 * P["c"][1]))
    info, _ = o.solve(20000)
    assert info["status"] == 0
    assert info["iterations"] == 660


def test_openmp_build_is_bitwise_identical():
    """bench.py's CPU-parallel baseline runs the OpenMP build of the same oracle
    source: every array, the history and the info must equal the serial build's
    bit for bit (sums stay serial per row; maxima are order-independent)."""
    oracle.set_threads(4)
    P = synth.random_problem(2, 37, 9, seed=5)
    runs = []
    for omp in (False, True):
        o = oracle.Oracle(P, oracle.default_params(rho0=(0.7, 0.3, 0.9, 0.5)), omp=omp)
        info, hist = o.run(60)
        runs.append((o.state(), info, hist))
    (S0, i0, h0), (S1, i1, h1) = runs
    for k in S0:
        assert np.array_equal(S0[k], S1[k]), k
    assert np.array_equal(h0, h1)
    assert i0 == i1
    A, B, Cc, D = (np.random.default_rng(3).uniform(-5, 5, 5000) for _ in range(4))
    A = np.abs(A) + 0.1
    x0, t0 = oracle.quartic_batch(A, B, Cc, D)
    x1, t1 = oracle.quartic_batch(A, B, Cc, D, omp=True)
    assert np.array_equal(x0, x1) and t0 == t1
