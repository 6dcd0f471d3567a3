"""Pins for the oracle's ADMM (Appendix A, Eq. (5)-(6)) against things
other than itself:
  * every primal block update is the minimiser of the augmented Lagrangian L
    (written out independently below) over its block;
  * the scaled-dual identities I1/I2 that hold only when the
    dual steps have the right signs and indices;
  * the KKT conditions of Eq. (2) at convergence (textbook, derived here) and an
    independent scipy SLSQP solution on tiny instances;
  * closed-form special cases (equal marginal cost, demand-only clamp,
    capacity-only water-filling by bisection);
  * residual bounds on the Eq. (2) violation, permutation / duplication of
    scenarios, an exact fixed point (r = sigma = 0).
No GPU."""

import json
import os

import numpy as np
import pytest
from scipy.optimize import minimize

import oracle
import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
PAPER = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_params.json")))

UNIT = dict(rho0=(1.0, 1.0, 1.0, 1.0))


def _prob_from_json(c):
    P = {k: np.array(c[k], dtype=float) for k in
         ("a2", "a1", "a0", "b2", "b1", "b0", "lo", "hi", "y", "c")}
    P.update(m=c["m"], n=c["n"], q=c["q"])
    return P


def g_of(P, x):
    return (P["b2"] * x + P["b1"]) * x + P["b0"]


def f_of(P, x):
    return (P["a2"] * x + P["a1"]) * x + P["a0"]


# ------------------------------------------------------------------ defaults
def test_paper_defaults():
    p = oracle.default_params()
    assert tuple(p["rho0"]) == tuple(PAPER["rho0"]["value"])
    assert p["tau"] == PAPER["tau"]["value"]
    assert (p["hi_ratio"], p["lo_ratio"]) == tuple(PAPER["band"]["value"])
    assert p["check_every"] == PAPER["check_every"]["value"]
    assert p["sigma_bar"] == PAPER["sigma_bar"]["value"]


# ------------------------------------------------------------------ builder
def test_builder_spec_examples():
    for c in GOLD["builder"]:
        cf = oracle.build_quartic(c["a2"], c["a1"], c["b2"], c["b1"], c["b0"], c["theta"],
                                  c["phi"], c["q"], c["rho"], c["delta"])
        assert np.allclose(cf, c["ABCD"], rtol=0, atol=1e-15), c["cite"]
        x, _ = oracle.quartic_argmin(*cf)
        assert abs(x - c["argmin"]) < 1e-12


def test_builder_symbolic_expansion():
    """A..D equal the polynomial coefficients of the (6a) objective (PAPER.md:
    454-461), expanded symbolically by sympy at random rational points."""
    import sympy as sp

    X = sp.Symbol("x")
    rng = np.random.default_rng([190310041, 21])
    for trial in range(40):
        v = rng.uniform(-3, 3, 12)
        a2, b2 = abs(v[0]), abs(v[1])
        a1, b1, b0, th, ph, x1, nu = v[2:9]
        rho = np.abs(v[9:12]).tolist() + [abs(v[0]) + 0.1]
        q = 1 + trial % 5
        delta = trial % 2
        R = [sp.Rational(float(t)) for t in (a2, a1, b2, b1, b0, th, ph, x1, nu)]
        Rr = [sp.Rational(float(t)) for t in rho]
        A2, A1, B2, B1, B0, TH, PH, X1, NU = R
        g = B2 * X ** 2 + B1 * X + B0
        J = (A2 * X ** 2 + A1 * X) / q + Rr[0] / 2 * (TH - g) ** 2 + Rr[2] / 2 * (PH - X) ** 2
        if delta:
            J += Rr[3] / 2 * (X1 - X + NU) ** 2
        poly = sp.Poly(sp.expand(J), X)
        want = [float(poly.coeff_monomial(X ** p)) for p in (4, 3, 2, 1)]
        got = oracle.build_quartic(a2, a1, b2, b1, b0, th, ph, q, rho, delta, x1, nu)
        for w, gt in zip(want, got):
            assert abs(w - gt) <= 1e-12 * (1 + abs(w))


# ------------------------------------------------------- augmented Lagrangian
def x_terms(P, q_tot, rho, S0, xmix, i, j, k, xi):
    """The xi-dependent terms of L for element (i,j,k) with
    every other variable fixed.  Written from the paper, not the oracle."""
    e = (i, j, k)
    gx = (P["b2"][e] * xi + P["b1"][e]) * xi + P["b0"][e]
    val = (P["a2"][e] * xi * xi + P["a1"][e] * xi + P["a0"][e]) / q_tot
    val = val + rho[0] / 2 * (S0["z"][e] - gx + S0["lam"][e]) ** 2
    others = sum(xmix[l, j, k] for l in range(P["m"]) if l != i)
    val = val + rho[2] / 2 * (S0["s"][j, k] - (others + xi) + P["y"][j, k] + S0["mu"][j, k]) ** 2
    if k == 0:
        val = val + rho[3] / 2 * (S0["x1"][i] - xi + S0["nu"][i, j]) ** 2
    return val


def _take_one(P, params, warm=0):
    o = oracle.Oracle(P, params)
    if warm:
        o.run(warm)
    S0 = o.state()
    rho = o.rho.copy()
    o.run(1)
    return o, S0, rho, o.state()


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_x_update_minimises_L_exact_mode(seed):
    """(6a) in EXACT mode: each x_k^{(i,j)} minimises L over [lo, hi] given the
    latest values of the other sources (Gauss-Seidel over i, reading G2)."""
    P = synth.random_problem(3, 5, 2, seed=seed)
    o, S0, rho, S1 = _take_one(P, oracle.default_params(box_mode=oracle.BOX_EXACT, **UNIT),
                               warm=7)
    m, q, n = 3, 2, 5
    for i in range(m):
        xmix = np.where(np.arange(m)[:, None, None] < i, S1["x"], S0["x"])
        for j in range(q):
            for k in range(n):
                lo, hi = P["lo"][i, k], P["hi"][i, k]
                xs = np.linspace(lo, hi, 4001)
                vals = x_terms(P, q, rho, S0, xmix, i, j, k, xs)
                xstar = S1["x"][i, j, k]
                vstar = x_terms(P, q, rho, S0, xmix, i, j, k, xstar)
                assert lo <= xstar <= hi
                assert vstar <= vals.min() + 1e-12 * (1 + abs(vals.min()))
                for d in (1e-6, -1e-6):
                    xp = min(max(xstar + d, lo), hi)
                    assert vstar <= x_terms(P, q, rho, S0, xmix, i, j, k, xp) + 1e-13


@pytest.mark.parametrize("seed", [3, 4])
def test_x_update_project_mode_is_clamped_global_min(seed):
    """(6a) as printed: Pi_box(argmin over R)."""
    P = synth.random_problem(2, 4, 3, seed=seed)
    o, S0, rho, S1 = _take_one(P, oracle.default_params(**UNIT), warm=5)
    for i in range(2):
        xmix = np.where(np.arange(2)[:, None, None] < i, S1["x"], S0["x"])
        for j in range(3):
            for k in range(4):
                xs = np.linspace(-50, 50, 200001)
                vals = x_terms(P, 3, rho, S0, xmix, i, j, k, xs)
                xg = xs[np.argmin(vals)]
                want = min(max(xg, P["lo"][i, k]), P["hi"][i, k])
                assert abs(S1["x"][i, j, k] - want) <= 1e-3


@pytest.mark.parametrize("seed", [0, 5])
def test_other_blocks_minimise_L(seed):
    """(6b)-(6e) are block minimisers of L; checked through their optimality
    conditions, derived here from PAPER.md:391-407."""
    P = synth.random_problem(2, 6, 3, seed=seed)
    o, S0, rho, S1 = _take_one(P, oracle.default_params(**UNIT), warm=4)
    g1 = g_of(P, S1["x"])
    n = P["n"]
    # z: d/dz_k = rho1 (z_k - g_k + lam_k) - rho2 (h - 1'z + p) = 0
    lhs = rho[0] * (S1["z"] - g1 + S0["lam"])
    rhs = rho[1] * (S0["h"] - S1["z"].sum(axis=2) + S0["p"])[:, :, None]
    assert np.allclose(lhs, np.broadcast_to(rhs, lhs.shape), atol=1e-12)
    # x1: sum_j (x1 - x_1^{(i,j)} + nu^{(i,j)}) = 0  (mean, erratum E4)
    assert np.allclose((S1["x1"][:, None] - S1["x"][:, :, 0] + S0["nu"]).sum(axis=1), 0,
                       atol=1e-12)
    # h: minimiser of (h - 1'z + p)^2 over h <= c
    t = S1["z"].sum(axis=2) - S0["p"]
    assert np.all(S1["h"] <= P["c"][:, None])
    inner = S1["h"] < P["c"][:, None]
    assert np.allclose(S1["h"][inner], t[inner], atol=1e-12)
    assert np.all(t[~inner] >= P["c"][:, None].repeat(3, 1)[~inner] - 1e-12)
    # s: minimiser of ||s - sum x + y + mu||^2 over s >= 0
    v = S1["x"].sum(axis=0) - P["y"] - S0["mu"]
    assert np.all(S1["s"] >= 0)
    assert np.allclose(S1["s"][v > 0], v[v > 0], atol=1e-12)
    assert np.all(S1["s"][v <= 0] == 0)
    del n


def test_scaled_dual_identities():
    """I1: lambda is constant over k from iteration 1; I2: s mu = 0, mu >= 0.
    Both fail for a wrong sign or index in (6f)/(6g)."""
    P = synth.random_problem(2, 7, 3, seed=6)
    o = oracle.Oracle(P, oracle.default_params(**UNIT))
    for it in range(40):
        o.run(1)
        lam = o.lam
        spread = lam.max(axis=2) - lam.min(axis=2)
        assert np.all(spread <= 1e-12 * (1 + np.abs(lam).max()))
        assert np.all(o.mu >= -1e-12)
        assert np.all(np.minimum(o.s, np.abs(o.mu)) <= 1e-12)
        # invariants after every iteration
        assert np.all(o.x >= P["lo"][:, None, :]) and np.all(o.x <= P["hi"][:, None, :])
        assert np.all(o.s >= 0) and np.all(o.h <= P["c"][:, None])
        # rho1 lam = rho2 p is reached only at a fixed point; its sign is checked at KKT


# ------------------------------------------------------------ whole solves
@pytest.mark.parametrize("case", GOLD["solve"], ids=lambda c: c["cite"][:10])
def test_spec_solve_examples(case):
    P = _prob_from_json(case)
    o = oracle.Oracle(P, oracle.default_params(r_bar=1e-9, sigma_bar=1e-9, **UNIT))
    info, _ = o.solve(100000)
    assert info["status"] == 0
    assert np.allclose(o.x, np.array(case["x"]), atol=1e-7)
    assert abs(info["objective"] - case["objective"]) < 1e-6


def kkt_violation(P, o):
    """KKT conditions of Eq. (2) at the oracle's solution with
    multipliers read from the scaled duals: demand w = rho3 mu >= 0, capacity
    kappa = -rho1 lam = -rho2 p >= 0, consensus xi = -rho4 nu."""
    rho = o.rho
    x = o.x
    q = P["q"]
    w = rho[2] * o.mu                   # [q][n]
    kap = -rho[0] * o.lam[:, :, 0]     # [m][q]
    kap2 = -rho[1] * o.p
    xi = -rho[3] * o.nu                 # [m][q]
    fp = (2 * P["a2"] * x + P["a1"]) / q
    gp = 2 * P["b2"] * x + P["b1"]
    grad = fp + kap[:, :, None] * gp - w[None]
    grad[:, :, 0] += xi
    lo = P["lo"][:, None, :]; hi = P["hi"][:, None, :]
    gap = np.where(x <= lo, np.minimum(grad, 0), np.where(x >= hi, np.maximum(grad, 0), grad))
    sc = 1 + np.abs(fp).max()
    G = g_of(P, x).sum(axis=2)
    dem = x.sum(axis=0) - P["y"]
    return dict(
        stationarity=np.abs(gap).max() / sc,
        dual_sign=max(-w.min(), -kap.min(), 0) / sc,
        kappa_agree=np.abs(kap - kap2).max() / sc,
        comp_dem=np.abs(w * dem).max() / (sc * (1 + np.abs(P["y"]).max())),
        comp_cap=np.abs(kap * np.where(np.isfinite(P["c"][:, None]), G - P["c"][:, None], 0)).max()
        / (sc * (1 + np.abs(G).max())),
        demand=max(0, -dem.min()) / (1 + np.abs(P["y"]).max()),
        capacity=max(0, (G - P["c"][:, None]).max()) / (1 + np.abs(G).max()),
        consensus=np.ptp(x[:, :, 0], axis=1).max() / (1 + np.abs(x).max()),
        xi_sum=np.abs(xi.sum(axis=1)).max() / sc,
    )


@pytest.mark.parametrize("seed", range(6))
@pytest.mark.parametrize("mode", [oracle.BOX_PROJECT, oracle.BOX_EXACT])
def test_kkt_certificate(seed, mode):
    P = synth.random_problem(2, 4, 2, seed=seed)
    o = oracle.Oracle(P, oracle.default_params(r_bar=1e-11, sigma_bar=1e-11, box_mode=mode,
                                               **UNIT))
    info, _ = o.solve(500000)
    assert info["status"] == 0
    v = kkt_violation(P, o)
    assert max(v.values()) < 1e-8, v


def _slsqp(P):
    m, n, q = P["m"], P["n"], P["q"]
    N = m * q * n

    def obj(v):
        return f_of(P, v.reshape(m, q, n)).sum() / q

    def objg(v):
        x = v.reshape(m, q, n)
        return ((2 * P["a2"] * x + P["a1"]) / q).ravel()

    cons = [dict(type="ineq", fun=lambda v: (v.reshape(m, q, n).sum(0) - P["y"]).ravel())]
    fin = np.isfinite(P["c"])
    cons.append(dict(type="ineq",
                     fun=lambda v: (P["c"][:, None] - g_of(P, v.reshape(m, q, n)).sum(2))[fin]
                     .ravel()))
    if q > 1:
        cons.append(dict(type="eq", fun=lambda v: (v.reshape(m, q, n)[:, 1:, 0]
                                                    - v.reshape(m, q, n)[:, :1, 0]).ravel()))
    bounds = list(zip(np.broadcast_to(P["lo"][:, None, :], (m, q, n)).ravel(),
                      np.broadcast_to(P["hi"][:, None, :], (m, q, n)).ravel()))
    best = None
    rng = np.random.default_rng(0)
    for s in range(5):
        x0 = rng.uniform([b[0] for b in bounds], [b[1] for b in bounds])
        r = minimize(obj, x0, jac=objg, bounds=bounds, constraints=cons, method="SLSQP",
                     options=dict(ftol=1e-15, maxiter=2000))
        if r.success and (best is None or r.fun < best.fun):
            best = r
    return best


@pytest.mark.parametrize("seed", range(5))
def test_objective_matches_slsqp(seed):
    P = synth.random_problem(2, 3, 2, seed=100 + seed)
    o = oracle.Oracle(P, oracle.default_params(r_bar=1e-11, sigma_bar=1e-11, **UNIT))
    info, _ = o.solve(500000)
    ref = _slsqp(P)
    assert ref is not None
    assert abs(info["objective"] - ref.fun) <= 1e-7 * (1 + abs(ref.fun))


def test_demand_only_closed_form():
    """m=1, q=1, g=0, c=inf: x_k = clamp(max(y_k, -a1/2a2), lo, hi)."""
    rng = np.random.default_rng(7)
    n = 9
    P = dict(m=1, n=n, q=1, a2=rng.uniform(0.5, 2, (1, 1, n)), a1=rng.uniform(-2, 2, (1, 1, n)),
             a0=np.zeros((1, 1, n)), b2=np.zeros((1, 1, n)), b1=np.zeros((1, 1, n)),
             b0=np.zeros((1, 1, n)), lo=np.full((1, n), -3.0), hi=np.full((1, n), 3.0),
             y=rng.uniform(-2, 2.5, (1, n)), c=np.array([np.inf]))
    o = oracle.Oracle(P, oracle.default_params(r_bar=1e-11, sigma_bar=1e-11, **UNIT))
    info, _ = o.solve(200000)
    want = np.clip(np.maximum(P["y"][0], -P["a1"][0, 0] / (2 * P["a2"][0, 0])), -3, 3)
    assert info["status"] == 0
    assert np.allclose(o.x[0, 0], want, atol=1e-8)


def test_capacity_only_water_filling():
    """m=1, q=1, demand inactive, capacity binding: x_k(kappa) =
    clamp(-(a1 + kappa b1) / (2 (a2 + kappa b2))); kappa by bisection on
    sum_k g(x_k(kappa)) = c."""
    rng = np.random.default_rng(8)
    n = 12
    a2 = rng.uniform(0.5, 2, n); a1 = rng.uniform(-6, -2, n)
    b2 = rng.uniform(0.05, 0.5, n); b1 = rng.uniform(0.5, 1.5, n)
    lo, hi = -1.0, 4.0
    xu = np.clip(-a1 / (2 * a2), lo, hi)  # unconstrained optimum
    c = 0.6 * ((b2 * xu + b1) * xu).sum()
    P = dict(m=1, n=n, q=1, a2=a2[None, None], a1=a1[None, None], a0=np.zeros((1, 1, n)),
             b2=b2[None, None], b1=b1[None, None], b0=np.zeros((1, 1, n)),
             lo=np.full((1, n), lo), hi=np.full((1, n), hi), y=np.full((1, n), -10.0),
             c=np.array([c]))

    def xk(kap):
        return np.clip(-(a1 + kap * b1) / (2 * (a2 + kap * b2)), lo, hi)

    def use(kap):
        x = xk(kap)
        return ((b2 * x + b1) * x).sum()

    a, b = 0.0, 1e3
    assert use(a) > c
    for _ in range(200):
        mid = 0.5 * (a + b)
        if use(mid) > c:
            a = mid
        else:
            b = mid
    want = xk(0.5 * (a + b))
    o = oracle.Oracle(P, oracle.default_params(r_bar=1e-11, sigma_bar=1e-11, **UNIT))
    info, _ = o.solve(500000)
    assert info["status"] == 0
    assert np.allclose(o.x[0, 0], want, atol=1e-7)


def test_residuals_bound_eq2_violation():
    """At termination the Eq. (2) violations are bounded by the residual terms:
    demand shortfall <= r1, capacity excess <= n r2 + r3, consensus spread
    <= 2 r4 (derived from (5): s >= 0, z - g, h - 1'z, x_1 - x1)."""
    P = synth.phev_problem(200, 4)
    dE = P["c"][1]
    for rb in (1e-3, 1e-4, 1e-5, 1e-6):
        o = oracle.Oracle(P, oracle.default_params(r_bar=rb * dE))
        info, hist = o.solve(200000)
        assert info["status"] == 0
        r1, r2, r3, r4 = hist[-1, 7:11]
        x = o.x
        G = g_of(P, x).sum(axis=2)
        short = (P["y"] - x.sum(axis=0)).max()
        excess = (G[1] - P["c"][1]).max()
        assert short <= r1 * (1 + 1e-9) + 1e-9
        assert excess <= P["n"] * r2 + r3 + 1e-6
        assert np.ptp(x[:, :, 0], axis=1).max() <= 2 * r4 * (1 + 1e-9) + 1e-9


def test_exact_fixed_point_gives_zero_residuals():
    """A state that one iteration leaves unchanged has r = sigma = 0
    (SPEC.md:311).  m=n=q=1, f = x^2 - 2x, g = 0, y = -100, box [0, 10],
    rho = 1: the optimum x = 1 with z = 0, s = 101 and zero duals is a fixed
    point (the x-update is the quadratic 2x^2 - 4x)."""
    P = dict(m=1, n=1, q=1, a2=np.ones((1, 1, 1)), a1=-2 * np.ones((1, 1, 1)),
             a0=np.zeros((1, 1, 1)), b2=np.zeros((1, 1, 1)), b1=np.zeros((1, 1, 1)),
             b0=np.zeros((1, 1, 1)), lo=np.zeros((1, 1)), hi=np.full((1, 1), 10.0),
             y=np.full((1, 1), -100.0), c=np.array([np.inf]))
    o = oracle.Oracle(P, oracle.default_params(**UNIT))
    o.x[...] = 1.0; o.z[...] = 0.0; o.lam[...] = 0.0
    o.s[...] = 101.0; o.mu[...] = 0.0; o.h[...] = 0.0; o.p[...] = 0.0
    o.x1[...] = 1.0; o.nu[...] = 0.0
    info, hist = o.run(10)
    assert hist[0, 1] == 0.0 and hist[0, 2] == 0.0
    assert o.x[0, 0, 0] == 1.0 and o.s[0, 0] == 101.0


def test_scenario_permutation_and_duplication():
    P = synth.phev_problem(120, 4)
    dE = P["c"][1]
    prm = oracle.default_params(r_bar=1e-8 * dE, sigma_bar=1e-4)
    o = oracle.Oracle(P, prm)
    info, _ = o.solve(400000)
    perm = np.array([2, 0, 3, 1])
    Pp = dict(P)
    for k in ("a2", "a1", "a0", "b2", "b1", "b0"):
        Pp[k] = P[k][:, perm]
    Pp["y"] = P["y"][perm]
    op = oracle.Oracle(Pp, prm)
    infp, _ = op.solve(400000)
    # same iterates up to the summation order of the Neumaier sums over j
    assert abs(infp["objective"] - info["objective"]) <= 1e-11 * abs(info["objective"])
    assert np.allclose(op.x, o.x[:, perm], rtol=0, atol=1e-6)
    # duplicating every scenario (q -> 2q) leaves the Eq. (2) optimum unchanged
    Pd = dict(P)
    for k in ("a2", "a1", "a0", "b2", "b1", "b0"):
        Pd[k] = np.concatenate([P[k], P[k]], axis=1)
    Pd["y"] = np.concatenate([P["y"], P["y"]], axis=0)
    Pd["q"] = 8
    od = oracle.Oracle(Pd, prm)
    infd, _ = od.solve(400000)
    assert abs(infd["objective"] - info["objective"]) <= 1e-6 * abs(info["objective"])


def test_rho_schedule_follows_paper_rule():
    """at each check all rho scale by tau if r/sigma > 1.2
    rbar/sigmabar, by 1/tau if < 0.8 rbar/sigmabar; nothing changes between
    checks; duals follow (reading G11)."""
    P = synth.phev_problem(150, 3)
    prm = oracle.default_params(r_bar=1e-6 * P["c"][1])
    o = oracle.Oracle(P, prm)
    info, hist = o.run(600)
    thr_hi = 1.2 * prm["r_bar"] / prm["sigma_bar"]
    thr_lo = 0.8 * prm["r_bar"] / prm["sigma_bar"]
    rho = np.array(prm["rho0"])
    nup = ndn = 0
    for row in hist:
        assert np.allclose(row[3:7], rho, rtol=1e-15, atol=0)
        r, s, conv = row[1], row[2], row[14]
        if conv:
            continue
        ratio = r / s if s > 0 else np.inf
        if ratio > thr_hi:
            rho = rho * 1.1; nup += 1
        elif ratio < thr_lo:
            rho = rho / 1.1; ndn += 1
    assert nup + ndn > 0
    assert np.allclose(o.rho, rho, rtol=1e-14)


def test_phev_paper_scale_solve():
    """Paper-scale sanity on a PHEV-shaped instance (q=5): converges at the
    paper's thresholds, battery capacity binds, demand met."""
    P = synth.phev_problem(1000, 5)
    o = oracle.Oracle(P, oracle.default_params(r_bar=1e-6 * P["c"][1]))
    info, _ = o.solve(20000)
    assert info["status"] == 0 and info["ties"] == 0
    G = g_of(P, o.x).sum(axis=2)
    assert np.all(np.abs(G[1] - P["c"][1]) <= 1e-3 * P["c"][1])
    assert (P["y"] - o.x.sum(axis=0)).max() <= 1e-6 * P["c"][1]
    assert np.ptp(o.x[:, :, 0], axis=1).max() <= 2e-6 * P["c"][1]
