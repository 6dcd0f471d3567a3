"""Pins for the oracle's Algorithm 1: the quartic minimiser
is checked against things other than itself -- exact worked cases, 60-digit
mpmath stationary points, dense grid + golden section, derivative signs,
scale covariance and the middle-root property.  No GPU."""

import json
import math
import os

import mpmath as mp
import numpy as np
import pytest

import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


# ------------------------------------------------------------------ exact cases
@pytest.mark.parametrize("case", GOLD["cubic"], ids=lambda c: c["cite"][:12])
def test_cubic_exact(case):
    roots, br = oracle.cubic_roots(*case["bcd"])
    assert br == case["branch"]
    assert np.allclose(sorted(roots), case["roots"], atol=1e-12, rtol=0)


@pytest.mark.parametrize("case", GOLD["quartic_argmin"], ids=lambda c: c["cite"][:12])
def test_quartic_exact(case):
    x, tie = oracle.quartic_argmin(*case["ABCD"])
    assert abs(x - case["x"]) <= 1e-12
    assert tie == case.get("tie", False)


@pytest.mark.parametrize("case", GOLD["quadratic"], ids=lambda c: c["cite"][:12])
def test_quadratic_exact(case):
    a2, a1 = case["a2a1"]
    x, _ = oracle.quartic_argmin(0.0, 0.0, a2, a1)  # J = a2 x^2 + a1 x
    assert abs(x - case["x"]) <= 1e-12


@pytest.mark.parametrize("case", GOLD["interval_exact"], ids=lambda c: c["cite"][:12])
def test_interval_exact(case):
    x, _ = oracle.quartic_boxmin(*case["ABCD"], *case["lohi"], mode=oracle.BOX_EXACT)
    assert abs(x - case["x"]) <= 1e-12


def test_project_vs_exact_differ_when_box_cuts_between_wells():
    # x^4 - 2x^2 on [-0.5, 2]: clamp(argmin_R) = clamp(-1) = -0.5 (J = -0.4375)
    # while the box minimiser is +1 (J = -1).  Reading G3.
    xp, _ = oracle.quartic_boxmin(1, 0, -2, 0, -0.5, 2.0, mode=oracle.BOX_PROJECT)
    xe, _ = oracle.quartic_boxmin(1, 0, -2, 0, -0.5, 2.0, mode=oracle.BOX_EXACT)
    assert xp == -0.5 and abs(xe - 1.0) < 1e-15


# ------------------------------------------------------------- mpmath truth
def _mp_stationary(A, B, C, D):
    mp.mp.dps = 60
    cs = [mp.mpf(4 * A), mp.mpf(3 * B), mp.mpf(2 * C), mp.mpf(D)]
    rts = mp.polyroots(cs, maxsteps=500, extraprec=400)
    out = []
    for r in rts:
        if abs(mp.im(r)) <= mp.mpf(10) ** -40 * (1 + abs(r)):
            out.append(mp.re(r))
    return out


def _mpJ(A, B, C, D, x):
    x = mp.mpf(x)
    return ((mp.mpf(A) * x + B) * x + C) * x * x + mp.mpf(D) * x


def _true_argmin(A, B, C, D, lo=None, hi=None):
    """(x_true, tie) from 60-digit stationary points (+ endpoints if boxed)."""
    cand = _mp_stationary(A, B, C, D)
    if lo is not None:
        cand = [c for c in cand if lo < c < hi] + [mp.mpf(lo), mp.mpf(hi)]
    vals = sorted((_mpJ(A, B, C, D, c), c) for c in cand)
    best = vals[0]
    tie = False
    for v, c in vals[1:]:
        if abs(c - best[1]) > mp.mpf(10) ** -30 * (1 + abs(c)) and \
                abs(v - best[0]) <= mp.mpf(1e-12) * (abs(v) + abs(best[0]) + 1e-300):
            tie = True
    return best[1], tie


def _families(rng, N):
    fam = {}
    A = rng.uniform(0.1, 10, N); B = rng.uniform(-10, 10, N)
    fam["R"] = np.stack([A, B, rng.uniform(-10, 10, N), rng.uniform(-10, 10, N)], 1)
    C = 3 * B * B / (8 * A) + rng.uniform(0, 10, N)
    fam["C"] = np.stack([A, B, C, rng.uniform(-10, 10, N)], 1)
    # PHEV-shaped battery quartics (SURVEY.md Appendix V "small-root cancellation"):
    rho1, rho3 = 1e-4, 5e-6
    b2 = 10 ** rng.uniform(-8, -4, N)
    b1 = np.ones(N)
    th = rng.uniform(-1e5, 1e5, N)
    ph = rng.uniform(-5e4, 5e4, N)
    fam["phev"] = np.stack([rho1 * b2 * b2 / 2, rho1 * b2 * b1,
                            rho1 * (b1 * b1 - 2 * b2 * th) / 2 + rho3 / 2,
                            -rho1 * b1 * th - rho3 * ph], 1)
    # cubics with roots spread over 10^+-6 (cancellation stress)
    r = (10 ** rng.uniform(-6, 6, (N, 3))) * rng.choice([-1, 1], (N, 3))
    a = rng.uniform(0.5, 2, N)
    e1 = r.sum(1); e2 = r[:, 0] * r[:, 1] + r[:, 0] * r[:, 2] + r[:, 1] * r[:, 2]
    e3 = r.prod(1)
    # J' = 4a (x-r1)(x-r2)(x-r3) = 4a x^3 - 4a e1 x^2 + 4a e2 x - 4a e3
    fam["spread"] = np.stack([a, -4 * a * e1 / 3, 2 * a * e2, -4 * a * e3], 1)
    return fam


@pytest.mark.parametrize("fam", ["R", "C", "phev", "spread"])
def test_argmin_vs_mpmath(fam):
    rng = np.random.default_rng([190310041, 11, ord(fam[0])])
    cases = _families(rng, 400)[fam]
    bad = []
    for A, B, Cc, D in cases:
        x, tie = oracle.quartic_argmin(A, B, Cc, D)
        xt, ttie = _true_argmin(A, B, Cc, D)
        if tie or ttie:
            # several minimisers are correct: J(x) must equal the optimum
            Jx, Jt = _mpJ(A, B, Cc, D, x), _mpJ(A, B, Cc, D, xt)
            assert Jx - Jt <= 1e-12 * (abs(Jt) + 1)
            continue
        err = abs(mp.mpf(x) - xt) / max(1, abs(xt))
        # the argmin is ill-conditioned at near-double stationary points; there
        # the objective (not x) is what is determined
        if err > 1e-13:
            Jx, Jt = _mpJ(A, B, Cc, D, x), _mpJ(A, B, Cc, D, xt)
            if Jx - Jt > 1e-14 * (abs(Jt) + 1):
                bad.append((A, B, Cc, D, x, float(xt), float(err)))
    assert not bad, bad[:5]


def test_degenerate_A_is_not_a_quadratic():
    # Reading G9: A = 5e-17 is tiny but not zero; the argmin is 19410.9,
    # the quadratic fallback -D/2C would give 20544.6.
    A, B, Cc, D = 5e-17, 1e-10, 5.05e-5, -2.075
    x, _ = oracle.quartic_argmin(A, B, Cc, D)
    xt, _ = _true_argmin(A, B, Cc, D)
    assert abs(x - float(xt)) <= 1e-12 * abs(float(xt))
    assert abs(x - 19410.9) < 0.1


@pytest.mark.parametrize("fam", ["R", "C", "phev"])
def test_boxmin_exact_vs_mpmath(fam):
    rng = np.random.default_rng([190310041, 12, ord(fam[0])])
    cases = _families(rng, 300)[fam]
    scale = 1e5 if fam == "phev" else 5.0
    for A, B, Cc, D in cases:
        u, v = sorted(rng.uniform(-scale, scale, 2))
        x, tie = oracle.quartic_boxmin(A, B, Cc, D, u, v, mode=oracle.BOX_EXACT)
        xt, ttie = _true_argmin(A, B, Cc, D, u, v)
        Jx, Jt = _mpJ(A, B, Cc, D, x), _mpJ(A, B, Cc, D, xt)
        assert u <= x <= v
        assert Jx - Jt <= 1e-13 * (abs(Jt) + 1)
        # project mode = clamp of the global argmin
        xp, _ = oracle.quartic_boxmin(A, B, Cc, D, u, v, mode=oracle.BOX_PROJECT)
        xg, _ = oracle.quartic_argmin(A, B, Cc, D)
        assert xp == min(max(xg, u), v)


def test_exact_equals_best_of_clamped_extreme_roots():
    """Reading G3's lemma (used by the CUDA path): for A > 0 with stationary
    points x1 <= x2 <= x3, argmin_[lo,hi] J is attained in {clamp(x1), clamp(x3)}.
    Checked with mpmath truth, independent of the oracle."""
    rng = np.random.default_rng([190310041, 13])
    fam = _families(rng, 300)
    for A, B, Cc, D in np.concatenate([fam["R"], fam["phev"]]):
        st = sorted(_mp_stationary(A, B, Cc, D))
        sc = 1e5 if abs(A) < 1e-3 else 5.0
        u, v = sorted(rng.uniform(-sc, sc, 2))
        xt, _ = _true_argmin(A, B, Cc, D, u, v)
        c1 = min(max(st[0], u), v)
        c3 = min(max(st[-1], u), v)
        best = min(_mpJ(A, B, Cc, D, c1), _mpJ(A, B, Cc, D, c3))
        assert best - _mpJ(A, B, Cc, D, xt) <= mp.mpf(10) ** -40 * (1 + abs(best))


# ------------------------------------------------------ grid / golden section
def _grid_golden(A, B, Cc, D, lo, hi, npts=10000):
    xs = np.linspace(lo, hi, npts)
    J = (((A * xs + B) * xs + Cc) * xs + D) * xs
    i = int(np.argmin(J))
    a, b = xs[max(i - 1, 0)], xs[min(i + 1, npts - 1)]
    g = (math.sqrt(5) - 1) / 2
    f = lambda t: (((A * t + B) * t + Cc) * t + D) * t  # noqa: E731
    for _ in range(200):
        c, d = b - g * (b - a), a + g * (b - a)
        if f(c) < f(d):
            b = d
        else:
            a = c
    t = 0.5 * (a + b)
    return min(f(t), J[i])


@pytest.mark.parametrize("fam", ["R", "C"])
def test_argmin_vs_dense_grid(fam):
    """SPEC.md:61 / :546: f(x*) <= f_grid + 1e-8 (1 + |f_grid|) over a
    root-bound bracket (Cauchy bound of J')."""
    rng = np.random.default_rng([190310041, 14, ord(fam)])
    for A, B, Cc, D in _families(rng, 500)[fam]:
        bound = 1 + max(abs(3 * B), abs(2 * Cc), abs(D)) / (4 * A)
        x, _ = oracle.quartic_argmin(A, B, Cc, D)
        fx = (((A * x + B) * x + Cc) * x + D) * x
        fg = _grid_golden(A, B, Cc, D, -bound, bound)
        assert fx <= fg + 1e-8 * (1 + abs(fg))


# ------------------------------------------------------ calculus properties
def test_derivative_signs_exact_mode():
    rng = np.random.default_rng([190310041, 15])
    for A, B, Cc, D in _families(rng, 500)["R"]:
        lo, hi = sorted(rng.uniform(-5, 5, 2) ** 2 * np.sign(rng.uniform(-1, 1, 2)))
        x, _ = oracle.quartic_boxmin(A, B, Cc, D, lo, hi, mode=oracle.BOX_EXACT)
        d1 = ((4 * A * x + 3 * B) * x + 2 * Cc) * x + D
        d2 = (12 * A * x + 6 * B) * x + 2 * Cc
        scale = 4 * A * abs(x) ** 3 + 3 * abs(B) * x * x + 2 * abs(Cc) * abs(x) + abs(D) + 1
        if lo < x < hi:
            assert abs(d1) <= 1e-10 * scale and d2 >= -1e-8 * (abs(12 * A * x * x) + 1)
        elif x == lo:
            assert d1 >= -1e-10 * scale  # J increases into the box
        else:
            assert x == hi and d1 <= 1e-10 * scale


def test_scale_covariance():
    """argmin(sA, sB, sC, sD) = argmin(A, B, C, D), s > 0."""
    rng = np.random.default_rng([190310041, 16])
    for A, B, Cc, D in _families(rng, 300)["R"]:
        x0, t0 = oracle.quartic_argmin(A, B, Cc, D)
        x1, _ = oracle.quartic_argmin(4 * A, 4 * B, 4 * Cc, 4 * D)  # power of 2: exact
        assert x0 == x1
        x2, _ = oracle.quartic_argmin(3.7 * A, 3.7 * B, 3.7 * Cc, 3.7 * D)
        if not t0:
            assert abs(x2 - x0) <= 1e-9 * max(1, abs(x0))


def test_middle_root_is_a_maximiser():
    """SPEC.md:88 / PAPER.md:166: the middle sorted root has J'' <= 0."""
    rng = np.random.default_rng([190310041, 17])
    n3 = 0
    for A, B, Cc, D in _families(rng, 2000)["R"]:
        b, c, d = 3 * B / (4 * A), Cc / (2 * A), D / (4 * A)
        roots, br = oracle.cubic_roots(b, c, d)
        if br != 2:
            continue
        n3 += 1
        xm = roots[1]
        assert roots[0] <= roots[1] <= roots[2]
        d2 = (12 * A * xm + 6 * B) * xm + 2 * Cc
        assert d2 <= 1e-8 * (abs(12 * A * xm * xm) + abs(6 * B * xm) + abs(2 * Cc))
    assert n3 > 300  # family R takes the trig branch about a quarter of the time


def test_cubic_root_residuals_and_count():
    """SPEC.md:44/:50/:84: every root satisfies |p(x)| <= 1e-9 max(1, |x|^3) and
    the number of real roots agrees with numpy's companion-matrix eigenvalues."""
    rng = np.random.default_rng([190310041, 18])
    for b, c, d in rng.uniform(-10, 10, (3000, 3)):
        roots, br = oracle.cubic_roots(b, c, d)
        for x in roots:
            assert abs(((x + b) * x + c) * x + d) <= 1e-9 * max(1, abs(x) ** 3)
        ev = np.roots([1, b, c, d])
        nreal = int(np.sum(np.abs(ev.imag) <= 1e-7 * (1 + np.abs(ev))))
        if abs(((c / 3 - b * b / 9) ** 3 + (b * c / 6 - b ** 3 / 27 - d / 2) ** 2)) > 1e-6:
            assert len(roots) == nreal


def test_triple_root_continuity():
    """near the Q=R=0 singularity the root moves continuously.
    (x-1)^3 + s = 0 has the single real root 1 - cbrt(s) (closed form)."""
    for s in (1e-6, -1e-6, 1e-9, -1e-12):
        d = -1.0 + s
        s_eff = d + 1.0  # exact (Sterbenz): the perturbation actually represented
        roots, br = oracle.cubic_roots(-3.0, 3.0, d)
        assert br == 1 and len(roots) == 1
        # a triple root is determined only to ~cbrt(eps) by fp64 coefficients
        assert abs(roots[0] - (1.0 - np.cbrt(s_eff))) <= 2 * np.cbrt(4 * 2.2e-16)


def test_batch_matches_scalar():
    rng = np.random.default_rng([190310041, 19])
    F = _families(rng, 200)["R"]
    lo = rng.uniform(-5, 0, 200); hi = rng.uniform(0, 5, 200)
    for mode in (oracle.BOX_PROJECT, oracle.BOX_EXACT):
        xb, _ = oracle.quartic_batch(F[:, 0], F[:, 1], F[:, 2], F[:, 3], lo, hi, mode)
        for e in range(200):
            assert xb[e] == oracle.quartic_boxmin(*F[e], lo[e], hi[e], mode)[0]
