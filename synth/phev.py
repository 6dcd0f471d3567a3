"""PHEV-shaped synthetic problem instances (units W, J, s; dt = 1 s).

Recipe:
  * base cycle: seeded trips stop / accelerate / cruise / brake, peak 10..25 m/s;
    road power y = M v a + 0.5 rho_air CdA v^3 + C_rr M g v, M = 1900 kg
    (§IV-A "a 1900 kg vehicle"); engine speed from speed bands,
    800..4500 rpm.
  * scenario j: stop durations shifted by U{-5..5} s ("the times at which the
    vehicle stopped were also modified"), plus Gaussian white
    noise of 250 W and 50 rpm low-passed at 0.02 Hz (first-order
    filter), negative demand scaled by 0.4 ("40% is assumed to be
    recovered through regenerative braking").
  * engine i=1: f = a2 x^2 + a1 x + a0 with a2 = 2e-6 (1 + w/3000) W^-1,
    a1 = 2.4, a0 = 800 w/3000 W; g = 0; box [0, 100 kW]; c = +inf
    (PAPER.md:258-259, :275, :299).
  * battery i=2: f = 0; g = x + b2 x^2, b2 = 1e-6 (0.8 + 0.4 w/4500) W^-1;
    box [-50 kW, 50 kW]; c = dE = (0.6 - 0.5) E_max, E_max = 21.5 Ah * 350 V
    (350 V is the SPEC.md:475 reading).

Everything here is data generation; none of the method's arithmetic lives here.
Arrays are float64, C-contiguous, in the boundary layout:
  a2,a1,a0,b2,b1,b0 : [m][q][n]     lo,hi : [m][n]     y : [q][n]     c : [m]
"""

from __future__ import annotations

import numpy as np

BASE_SEED = 190310041
_CYCLE_STREAM = 0xC7C1E

# vehicle / powertrain constants
MASS = 1900.0  # kg
CDA = 0.7  # m^2
RHO_AIR = 1.2  # kg/m^3
C_RR = 0.01
G = 9.81
ENGINE_MAX = 1.0e5  # W, "100 kW ... engine"
MOTOR_MAX = 5.0e4  # W, "50 kW electric motor"
E_MAX = 21.5 * 3600.0 * 350.0  # J, 21.5 Ah at 350 V (SPEC.md:475 reading)
E0_FRAC, EN_FRAC = 0.6, 0.5
DELTA_E = (E0_FRAC - EN_FRAC) * E_MAX
REGEN = 0.4
NOISE_W, NOISE_RPM = 250.0, 50.0
LPF_A = float(np.exp(-2.0 * np.pi * 0.02 * 1.0))  # 0.02 Hz cutoff, 1 s sampling


def _segments(rng: np.random.Generator, length: int):
    """Draw trip segments until their total duration covers `length` steps.

    Returns a list of (kind, profile) where kind is 'stop' or 'move' and profile
    is the per-second speed (m/s) of that segment.  Drawing is sequential, so a
    longer `length` only appends segments (prefix-consistent)."""
    segs = []
    total = 0
    first = True
    while total < length:
        stop = int(rng.integers(5, 16)) if first else int(rng.integers(10, 41))
        first = False
        segs.append(("stop", np.zeros(stop)))
        vpk = rng.uniform(10.0, 25.0)
        acc = rng.uniform(0.8, 1.5)
        dec = rng.uniform(1.0, 2.0)
        cruise = int(rng.integers(20, 121))
        t_up = int(np.ceil(vpk / acc))
        up = np.minimum(acc * np.arange(1, t_up + 1), vpk)
        ph = rng.uniform(0, 2 * np.pi)
        tt = np.arange(cruise)
        mid = vpk + 1.0 * np.sin(2 * np.pi * tt / 40.0 + ph)
        t_dn = int(np.ceil(vpk / dec))
        dn = np.maximum(vpk - dec * np.arange(1, t_dn + 1), 0.0)
        move = np.concatenate([up, mid, dn])
        segs.append(("move", move))
        total += stop + move.size
    return segs


def _base_segments(length: int):
    rng = np.random.default_rng([BASE_SEED, _CYCLE_STREAM])
    return _segments(rng, length)


def _speed_from_segments(segs, shifts, length):
    parts = []
    si = 0
    for kind, prof in segs:
        if kind == "stop":
            d = max(1, prof.size + int(shifts[si]))
            si += 1
            parts.append(np.zeros(d))
        else:
            parts.append(prof)
    v = np.concatenate(parts)
    if v.size < length:  # shifts shortened the cycle: hold the final stop
        v = np.concatenate([v, np.zeros(length - v.size)])
    return v[:length]


def _road_power(v: np.ndarray) -> np.ndarray:
    a = np.diff(v, prepend=0.0)
    return MASS * v * a + 0.5 * RHO_AIR * CDA * v**3 + C_RR * MASS * G * v


def _engine_speed(v: np.ndarray) -> np.ndarray:
    """Speed-band gear model: rpm per (m/s) by band, clamped to [800, 4500]."""
    edges = np.array([7.0, 12.0, 18.0, 25.0])
    factor = np.array([300.0, 180.0, 130.0, 100.0, 85.0])
    w = factor[np.searchsorted(edges, v, side="right")] * v
    return np.clip(w, 800.0, 4500.0)


def _lpf(u: np.ndarray) -> np.ndarray:
    """First-order low-pass y[k] = a y[k-1] + (1-a) u[k] along the last axis."""
    from scipy.signal import lfilter

    return lfilter([1.0 - LPF_A], [1.0, -LPF_A], u, axis=-1)


def scenarios(n: int, j0: int, q: int, seed: int = BASE_SEED, noise: bool = True):
    """Demand y[q][n] (W) and engine speed w[q][n] (rpm) for scenarios j0..j0+q-1."""
    segs = _base_segments(n + 64)
    nstops = sum(1 for k, _ in segs if k == "stop")
    y = np.empty((q, n))
    w = np.empty((q, n))
    nz_y = np.empty((q, n))
    nz_w = np.empty((q, n))
    for r in range(q):
        rng = np.random.default_rng([seed, j0 + r])
        shifts = rng.integers(-5, 6, size=nstops) if noise else np.zeros(nstops, int)
        v = _speed_from_segments(segs, shifts, n)
        y[r] = _road_power(v)
        w[r] = _engine_speed(v)
        nz_y[r] = rng.standard_normal(n) * NOISE_W
        nz_w[r] = rng.standard_normal(n) * NOISE_RPM
    if noise:
        y += _lpf(nz_y)
        w += _lpf(nz_w)
    w = np.maximum(w, 0.0)
    y = np.where(y < 0.0, REGEN * y, y)
    return y, w


def _assemble(y, w_list, sources, n, q):
    """sources: list of dicts with keys kind ('engine'|'storage'), scale, cap."""
    m = len(sources)
    a2 = np.zeros((m, q, n)); a1 = np.zeros((m, q, n)); a0 = np.zeros((m, q, n))
    b2 = np.zeros((m, q, n)); b1 = np.zeros((m, q, n)); b0 = np.zeros((m, q, n))
    lo = np.zeros((m, n)); hi = np.zeros((m, n)); c = np.zeros(m)
    for i, s in enumerate(sources):
        w = w_list
        if s["kind"] == "engine":
            a2[i] = 2e-6 * (1.0 + w / 3000.0) * s.get("scale", 1.0)
            a1[i] = 2.4
            a0[i] = 800.0 * w / 3000.0
            lo[i] = 0.0
            hi[i] = ENGINE_MAX
        else:
            b2[i] = 1e-6 * (0.8 + 0.4 * w / 4500.0) * s.get("scale", 1.0)
            b1[i] = 1.0
            lo[i] = -MOTOR_MAX
            hi[i] = MOTOR_MAX
        c[i] = s["cap"]
    return dict(m=m, n=n, q=q, a2=a2, a1=a1, a0=a0, b2=b2, b1=b1, b0=b0,
                lo=lo, hi=hi, y=np.ascontiguousarray(y), c=c)


def phev_problem(n: int = 1000, q: int = 50, j0: int = 0, seed: int = BASE_SEED,
                 noise: bool = True):
    """Eq. (7) instance: m=2 (engine, battery)."""
    y, w = scenarios(n, j0, q, seed, noise)
    return _assemble(y, w, [dict(kind="engine", cap=np.inf),
                            dict(kind="storage", cap=DELTA_E)], n, q)


def toy_problem():
    """BASELINE.json configs[0]: n=10, m=2, q=1.  Window starts at the first
    step of scenario 0 with y >= 5 kW; c2 = 0.3 * sum_k max(y_k, 0) so the
    capacity constraint is active (SURVEY.md §8(d) 'Toy')."""
    y, w = scenarios(600, 0, 1)
    k0 = int(np.argmax(y[0] >= 5000.0))
    y = y[:, k0:k0 + 10].copy()
    w = w[:, k0:k0 + 10].copy()
    cap = 0.3 * float(np.maximum(y, 0).sum())
    return _assemble(y, w, [dict(kind="engine", cap=np.inf),
                            dict(kind="storage", cap=cap)], 10, 1)


def horizon_problem(n: int, seed: int = BASE_SEED):
    """BASELINE.json configs[2]: m=4, q=1 (two engine-like sources with a2
    scaled x1 and x1.5, two storage-like with c = 0.1 sum_k max(y_k, 0))."""
    y, w = scenarios(n, 0, 1, seed)
    cap = 0.1 * float(np.maximum(y, 0).sum())
    return _assemble(y, w, [dict(kind="engine", cap=np.inf, scale=1.0),
                            dict(kind="engine", cap=np.inf, scale=1.5),
                            dict(kind="storage", cap=cap, scale=1.0),
                            dict(kind="storage", cap=cap, scale=1.5)], n, 1)


def random_problem(m: int, n: int, q: int, seed: int, scale: float = 1.0,
                   cap_slack: float = 0.05, general: bool = True):
    """Small generic convex instance (every source has both f and g, nonzero
    b0, random bounds) for oracle pins and ragged-tail parity cases.  Units are
    O(scale).  Feasible by construction: a random point x_f inside the box
    meets the demand y = sum_i x_f - U[0, 0.3] and uses the capacity
    c_i = max_j sum_k g(x_f) + cap_slack n scale, so the cost (which pulls
    the sources towards larger x) usually makes the capacity bind."""
    rng = np.random.default_rng([seed, 0xA11])
    a2 = rng.uniform(0.2, 2.0, (m, q, n)) / scale
    a1 = rng.uniform(-3.0, -0.5, (m, q, n))
    a0 = rng.uniform(-1.0, 1.0, (m, q, n)) * scale
    if general:
        b2 = rng.uniform(0.0, 0.5, (m, q, n)) / scale
        b1 = rng.uniform(0.2, 1.5, (m, q, n))
        b0 = rng.uniform(-0.2, 0.2, (m, q, n)) * scale
    else:
        b2 = np.zeros((m, q, n)); b1 = np.ones((m, q, n)); b0 = np.zeros((m, q, n))
    lo = -rng.uniform(0.5, 2.0, (m, n)) * scale
    hi = rng.uniform(0.5, 3.0, (m, n)) * scale
    xf = rng.uniform(lo[:, None, :], hi[:, None, :], (m, q, n))
    y = xf.sum(axis=0) - rng.uniform(0.0, 0.3, (q, n)) * scale
    gx = (b2 * xf + b1) * xf + b0
    c = gx.sum(axis=2).max(axis=1) + cap_slack * n * scale
    return dict(m=m, n=n, q=q, a2=a2, a1=a1, a0=a0, b2=b2, b1=b1, b0=b0,
                lo=lo, hi=hi, y=y, c=c)


# ---------------------------------------------------------------------------
# Algorithm 2 (shrinking-horizon supervisory control) data
SUPERVISOR_SAMPLE_BASE = 1 << 20  # scenario streams of instant t: j = BASE + t * 4096 + r
TRUE_STREAM = (1 << 20) - 1       # the realised drive (one extra stream)


def supervisor_problem(N: int, q: int, t: int, delta_e: float, seed: int = BASE_SEED):
    """Step-1/2 data of Algorithm 2 at sampling instant t of an N-step trip:
    q fresh demand / speed samples of the remaining horizon k = t..N-1
    (n = N - t), engine and battery maps from the sampled speeds, and the
    battery capacity c2 = dE = E_t - E_n."""
    if not 0 <= t < N:
        raise ValueError("t must be in [0, N)")
    y, w = scenarios(N, SUPERVISOR_SAMPLE_BASE + t * 4096, q, seed)
    y = np.ascontiguousarray(y[:, t:])
    w = np.ascontiguousarray(w[:, t:])
    return _assemble(y, w, [dict(kind="engine", cap=np.inf),
                            dict(kind="storage", cap=float(delta_e))], N - t, q)


def realised_drive(N: int, seed: int = BASE_SEED):
    """The drive that actually happens (demand y[N], speed w[N]): one more
    independent sample of the same distribution."""
    y, w = scenarios(N, TRUE_STREAM, 1, seed)
    return y[0].copy(), w[0].copy()


def battery_loss_coeffs(w):
    """b2 of the battery map g = x + b2 x^2 at engine speed w (same map as the
    storage source of _assemble)."""
    return 1e-6 * (0.8 + 0.4 * np.asarray(w) / 4500.0)
