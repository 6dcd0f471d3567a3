"""The seeded input generators: seeding contract and the paper's recipe
(PAPER.md:299-306).  No GPU."""

import json
import os

import numpy as np

import synth
from synth import phev

PAPER = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_params.json")))


def test_scenario_rows_independent_of_q_and_shard():
    a = synth.phev_problem(300, 6)
    b = synth.phev_problem(300, 2, j0=3)
    for k in ("a2", "a0", "b2"):
        assert np.array_equal(a[k][:, 3:5], b[k])
    assert np.array_equal(a["y"][3:5], b["y"])


def test_horizon_prefix_consistent_base_cycle():
    y1, _ = phev.scenarios(200, 0, 1, noise=False)
    y2, _ = phev.scenarios(500, 0, 1, noise=False)
    assert np.array_equal(y1[0], y2[0, :200])


def test_paper_constants():
    assert phev.MASS == PAPER["vehicle_mass_kg"]["value"]
    assert phev.ENGINE_MAX == PAPER["engine_max_W"]["value"]
    assert phev.MOTOR_MAX == PAPER["motor_max_W"]["value"]
    assert phev.NOISE_W == PAPER["noise_W"]["value"]
    assert phev.NOISE_RPM == PAPER["noise_rpm"]["value"]
    assert phev.REGEN == PAPER["regen_frac"]["value"]
    assert abs(phev.DELTA_E - 0.1 * PAPER["battery_Ah"]["value"] * 3600 * 350) < 1e-6
    assert abs(phev.LPF_A - np.exp(-2 * np.pi * PAPER["lpf_cutoff_Hz"]["value"])) < 1e-15


def test_phev_structure():
    P = synth.phev_problem(400, 3)
    assert P["m"] == 2 and P["a2"].shape == (2, 3, 400)
    # g^(1) = 0 and f^(2) = 0; convex (Assumption 1)
    assert not P["b2"][0].any() and not P["b1"][0].any()
    assert not P["a2"][1].any() and not P["a1"][1].any()
    assert (P["a2"] >= 0).all() and (P["b2"] >= 0).all()
    assert np.all(P["lo"][0] == 0) and np.all(P["hi"][0] == 1e5)
    assert np.isinf(P["c"][0]) and P["c"][1] == phev.DELTA_E
    # demand within the combined source limits
    assert P["y"].max() < 1.5e5


def test_regen_and_noise():
    yc, _ = phev.scenarios(2000, 0, 4, noise=False)
    assert (yc < 0).any()
    # without noise the negative part is exactly 0.4 x the road power
    segs = phev._base_segments(2000 + 64)
    v = phev._speed_from_segments(segs, np.zeros(100, int), 2000)
    road = phev._road_power(v)
    assert np.allclose(yc[0], np.where(road < 0, 0.4 * road, road))
    # noise: low-passed white noise of 250 W: std 250 sqrt((1-a)/(1+a))
    rng = np.random.default_rng(0)
    u = rng.standard_normal((8, 20000)) * 250
    f = phev._lpf(u)
    want = 250 * np.sqrt((1 - phev.LPF_A) / (1 + phev.LPF_A))
    assert abs(f.std() / want - 1) < 0.05
    # attenuation above the 0.02 Hz cutoff
    P = np.abs(np.fft.rfft(f, axis=1)) ** 2
    fr = np.fft.rfftfreq(20000, 1.0)
    assert P[:, fr > 0.1].mean() < 0.5 * P[:, (fr > 0) & (fr < 0.01)].mean()


def test_toy_window():
    T = synth.toy_problem()
    assert T["n"] == 10 and T["q"] == 1 and T["y"][0, 0] >= 5000
    assert T["c"][1] == 0.3 * np.maximum(T["y"], 0).sum()


def test_horizon_problem():
    H = synth.horizon_problem(500)
    assert H["m"] == 4 and H["q"] == 1
    assert np.allclose(H["a2"][1], 1.5 * H["a2"][0])
    assert np.isinf(H["c"][:2]).all() and np.isfinite(H["c"][2:]).all()
