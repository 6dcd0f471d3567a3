"""Algorithm 2 (shrinking-horizon supervisory control; SURVEY.md
§8(f) F1): the controller loop of paper_1903_10041_b200.supervisor run on the CPU
oracle (no GPU) and, marked gpu, on the CUDA path against the oracle loop."""

import numpy as np
import pytest

import oracle
import synth
from paper_1903_10041_b200.supervisor import ShrinkingHorizonController, shift_state, with_zeta


def oracle_backend(P, r_bar, sigma_bar, max_iter, warm=None, rho=None):
    prm = oracle.default_params(r_bar=r_bar, sigma_bar=sigma_bar)
    if rho is not None:
        prm["rho0"] = tuple(float(v) for v in rho)
    o = oracle.Oracle(P, prm)
    if warm is not None:  # the oracle's state arrays are shared with its C core
        for k in ("x", "z", "lam", "s", "mu", "h", "p", "nu", "x1"):
            getattr(o, k)[...] = warm[k]
    info, _ = o.solve(max_iter)
    return with_zeta(o.state(), P), info


N, Q = 120, 4


def test_shift_state_keeps_reduced_state_identities():
    P0 = synth.supervisor_problem(N, Q, 0, synth.DELTA_E)
    S, info = oracle_backend(P0, 1e-6 * synth.DELTA_E, 1e-2, 20000)
    P1 = synth.supervisor_problem(N, Q, 1, synth.DELTA_E)
    W = shift_state(S, P1)
    assert W["x"].shape == (2, Q, N - 1) and W["s"].shape == (Q, N - 1)
    g = (P1["b2"] * W["x"] + P1["b1"]) * W["x"] + P1["b0"]
    off = W["z"] - g
    assert np.abs(off - off[:, :, :1]).max() <= 1e-9 * max(1.0, np.abs(g).max())  # I1 (z)
    # I1 (lam): constant over k up to the rounding of the literal update lam += z - g(x)
    assert np.abs(W["lam"] - W["lam"][:, :, :1]).max() <= 1e-15 * 8 * np.abs(W["z"]).max()
    ys = np.abs(P1["y"]).max()  # I2 up to the rounding of the literal (6e)/(6f)
    assert np.minimum(np.abs(W["s"]), np.abs(W["mu"])).max() <= 1e-12 * ys
    assert W["mu"].min() >= -1e-12 * ys
    assert np.all((W["x"] >= P1["lo"][:, None, :]) & (W["x"] <= P1["hi"][:, None, :]))
    np.testing.assert_array_equal(W["x1"], W["x"][:, :, 0].mean(axis=1))
    assert np.all(W["nu"] == 0.0)


def test_controller_loop_on_oracle():
    steps = 4
    warm = ShrinkingHorizonController(N, Q, backend=oracle_backend, warm_start=True)
    cold = ShrinkingHorizonController(N, Q, backend=oracle_backend, warm_start=False)
    lw, lc = warm.run(steps), cold.run(steps)
    E = synth.E0_FRAC * synth.E_MAX
    for t, (a, b) in enumerate(zip(lw, lc)):
        assert a["t"] == t and a["n"] == N - t             # the horizon shrinks by one step
        assert a["status"] == 0 and b["status"] == 0       # converged (r < r_bar, sigma < sigma_bar)
        assert abs(a["E"] - E) <= 1e-6 * E                 # E_{t+1} = E_t - g(x_1^(2))
        E -= a["battery_energy"]
        assert 0.0 <= a["x1"][0] <= synth.phev.ENGINE_MAX
        assert -synth.phev.MOTOR_MAX <= a["x1"][1] <= synth.phev.MOTOR_MAX
        assert a["dE"] == pytest.approx(a["E"] - synth.EN_FRAC * synth.E_MAX)
        # the applied step meets every sampled demand (Eq. (7) demand row at k = 1,
        # within the primal tolerance r_bar = 1e-6 dE)
        assert a["x1"].sum() >= a["demand_samples_max"] - 1e-6 * a["dE"]
        # warm and cold starts reach the same optimal value (the battery split is not
        # unique when the energy budget does not bind, so x1 itself may differ)
        assert abs(a["objective"] - b["objective"]) <= 1e-5 * abs(b["objective"])
    assert lw[0]["iterations"] == lc[0]["iterations"]      # instant 0: no warm start yet
    assert [r["warm"] for r in lw] == [False] + [True] * (steps - 1)
    assert not any(r["warm"] for r in lc)


@pytest.mark.gpu
def test_controller_loop_gpu_matches_oracle():
    from paper_1903_10041_b200.supervisor import GpuBackend

    steps = 4
    gpu = ShrinkingHorizonController(N, Q, backend=GpuBackend(), warm_start=True)
    orc = ShrinkingHorizonController(N, Q, backend=oracle_backend, warm_start=True)
    lg, lo = gpu.run(steps), orc.run(steps)
    for a, b in zip(lg, lo):
        assert a["status"] == 0
        assert abs(a["iterations"] - b["iterations"]) <= 10  # one check period at most
        assert np.abs(a["x1"] - b["x1"]).max() <= 1e-6 * synth.phev.ENGINE_MAX
        assert abs(a["E"] - b["E"]) <= 1e-9 * b["E"] + 1e-3
        assert abs(a["objective"] - b["objective"]) <= 1e-6 * abs(b["objective"])
