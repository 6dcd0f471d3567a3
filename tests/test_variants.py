"""F3: nominal Eq. (1) and the open-loop robust variant
 as q = 1 instances, checked on the oracle (CPU) and on the
GPU path against the oracle."""

import numpy as np
import pytest

import oracle
import synth
from paper_1903_10041_b200.variants import nominal_problem, open_loop_problem


def _sampled(n=200, q=6):
    P = synth.phev_problem(n, q)
    P["c"] = np.array([np.inf, 0.02 * synth.DELTA_E])  # short horizon: make the budget bind
    return P


def test_open_loop_instance_shape_and_demand():
    P = _sampled()
    Q = open_loop_problem(P)
    assert Q["q"] == 1 and Q["y"].shape == (1, P["n"]) and Q["a2"].shape == (2, 1, P["n"])
    np.testing.assert_array_equal(Q["y"][0], P["y"].max(axis=0))
    np.testing.assert_allclose(Q["b2"][:, 0], P["b2"].mean(axis=1))
    N = nominal_problem(P, j=3)
    np.testing.assert_array_equal(N["y"][0], P["y"][3])
    np.testing.assert_array_equal(N["a2"][:, 0], P["a2"][:, 3])


def test_open_loop_solution_meets_every_sampled_demand():
    P = _sampled()
    Q = open_loop_problem(P)
    r_bar = 1e-6 * Q["c"][1]
    o = oracle.Oracle(Q, oracle.default_params(r_bar=r_bar))
    info, _ = o.solve(200000)
    assert info["status"] == 0
    x = o.x[:, 0, :]
    # robust feasibility: the single sequence covers max_j y_k^{(j)} hence every sample
    assert np.all(x.sum(axis=0) >= P["y"].max(axis=0) - 10 * r_bar)
    g = (Q["b2"][1, 0] * x[1] + Q["b1"][1, 0]) * x[1] + Q["b0"][1, 0]
    assert g.sum() <= Q["c"][1] * (1 + 1e-6)
    # the open-loop plan is dearer than planning for the mean-map nominal demand of
    # any single sample (its feasible set is a subset of each one's)
    for j in (0, 2, 5):
        Nj = nominal_problem(P, j)
        Nj.update({k: Q[k] for k in ("a2", "a1", "a0", "b2", "b1", "b0")})
        oj = oracle.Oracle(Nj, oracle.default_params(r_bar=r_bar))
        ij, _ = oj.solve(200000)
        assert ij["objective"] <= info["objective"] * (1 + 1e-6)


@pytest.mark.gpu
def test_open_loop_gpu_matches_oracle():
    from paper_1903_10041_b200.variants import solve

    P = _sampled()
    for Q in (open_loop_problem(P), nominal_problem(P, 1)):
        r_bar = 1e-6 * Q["c"][1]
        o = oracle.Oracle(Q, oracle.default_params(r_bar=r_bar))
        io, _ = o.solve(200000)
        x, ig = solve(Q, r_bar)
        assert ig["converged"]
        assert abs(ig["iterations"] - io["iterations"]) <= 10
        assert abs(ig["objective"] - io["objective"]) <= 1e-6 * abs(io["objective"])
        assert np.abs(x - o.x[:, 0, :]).max() <= 1e-6 * 1e5
