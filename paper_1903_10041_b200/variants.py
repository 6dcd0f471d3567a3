"""Problem variants of arXiv 1903.10041 that reuse the hot path.

* nominal Eq. (1): one demand sequence, no scenarios -- the q = 1
  instance of Eq. (2), whose consensus constraint x_1^{(i,1)} = x_1^{(i)} is vacuous;
* open-loop robust variant: "optimizes a single sequence
  {x_k^{(i)}} for each i with the predicted power demand sequence replaced by
  {max_j y_k^{(j)}}".  Eq. (1) has scenario-independent maps, the sampled PHEV
  maps are not (they follow the sampled speeds): reading F3-a, the open-loop
  instance uses the scenario mean of each coefficient (maps="mean"), or the
  maps of one scenario (maps=j).

The transformation is input preparation on the host (a max and a mean over
the q samples); the solve is the library's q = 1 path on the GPU.
"""

from __future__ import annotations

import numpy as np

_COEF = ("a2", "a1", "a0", "b2", "b1", "b0")


def nominal_problem(P, j=0):
    """Eq. (1) instance from scenario j of a sampled problem (its demand and maps)."""
    Q = {k: P[k] for k in ("m", "lo", "hi", "c")}
    Q.update(n=P["n"], q=1)
    for k in _COEF:
        Q[k] = np.ascontiguousarray(P[k][:, j:j + 1, :])
    Q["y"] = np.ascontiguousarray(P["y"][j:j + 1, :])
    return Q


def open_loop_problem(P, maps="mean"):
    """Open-loop robust instance: demand max_j y_k^{(j)}, q = 1."""
    Q = {k: P[k] for k in ("m", "lo", "hi", "c")}
    Q.update(n=P["n"], q=1)
    for k in _COEF:
        if maps == "mean":
            Q[k] = np.ascontiguousarray(P[k].mean(axis=1, keepdims=True))
        else:
            Q[k] = np.ascontiguousarray(P[k][:, int(maps):int(maps) + 1, :])
    Q["y"] = np.ascontiguousarray(P["y"].max(axis=0, keepdims=True))
    return Q


def solve(Q, r_bar, sigma_bar=1e-2, max_iter=200000, device=0, **params):
    """Solve a q = 1 variant on the GPU; returns (x [m][n], info)."""
    from .solver import AdmmSolver

    s = AdmmSolver(Q["m"], Q["n"], 1, device=device, r_bar=r_bar, sigma_bar=sigma_bar, **params)
    try:
        s.set_problem(Q)
        info = s.solve(r_bar, sigma_bar, max_iter)
        x, x1, sol = s.solution()
        return x[:, 0, :].copy(), {**info, **sol}
    finally:
        s.close()
