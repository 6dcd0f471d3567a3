"""Algorithm 2 of arXiv 1903.10041 -- shrinking-horizon supervisory PHEV control
(PAPER.md:284-295), SURVEY.md §8(f) row F1.

At each sampling instant t of an N-step trip:
  1. draw q demand samples of the remaining horizon k = t..N-1 (synth),
  2. set dE = E_t - E_n and build f^{(1,j)}, g^{(2,j)} from the sampled speeds,
  3. solve Eq. (7) by the ADMM iteration (6a)-(6i) until r < r_bar, sigma < sigma_bar
     (r_bar = 1e-6 dE, sigma_bar = 1e-2) -- on the GPU, through the
     C ABI (AdmmSolver), optionally warm-started from the previous instant's
     solution shifted by one step (admm_set_state),
  4. apply x_1^{(1)}, x_1^{(2)}: the battery energy falls by g^{(2)}(x_1^{(2)}) at
     the realised speed (E_{t+1} = E_t - g), the engine burns f^{(1)}(x_1^{(1)}).

The loop itself is host bookkeeping (array slicing, energy accounting); every
step of the ADMM runs in the library's kernels.  `backend` is injectable so the
tests can run the identical loop on the CPU oracle.
"""

from __future__ import annotations

import time

import numpy as np

import synth


def shift_state(S, P_new):
    """Warm start for instant t+1 from the state S of instant t: drop step k = 0
    and keep the rest (x, lam, s, mu shifted; per-row h, p kept; nu = 0 for the
    new consensus cell; x1 = mean_j of the new first step), with z rebuilt so
    that z - g(x) is the old per-row offset zeta under the NEW maps g (identity
    I1 of the reduced state)."""
    if "zeta" not in S:
        raise ValueError("state must carry zeta (see with_zeta)")
    x = np.ascontiguousarray(S["x"][:, :, 1:])
    lam = np.ascontiguousarray(S["lam"][:, :, 1:])
    g_new = (P_new["b2"] * x + P_new["b1"]) * x + P_new["b0"]
    z = g_new + S["zeta"][:, :, None]
    return dict(x=x, z=np.ascontiguousarray(z), lam=lam,
                s=np.ascontiguousarray(S["s"][:, 1:]), mu=np.ascontiguousarray(S["mu"][:, 1:]),
                h=S["h"].copy(), p=S["p"].copy(), nu=np.zeros_like(S["nu"]),
                x1=x[:, :, 0].mean(axis=1))


def with_zeta(S, P):
    """Attach the per-row offset zeta = z - g(x) (taken at k = 0) to a literal state."""
    g = (P["b2"] * S["x"] + P["b1"]) * S["x"] + P["b0"]
    return dict(S, zeta=(S["z"] - g)[:, :, 0].copy())


class GpuBackend:
    """Solve one instant on the GPU through the C ABI (AdmmSolver)."""

    def __init__(self, device=0, exec_mode=0):
        self.device = device
        self.exec_mode = exec_mode

    def __call__(self, P, r_bar, sigma_bar, max_iter, warm=None, rho=None):
        from .solver import AdmmSolver

        kw = dict(r_bar=r_bar, sigma_bar=sigma_bar, exec_mode=self.exec_mode)
        if rho is not None:
            kw["rho"] = tuple(rho)
        s = AdmmSolver(P["m"], P["n"], P["q"], device=self.device, **kw)
        try:
            s.set_problem(P)
            if warm is not None:
                s.set_state(warm)
            info = s.solve(r_bar, sigma_bar, max_iter)
            S = with_zeta(s.state(), P)
            x, x1, sol = s.solution()
            return S, {**info, "objective": sol.get("objective", info.get("objective"))}
        finally:
            s.close()


class ShrinkingHorizonController:
    """Algorithm 2 on the synthetic PHEV cycle (N steps of 1 s)."""

    def __init__(self, N, q, backend=None, warm_start=True, r_rel=1e-6, sigma_bar=1e-2,
                 max_iter=50000, seed=synth.BASE_SEED):
        self.N, self.q = int(N), int(q)
        self.backend = backend if backend is not None else GpuBackend()
        self.warm_start = bool(warm_start)
        self.r_rel, self.sigma_bar, self.max_iter = float(r_rel), float(sigma_bar), int(max_iter)
        self.seed = seed
        self.t = 0
        self.E = synth.E0_FRAC * synth.E_MAX  # E_0 = 60 % of capacity
        self.En = synth.EN_FRAC * synth.E_MAX  # E_n = 50 %
        self.y_true, self.w_true = synth.realised_drive(self.N, seed)
        self._state = None
        self._rho = None
        self.log = []

    def step(self):
        if self.t >= self.N:
            raise StopIteration("trip finished")
        t = self.t
        dE = self.E - self.En                                        # step 2
        P = synth.supervisor_problem(self.N, self.q, t, dE, self.seed)  # steps 1-2
        warm = None
        if self.warm_start and self._state is not None:
            warm = shift_state(self._state, P)
        r_bar = self.r_rel * max(abs(dE), 1.0)
        t0 = time.perf_counter()
        S, info = self.backend(P, r_bar, self.sigma_bar, self.max_iter, warm=warm,
                               rho=self._rho if warm is not None else None)  # step 3
        dt = time.perf_counter() - t0
        x1 = np.array(S["x1"], dtype=float)
        # step 4: apply x_1^{(1)}, x_1^{(2)} against the realised speed
        b2 = float(synth.battery_loss_coeffs(self.w_true[t]))
        used = x1[1] + b2 * x1[1] ** 2
        self.log.append(dict(t=t, n=P["n"], dE=dE, E=self.E, x1=x1, battery_energy=used,
                             demand=float(self.y_true[t]),
                             demand_samples_max=float(P["y"][:, 0].max()),
                             iterations=int(info["iterations"]),
                             status=int(info["status"]), rho=list(info["rho"]),
                             objective=float(info["objective"]), seconds=dt,
                             warm=warm is not None))
        self.E -= used
        self._state = S
        self._rho = info["rho"]
        self.t += 1
        return self.log[-1]

    def run(self, steps):
        return [self.step() for _ in range(int(steps))]
