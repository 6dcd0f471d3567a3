"""AdmmSolver: the public Python API over the C ABI (include/admm.h).

Device memory comes from torch (one uint8 workspace tensor per context),
streams from torch.cuda; everything else is the library's CUDA path.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from ._lib import AdmmError  # noqa: F401

_F_KEYS = ("a2", "a1", "a0")
_G_KEYS = ("b2", "b1", "b0")


def _stack(parts):
    import torch

    if isinstance(parts[0], torch.Tensor):
        return torch.stack([p.to(torch.float64) for p in parts]).contiguous()
    return np.ascontiguousarray(np.stack([np.asarray(p, dtype=np.float64) for p in parts]))


def _arr(a):
    import torch

    if isinstance(a, torch.Tensor):
        return a.to(torch.float64).contiguous()
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


class AdmmSolver:
    """One ADMM context for m sources, n steps, q_total scenarios on one GPU, or
    this rank's part when `dist` (admm_dist, see dist.make_dist) is given: its
    scenario shard [j_begin, j_end) (mode ADMM_SHARD_SCENARIOS) or its horizon
    block [k_begin, k_end) of every scenario (ADMM_SHARD_HORIZON).  Arrays passed
    in and returned are this rank's part ([m][q][n] with the local q and n)."""

    def __init__(self, m, n, q_total, device=0, dist=None, stream=None, params=None,
                 coeff_bits=64, **param_kw):
        import torch

        self.m, self.n_total, self.q_total = int(m), int(n), int(q_total)
        self.device = int(device)
        self.q = int(dist.j_end - dist.j_begin) if dist is not None else self.q_total
        self.j0 = int(dist.j_begin) if dist is not None else 0
        hz = dist is not None and int(dist.mode) == _lib.ADMM_SHARD_HORIZON
        self.k0 = int(dist.k_begin) if hz else 0
        self.n = int(dist.k_end - dist.k_begin) if hz else self.n_total  # local horizon
        nbytes = _lib.admm_workspace_bytes(self.m, self.n, self.q, self.device)
        if nbytes == 0:
            raise AdmmError(_lib.ADMM_ERR_INVALID, "bad dimensions")
        # torch supplies the device memory (256-byte aligned by the caching allocator)
        self.workspace = torch.empty(nbytes, dtype=torch.uint8,
                                     device=torch.device("cuda", self.device))
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.ctx = _lib.admm_create(self.m, self.n_total, self.q_total, dist, self.device,
                                    self.workspace, self.stream)
        p = params if params is not None else _lib.admm_default_params()
        for k, v in param_kw.items():
            if k == "rho":
                for l in range(4):
                    p.rho[l] = v[l]
            else:
                setattr(p, k, v)
        _lib.admm_set_params(self.ctx, p)
        if coeff_bits != 64:
            _lib.admm_set_coeff_precision(self.ctx, coeff_bits)

    # -------------------------------------------------------------- problem
    def set_coeff_precision(self, bits):
        """F2: store a2, a1, b2, b1 in fp32 (bits=32) or fp64 (64) from the next
        set_problem on (include/admm.h: admm_set_coeff_precision)."""
        _lib.admm_set_coeff_precision(self.ctx, bits)

    @property
    def coeff_bits(self):
        return _lib.admm_get_coeff_precision(self.ctx)

    def set_problem(self, prob):
        """prob: dict with a2,a1,a0,b2,b1,b0 [m][q][n], lo,hi [m][n], y [q][n],
        c [m] (numpy = host, torch = host or device)."""
        f = _stack([prob[k] for k in _F_KEYS])
        g = _stack([prob[k] for k in _G_KEYS])
        self._keep = (f, g, _arr(prob["lo"]), _arr(prob["hi"]), _arr(prob["y"]), _arr(prob["c"]))
        _lib.admm_set_problem(self.ctx, *self._keep)
        self._keep = None

    def set_problem_packed(self, f, g, lo, hi, y, c):
        """Same as set_problem with the coefficient blocks already packed as
        f = [3][m][q][n] (a2,a1,a0) and g = [3][m][q][n] (b2,b1,b0) -- no
        host-side staging copy (e.g. pinned torch tensors)."""
        _lib.admm_set_problem(self.ctx, f, g, lo, hi, y, c)

    def reset(self):
        """Back to the initial state (reading G19) without re-sending data."""
        _lib.admm_reset(self.ctx)

    def set_params(self, **kw):
        p = _lib.admm_get_params(self.ctx)
        for k, v in kw.items():
            if k == "rho":
                for l in range(4):
                    p.rho[l] = v[l]
            else:
                setattr(p, k, v)
        _lib.admm_set_params(self.ctx, p)

    @property
    def params(self):
        return _lib.admm_get_params(self.ctx)

    # ------------------------------------------------------------ iterations
    def iterate(self, iters):
        _lib.admm_iterate(self.ctx, iters)

    def solve(self, r_bar, sigma_bar=1e-2, max_iter=200000):
        st, info = _lib.admm_solve(self.ctx, r_bar, sigma_bar, max_iter)
        info["converged"] = st == _lib.ADMM_OK
        return info

    # ---------------------------------------------------------------- output
    def solution(self, out_x=None, out_x1=None):
        """Returns (x, x1, info); x/x1 are host numpy unless out_* buffers given."""
        x = out_x if out_x is not None else np.empty((self.m, self.q, self.n))
        x1 = out_x1 if out_x1 is not None else np.empty(self.m)
        info = _lib.admm_get_solution(self.ctx, x, x1)
        return x, x1, info

    def state(self):
        m, q, n = self.m, self.q, self.n
        S = dict(x=np.empty((m, q, n)), z=np.empty((m, q, n)), lam=np.empty((m, q, n)),
                 s=np.empty((q, n)), mu=np.empty((q, n)), h=np.empty((m, q)),
                 p=np.empty((m, q)), nu=np.empty((m, q)), x1=np.empty(m))
        _lib.admm_get_state(self.ctx, **S)
        return S

    def set_state(self, S):
        _lib.admm_set_state(self.ctx, *[_arr(S[k]) for k in
                                        ("x", "z", "lam", "s", "mu", "h", "p", "nu", "x1")])

    def history(self):
        return _lib.admm_get_history(self.ctx)

    def timing(self):
        """(average device ms per iteration, device ms of the last call)."""
        return _lib.admm_get_timing(self.ctx)

    def engine(self):
        """(engine id of the last iterate/solve, kernels launched so far)."""
        return _lib.admm_get_engine(self.ctx)

    def close(self):
        if getattr(self, "ctx", None) is not None and self.ctx.value:
            _lib.admm_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def quartic_minimize_batch(A, B, C, D, lo=None, hi=None, out=None, box_mode=0, stream=None):
    import torch

    if out is None:
        out = torch.empty_like(A)
    _lib.quartic_minimize_batch(A, B, C, D, lo, hi, out, box_mode, stream)
    return out
