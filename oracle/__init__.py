"""ctypes binding of the plain C CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package.  The product
package paper_1903_10041_b200 never imports it, and this package never imports
the product.  See oracle.h for the cited algorithm.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SO_OMP = os.path.join(_HERE, "liboracle_omp.so")  # same source, OpenMP loops (CPU-parallel baseline)
_SRC = [os.path.join(_HERE, "oracle.c"), os.path.join(_HERE, "oracle.h")]

BOX_PROJECT, BOX_EXACT = 0, 1
HIST_COLS = 16

# paper defaults
PAPER_RHO0 = (1e-4, 2e-6, 5e-6, 5e-6)
PAPER_TAU = 1.1


def build(force: bool = False) -> str:
    """Compile liboracle.so (serial) and liboracle_omp.so (the same source with its
    OpenMP loops on) with gcc (plain C, -O2 -ffp-contract=off)."""
    for so, extra in ((_SO, []), (_SO_OMP, ["-fopenmp"])):
        if not force and os.path.exists(so):
            so_m = os.path.getmtime(so)
            if all(os.path.getmtime(s) <= so_m for s in _SRC):
                continue
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11", "-fPIC",
               *extra, "-shared", "-o", so + ".tmp", _SRC[0], "-lm"]
        subprocess.check_call(cmd)
        os.replace(so + ".tmp", so)
    return _SO


_libs = {}


class _Problem(C.Structure):
    _fields_ = [("m", C.c_int), ("n", C.c_long), ("q", C.c_long), ("q_total", C.c_long)] + [
        (nm, C.POINTER(C.c_double))
        for nm in ("a2", "a1", "a0", "b2", "b1", "b0", "lo", "hi", "y", "c")
    ] + [("n_total", C.c_long), ("k_off", C.c_long)]


class _State(C.Structure):
    _fields_ = [(nm, C.POINTER(C.c_double))
                for nm in ("x", "z", "lam", "s", "mu", "h", "p", "nu", "x1")] + [
        ("rho", C.c_double * 4), ("iter", C.c_long)]


class _Params(C.Structure):
    _fields_ = [("rho0", C.c_double * 4), ("tau", C.c_double), ("hi_ratio", C.c_double),
                ("lo_ratio", C.c_double), ("r_bar", C.c_double), ("sigma_bar", C.c_double),
                ("check_every", C.c_int), ("adapt_rho", C.c_int),
                ("rescale_duals", C.c_int), ("box_mode", C.c_int)]


class _Info(C.Structure):
    _fields_ = [("iterations", C.c_long), ("r", C.c_double), ("sigma", C.c_double),
                ("objective", C.c_double), ("rho", C.c_double * 4), ("status", C.c_int),
                ("ties", C.c_long), ("hist_rows", C.c_long)]


REDUCE_FN = C.CFUNCTYPE(None, C.POINTER(C.c_double), C.c_int, C.c_int, C.c_void_p)


def lib(omp: bool = False):
    """The serial oracle, or (omp=True) its OpenMP build; bitwise-identical results."""
    _lib = _libs.get(omp)
    if _lib is None:
        build()
        _lib = _libs[omp] = C.CDLL(_SO_OMP if omp else _SO)
        d = C.c_double
        _lib.orc_set_threads.argtypes = [C.c_int]
        _lib.orc_set_threads.restype = C.c_int
        pd = C.POINTER(C.c_double)
        _lib.orc_cubic_roots.argtypes = [d, d, d, pd, C.POINTER(C.c_int)]
        _lib.orc_cubic_roots.restype = C.c_int
        _lib.orc_quartic_argmin.argtypes = [d, d, d, d, C.POINTER(C.c_int)]
        _lib.orc_quartic_argmin.restype = d
        _lib.orc_quartic_boxmin.argtypes = [d, d, d, d, d, d, C.c_int, C.POINTER(C.c_int)]
        _lib.orc_quartic_boxmin.restype = d
        _lib.orc_quartic_batch.argtypes = [pd] * 7 + [C.c_long, C.c_int, C.POINTER(C.c_long)]
        _lib.orc_build_quartic.argtypes = [d] * 8 + [pd, C.c_int, d, d, pd]
        _lib.orc_validate.argtypes = [C.POINTER(_Problem), C.c_char_p, C.c_int]
        _lib.orc_validate.restype = C.c_int
        _lib.orc_init.argtypes = [C.POINTER(_Problem), C.POINTER(_State), C.POINTER(_Params),
                                  REDUCE_FN, C.c_void_p]
        _lib.orc_run.argtypes = [C.POINTER(_Problem), C.POINTER(_State), C.POINTER(_Params),
                                 C.c_long, C.c_int, C.POINTER(_Info), pd, C.c_long,
                                 REDUCE_FN, C.c_void_p]
        _lib.orc_run.restype = C.c_int
        _lib.orc_objective.argtypes = [C.POINTER(_Problem), pd, REDUCE_FN, C.c_void_p]
        _lib.orc_objective.restype = d
    return _lib


def _p(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


# ----------------------------------------------------------------- Algorithm 1
def cubic_roots(b, c, d):
    r = (C.c_double * 3)()
    br = C.c_int()
    nr = lib().orc_cubic_roots(b, c, d, r, C.byref(br))
    return [r[i] for i in range(nr)], br.value


def quartic_argmin(A, B, Cc, D):
    t = C.c_int()
    x = lib().orc_quartic_argmin(A, B, Cc, D, C.byref(t))
    return x, bool(t.value)


def quartic_boxmin(A, B, Cc, D, lo, hi, mode=BOX_PROJECT):
    t = C.c_int()
    x = lib().orc_quartic_boxmin(A, B, Cc, D, lo, hi, mode, C.byref(t))
    return x, bool(t.value)


def set_threads(n: int) -> int:
    """Threads of the OpenMP build (bench.py's CPU-parallel baseline); returns the count."""
    return lib(omp=True).orc_set_threads(int(n))


def quartic_batch(A, B, Cc, D, lo=None, hi=None, mode=BOX_PROJECT, omp=False):
    A, B, Cc, D = map(_f64, (A, B, Cc, D))
    N = A.size
    x = np.empty(N)
    ties = C.c_long()
    keep = (_f64(lo) if lo is not None else None, _f64(hi) if hi is not None else None)
    lo_p = _p(keep[0]) if lo is not None else None
    hi_p = _p(keep[1]) if hi is not None else None
    lib(omp).orc_quartic_batch(_p(A), _p(B), _p(Cc), _p(D), lo_p, hi_p, _p(x), N, mode,
                               C.byref(ties))
    return x, ties.value


def build_quartic(a2, a1, b2, b1, b0, theta, phi, q, rho, delta, x1=0.0, nu=0.0):
    out = (C.c_double * 4)()
    rr = (C.c_double * 4)(*rho)
    lib().orc_build_quartic(a2, a1, b2, b1, b0, theta, phi, float(q), rr, int(delta), x1, nu,
                            out)
    return tuple(out)


# ------------------------------------------------------------------------ ADMM
def default_params(r_bar=1e-6, sigma_bar=1e-2, box_mode=BOX_PROJECT, **kw):
    p = dict(rho0=PAPER_RHO0, tau=PAPER_TAU, hi_ratio=1.2, lo_ratio=0.8, r_bar=r_bar,
             sigma_bar=sigma_bar, check_every=10, adapt_rho=1, rescale_duals=1,
             box_mode=box_mode)
    p.update(kw)
    return p


class Oracle:
    """Literal ADMM state + runner over one (possibly sharded) problem.

    prob: dict from synth (m, n, q, a2.., lo, hi, y, c).  q_total defaults to
    prob['q'].  reduce: optional python callable reduce(np_array, op) that
    all-reduces in place (op 0 = sum, 1 = max) -- used by the gloo tests.
    omp: run on the OpenMP build (bitwise-identical results, CPU-parallel baseline).
    horizon=(n_total, k_off): this process holds steps [k_off, k_off + n) of an
    n_total-step horizon (horizon-block sharding; row sums over k go through reduce)."""

    def __init__(self, prob, params=None, q_total=None, reduce=None, omp=False, horizon=None):
        self._lib = lib(omp)
        self.prob = {k: (_f64(v) if isinstance(v, np.ndarray) else v) for k, v in prob.items()}
        P = self.prob
        m, n, q = int(P["m"]), int(P["n"]), int(P["q"])
        self.m, self.n, self.q = m, n, q
        self.q_total = int(q_total if q_total is not None else q)
        self.params = default_params() if params is None else dict(params)
        n_total, k_off = horizon if horizon is not None else (0, 0)
        self._P = _Problem(m, n, q, self.q_total,
                           *[_p(P[k]) for k in ("a2", "a1", "a0", "b2", "b1", "b0", "lo",
                                                "hi", "y", "c")], int(n_total), int(k_off))
        self.x = np.zeros((m, q, n)); self.z = np.zeros((m, q, n)); self.lam = np.zeros((m, q, n))
        self.s = np.zeros((q, n)); self.mu = np.zeros((q, n))
        self.h = np.zeros((m, q)); self.p = np.zeros((m, q)); self.nu = np.zeros((m, q))
        self.x1 = np.zeros(m)
        self._S = _State(*[_p(getattr(self, k)) for k in
                           ("x", "z", "lam", "s", "mu", "h", "p", "nu", "x1")])
        self._prm = self._mk_params()
        self._reduce_py = reduce
        if reduce is not None:
            def _cb(buf, ln, op, user):
                arr = np.ctypeslib.as_array(buf, shape=(ln,))
                reduce(arr, op)
            self._cb = REDUCE_FN(_cb)
        else:
            self._cb = REDUCE_FN()
        msg = C.create_string_buffer(256)
        if self._lib.orc_validate(C.byref(self._P), msg, 256) != 0:
            raise ValueError(msg.value.decode())
        self._lib.orc_init(C.byref(self._P), C.byref(self._S), C.byref(self._prm), self._cb, None)

    def _mk_params(self):
        p = self.params
        return _Params((C.c_double * 4)(*p["rho0"]), p["tau"], p["hi_ratio"], p["lo_ratio"],
                       p["r_bar"], p["sigma_bar"], p["check_every"], p["adapt_rho"],
                       p["rescale_duals"], p["box_mode"])

    @property
    def rho(self):
        return np.array(self._S.rho[:])

    @property
    def iter(self):
        return self._S.iter

    def run(self, iters, stop_on_converge=False, hist_cap=None):
        if hist_cap is None:
            hist_cap = iters // max(1, self.params["check_every"]) + 1
        hist = np.zeros((max(1, hist_cap), HIST_COLS))
        info = _Info()
        self._lib.orc_run(C.byref(self._P), C.byref(self._S), C.byref(self._prm), int(iters),
                      int(bool(stop_on_converge)), C.byref(info), _p(hist), hist_cap, self._cb,
                      None)
        rows = min(info.hist_rows, hist_cap)
        return dict(iterations=info.iterations, r=info.r, sigma=info.sigma,
                    objective=info.objective, rho=list(info.rho), status=info.status,
                    ties=info.ties), hist[:rows].copy()

    def solve(self, max_iter=200000):
        return self.run(max_iter, stop_on_converge=True)

    def objective(self, x=None):
        x = self.x if x is None else _f64(x)
        return self._lib.orc_objective(C.byref(self._P), _p(x), self._cb, None)

    def state(self):
        return {k: getattr(self, k).copy() for k in
                ("x", "z", "lam", "s", "mu", "h", "p", "nu", "x1")} | {"rho": self.rho}
