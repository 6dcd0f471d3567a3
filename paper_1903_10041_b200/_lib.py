"""ctypes binding of libadmm_b200.so (include/admm.h).  Argument marshalling
only: every step of the ADMM path runs in the library's CUDA kernels.  There
is no CPU fallback: if the library is missing this module raises ImportError.

Arrays may be numpy arrays (host) or torch tensors (host or CUDA); they must
be float64 and C-contiguous in the layouts of include/admm.h.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.environ.get("ADMM_SO") or os.path.join(_HERE, "libadmm_b200.so")  # ADMM_SO: dev builds

if not os.path.exists(SO_PATH):
    raise ImportError(
        f"{SO_PATH} not found: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(nvcc, sm_100a). There is no CPU fallback.")

_lib = C.CDLL(SO_PATH)

ADMM_OK, ADMM_ERR_INVALID, ADMM_NOT_CONVERGED, ADMM_ERR_NONCONVEX = 0, 1, 2, 3
ADMM_ERR_NUMERICAL, ADMM_ERR_CUDA, ADMM_ERR_NCCL, ADMM_ERR_STATE = 4, 5, 6, 7
ADMM_BOX_PROJECT, ADMM_BOX_EXACT = 0, 1
ADMM_EXEC_AUTO, ADMM_EXEC_STREAMING, ADMM_EXEC_PERSISTENT = 0, 1, 2
ADMM_HIST_COLS = 16
STATUS_NAMES = {0: "ADMM_OK", 1: "ADMM_ERR_INVALID", 2: "ADMM_NOT_CONVERGED",
                3: "ADMM_ERR_NONCONVEX", 4: "ADMM_ERR_NUMERICAL", 5: "ADMM_ERR_CUDA",
                6: "ADMM_ERR_NCCL", 7: "ADMM_ERR_STATE"}


ADMM_SHARD_SCENARIOS, ADMM_SHARD_HORIZON = 0, 1


class admm_dist(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32), ("j_begin", C.c_int64),
                ("j_end", C.c_int64), ("nccl_id", C.c_ubyte * 128), ("k_begin", C.c_int64),
                ("k_end", C.c_int64), ("mode", C.c_int32), ("reserved", C.c_int32)]


class admm_params(C.Structure):
    _fields_ = [("rho", C.c_double * 4), ("tau", C.c_double), ("hi_ratio", C.c_double),
                ("lo_ratio", C.c_double), ("r_bar", C.c_double), ("sigma_bar", C.c_double),
                ("check_every", C.c_int32), ("adapt_rho", C.c_int32),
                ("rescale_duals", C.c_int32), ("box_mode", C.c_int32), ("exec_mode", C.c_int32)]


class admm_info(C.Structure):
    _fields_ = [("iterations", C.c_int64), ("r", C.c_double), ("sigma", C.c_double),
                ("objective", C.c_double), ("rho", C.c_double * 4), ("status", C.c_int32),
                ("checks", C.c_int32)]

    def as_dict(self):
        return dict(iterations=self.iterations, r=self.r, sigma=self.sigma,
                    objective=self.objective, rho=list(self.rho), status=self.status,
                    checks=self.checks)


_vp = C.c_void_p
_ctx_p = C.c_void_p
_sigs = {
    "admm_default_params": (None, [C.POINTER(admm_params)]),
    "admm_workspace_bytes": (C.c_size_t, [C.c_int32, C.c_int64, C.c_int64, C.c_int32]),
    "admm_nccl_unique_id": (C.c_int, [C.c_ubyte * 128]),
    "admm_create": (C.c_int, [C.POINTER(_ctx_p), C.c_int32, C.c_int64, C.c_int64,
                              C.POINTER(admm_dist), C.c_int32, _vp, C.c_size_t, _vp]),
    "admm_set_problem": (C.c_int, [_ctx_p, _vp, _vp, _vp, _vp, _vp, _vp, C.c_int32]),
    "admm_reset": (C.c_int, [_ctx_p]),
    "admm_set_params": (C.c_int, [_ctx_p, C.POINTER(admm_params)]),
    "admm_get_params": (C.c_int, [_ctx_p, C.POINTER(admm_params)]),
    "admm_iterate": (C.c_int, [_ctx_p, C.c_int64]),
    "admm_solve": (C.c_int, [_ctx_p, C.c_double, C.c_double, C.c_int64, C.POINTER(admm_info)]),
    "admm_get_solution": (C.c_int, [_ctx_p, _vp, _vp, C.POINTER(admm_info), C.c_int32]),
    "admm_get_state": (C.c_int, [_ctx_p] + [_vp] * 9 + [C.c_int32]),
    "admm_set_state": (C.c_int, [_ctx_p] + [_vp] * 9 + [C.c_int32]),
    "admm_get_history": (C.c_int64, [_ctx_p, _vp, C.c_int64]),
    "admm_get_timing": (C.c_int, [_ctx_p, C.c_double * 2]),
    "admm_get_engine": (C.c_int, [_ctx_p, C.POINTER(C.c_int32), C.POINTER(C.c_int64)]),
    "admm_set_coeff_precision": (C.c_int, [_ctx_p, C.c_int32]),
    "admm_get_coeff_precision": (C.c_int, [_ctx_p, C.POINTER(C.c_int32)]),
    "admm_last_error": (C.c_char_p, [_ctx_p]),
    "admm_destroy": (None, [_ctx_p]),
    "quartic_minimize_batch": (C.c_int, [_vp] * 7 + [C.c_int64, C.c_int32, _vp]),
    "admm_build_info": (C.c_char_p, []),
}
for _name, (_res, _args) in _sigs.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args

EXPORTED = tuple(_sigs)


class AdmmError(RuntimeError):
    def __init__(self, status, msg=""):
        self.status = status
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")


def _ptr(a):
    """(pointer, on_device, keepalive) of a numpy array / torch tensor / None."""
    if a is None:
        return None, 0, None
    try:
        import torch

        if isinstance(a, torch.Tensor):
            if a.dtype != torch.float64 or not a.is_contiguous():
                raise TypeError("tensors must be float64 and contiguous")
            return a.data_ptr(), int(a.is_cuda), a
    except ImportError:  # pragma: no cover
        pass
    arr = np.asarray(a)
    if arr.dtype != np.float64 or not arr.flags["C_CONTIGUOUS"]:
        arr = np.ascontiguousarray(arr, dtype=np.float64)
    return arr.ctypes.data, 0, arr


def _check(ctx, st, allow=(ADMM_OK,)):
    if st not in allow:
        msg = _lib.admm_last_error(ctx).decode() if ctx else ""
        raise AdmmError(st, msg)
    return st


# ------------------------------------------------------------------ the ABI
def admm_default_params() -> admm_params:
    p = admm_params()
    _lib.admm_default_params(C.byref(p))
    return p


def admm_workspace_bytes(m, n, q_local, device=0) -> int:
    return int(_lib.admm_workspace_bytes(m, n, q_local, device))


def admm_nccl_unique_id() -> bytes:
    buf = (C.c_ubyte * 128)()
    _check(None, _lib.admm_nccl_unique_id(buf))
    return bytes(buf)


def admm_create(m, n, q_total, dist=None, device=0, workspace=None, stream=None):
    ctx = _ctx_p()
    dptr = C.byref(dist) if dist is not None else None
    wptr, wbytes = (None, 0)
    if workspace is not None:
        wptr, wbytes = workspace.data_ptr(), workspace.numel() * workspace.element_size()
    sptr = None
    if stream is not None:
        sptr = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
    st = _lib.admm_create(C.byref(ctx), m, n, q_total, dptr, device, wptr, wbytes, sptr)
    if st != ADMM_OK:
        msg = _lib.admm_last_error(ctx).decode() if ctx.value else ""
        if ctx.value:
            _lib.admm_destroy(ctx)
        raise AdmmError(st, msg)
    return ctx


def admm_set_problem(ctx, f, g, lo, hi, y, c):
    ps = [_ptr(a) for a in (f, g, lo, hi, y, c)]
    on_dev = int(any(p[1] for p in ps))
    return _check(ctx, _lib.admm_set_problem(ctx, *[p[0] for p in ps], on_dev))


def admm_reset(ctx):
    return _check(ctx, _lib.admm_reset(ctx))


def admm_set_params(ctx, params: admm_params):
    return _check(ctx, _lib.admm_set_params(ctx, C.byref(params)))


def admm_get_params(ctx) -> admm_params:
    p = admm_params()
    _check(ctx, _lib.admm_get_params(ctx, C.byref(p)))
    return p


def admm_iterate(ctx, iters):
    return _check(ctx, _lib.admm_iterate(ctx, int(iters)))


def admm_solve(ctx, r_bar, sigma_bar, max_iter):
    info = admm_info()
    st = _lib.admm_solve(ctx, float(r_bar), float(sigma_bar), int(max_iter), C.byref(info))
    _check(ctx, st, allow=(ADMM_OK, ADMM_NOT_CONVERGED))
    return st, info.as_dict()


def admm_get_solution(ctx, x=None, x1=None):
    info = admm_info()
    px, dx, kx = _ptr(x)
    p1, d1, k1 = _ptr(x1)
    _check(ctx, _lib.admm_get_solution(ctx, px, p1, C.byref(info), int(dx or d1)))
    return info.as_dict()


def admm_get_state(ctx, x=None, z=None, lam=None, s=None, mu=None, h=None, p=None, nu=None,
                   x1=None):
    ps = [_ptr(a) for a in (x, z, lam, s, mu, h, p, nu, x1)]
    devs = {q[1] for q in ps if q[0] is not None}
    if len(devs) > 1:
        raise ValueError("all state buffers must be on the same side (host or device)")
    on_dev = devs.pop() if devs else 0
    return _check(ctx, _lib.admm_get_state(ctx, *[q[0] for q in ps], on_dev))


def admm_set_state(ctx, x, z, lam, s, mu, h, p, nu, x1):
    ps = [_ptr(a) for a in (x, z, lam, s, mu, h, p, nu, x1)]
    on_dev = int(any(q[1] for q in ps))
    return _check(ctx, _lib.admm_set_state(ctx, *[q[0] for q in ps], on_dev))


def admm_get_history(ctx, max_rows=100000):
    out = np.zeros((max_rows, ADMM_HIST_COLS))
    n = _lib.admm_get_history(ctx, out.ctypes.data, max_rows)
    return out[:n].copy()


def admm_get_timing(ctx):
    t = (C.c_double * 2)()
    _check(ctx, _lib.admm_get_timing(ctx, t))
    return t[0], t[1]


ENGINE_NAMES = {0: "none", 1: "sweep_kernel", 2: "persist_kernel", 3: "persist_cluster_kernel",
                4: "sweep2_kernel", 5: "persist_cluster2_kernel"}


def admm_get_engine(ctx):
    """(engine id of the last call, kernels launched by this context so far)."""
    e, n = C.c_int32(0), C.c_int64(0)
    _check(ctx, _lib.admm_get_engine(ctx, C.byref(e), C.byref(n)))
    return int(e.value), int(n.value)


def admm_set_coeff_precision(ctx, bits: int):
    """F2: storage precision (64 or 32) of a2, a1, b2, b1 applied by the next set_problem."""
    return _check(ctx, _lib.admm_set_coeff_precision(ctx, int(bits)))


def admm_get_coeff_precision(ctx) -> int:
    b = C.c_int32(0)
    _check(ctx, _lib.admm_get_coeff_precision(ctx, C.byref(b)))
    return int(b.value)


def admm_last_error(ctx) -> str:
    return _lib.admm_last_error(ctx).decode()


def admm_destroy(ctx):
    _lib.admm_destroy(ctx)


def quartic_minimize_batch(A, B, Cc, D, lo, hi, x, box_mode=ADMM_BOX_PROJECT, stream=None):
    """All arrays CUDA float64 tensors of length N (lo/hi may be None)."""
    ps = [_ptr(a) for a in (A, B, Cc, D, lo, hi, x)]
    for q in ps:
        if q[0] is not None and not q[1]:
            raise ValueError("quartic_minimize_batch takes device tensors")
    sptr = None
    if stream is not None:
        sptr = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
    N = A.numel()
    return _check(None, _lib.quartic_minimize_batch(*[q[0] for q in ps], N, box_mode, sptr))


def admm_build_info() -> str:
    return _lib.admm_build_info().decode()
