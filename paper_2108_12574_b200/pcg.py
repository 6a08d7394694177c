"""Preconditioned conjugate gradient (mirrors
/root/reference/pkg/src/iedd/pcg.py:15-136).

With a native operator (KernelMatvec) and a native or identity
preconditioner the whole loop runs in libiedd_b200.so (ie_pcg_f64): the
vectors never leave the device, the true residual is folded into a 2-RHS
A-pass, and the host sees one status scalar per iteration.  Any other
callables (the reference's duck typing, pcg.py:26-33) run through the same
control flow with device-resident vectors and host callbacks.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .precond import Preconditioner
from .toeplitz import KernelMatvec, to_device_vector, to_host

STAGNATION_WINDOW = 30
STAGNATION_FACTOR = 1e-3


@dataclass
class PcgReport:
    n_it: int
    achieved_residual: float
    t_pcg: float
    t_s: float
    residual_history: list = field(repr=False)
    stagnated: bool = False
    converged: bool = False


def _as_callable(operator):
    if callable(operator):
        return operator
    if hasattr(operator, "matvec"):
        return operator.matvec
    if hasattr(operator, "apply"):
        return operator.apply
    raise TypeError(f"cannot apply operator of type {type(operator).__name__}")


def make_rhs(matvec, n: int, mode: str = "random", seed: int = 0):
    """Right-hand side for Au = f (pcg.py:36-51)."""
    if mode == "random":
        u_exact = np.random.default_rng(seed).standard_normal(n)
        return _as_callable(matvec)(u_exact), u_exact
    if mode == "noise":
        return np.random.default_rng(seed).standard_normal(n), None
    if mode == "ones":
        return np.ones(n), None
    raise ValueError(f"rhs mode must be 'random', 'noise' or 'ones', got {mode!r}")


def _native(matvec, precond) -> bool:
    if not isinstance(matvec, KernelMatvec):
        return False
    return precond is None or (isinstance(precond, Preconditioner) and precond.n == matvec.N)


def solve(matvec, precond, f, tol: float = 1e-12, max_iters: int | None = None):
    """Run PCG on Au = f from u0 = 0 (pcg.py:54-136)."""
    if not 0.0 < tol < 1.0:
        raise ValueError(f"tol must be in (0, 1), got {tol}")
    if _native(matvec, precond):
        return _solve_native(matvec, precond, f, tol, max_iters)
    return _solve_generic(matvec, precond, f, tol, max_iters)


def _solve_native(A: KernelMatvec, T, f, tol, max_iters):
    torch = _lib.torch_cuda()
    fd, was_np = to_device_vector(f, A.N)
    n = A.N
    if max_iters is None:
        max_iters = max(2 * n, 100)
    # numpy in -> numpy out: u goes straight to page-locked host memory, its copy
    # overlapping the closing residual pass (ie_pcg_host_f64)
    u = torch.empty(n, dtype=torch.float64, pin_memory=True) if was_np else torch.empty_like(fd)
    hist = np.zeros(max_iters + 1, dtype=np.float64)
    n_it = ctypes.c_int64(0)
    flags = np.zeros(2, dtype=np.int32)
    times = np.zeros(2, dtype=np.float64)
    fail_it = ctypes.c_int64(0)
    fail_val = ctypes.c_double(0.0)
    th = T.handle if (T is not None and T.handle is not None) else None
    entry = _lib.lib().ie_pcg_host_f64 if was_np else _lib.lib().ie_pcg_f64
    rc = entry(A.handle, th, _lib.ptr(fd), _lib.ptr(u), tol, max_iters,
                               _lib.np_ptr(hist), ctypes.byref(n_it), _lib.np_ptr(flags), _lib.np_ptr(times),
                               ctypes.byref(fail_it), ctypes.byref(fail_val), _lib.stream_ptr())
    if rc == _lib.IE_ERR_BREAKDOWN:
        raise FloatingPointError(f"PCG breakdown at iteration {fail_it.value}: p^T A p = {fail_val.value}")
    if rc == _lib.IE_ERR_NONFINITE:
        raise FloatingPointError(f"non-finite residual at iteration {fail_it.value}")
    _lib.check(rc, "pcg.solve")
    k = n_it.value
    history = [float(x) for x in hist[: k + 1]]
    rep = PcgReport(n_it=k, achieved_residual=history[-1], t_pcg=float(times[0]), t_s=float(times[1]),
                    residual_history=history, stagnated=bool(flags[1]), converged=bool(flags[0]))
    return (u.numpy() if was_np else u), rep


def _device_op(op, n, identity_ok=False):
    """Wrap a native or host callable as device tensor -> device tensor."""
    torch = _lib.torch_cuda()
    if op is None and identity_ok:
        return lambda x: x.clone()
    if isinstance(op, KernelMatvec):
        def a(x):
            y = torch.empty_like(x)
            op.matvec_device(x, y)
            return y
        return a
    if isinstance(op, Preconditioner) and op.handle is None:  # identity(n) (precond.py:133-134)
        return lambda x: x.clone()
    if isinstance(op, Preconditioner):
        def t(x):
            z = torch.empty_like(x)
            op.apply_device(x, z)
            return z
        return t
    fn = _as_callable(op)

    def host(x):
        y = np.asarray(fn(x.cpu().numpy()), dtype=float)
        return torch.from_numpy(np.ascontiguousarray(y)).cuda()
    return host


def _solve_generic(matvec, precond, f, tol, max_iters):
    torch = _lib.torch_cuda()
    fa = f if isinstance(f, torch.Tensor) else np.asarray(f, dtype=float)
    n = int(fa.shape[0])
    fd, was_np = to_device_vector(fa, n)
    A = _device_op(matvec, n)
    T = _device_op(precond, n, identity_ok=True)
    if max_iters is None:
        max_iters = max(2 * n, 100)
    norm_f = float(torch.linalg.vector_norm(fd))
    u = torch.zeros_like(fd)
    if norm_f == 0.0:
        return to_host(u, was_np), PcgReport(0, 0.0, 0.0, 0.0, [0.0], converged=True)
    t0 = time.perf_counter()
    t_prec, n_prec = 0.0, 0
    r = fd.clone()
    tp = time.perf_counter()
    z = T(r)
    torch.cuda.synchronize()
    t_prec += time.perf_counter() - tp
    n_prec += 1
    p = z.clone()
    rho = float(torch.dot(r, z))
    history = [1.0]
    stagnated = converged = False
    k = 0
    while k < max_iters:
        k += 1
        q = A(p)
        denom = float(torch.dot(p, q))
        if not np.isfinite(denom) or denom <= 0.0:
            raise FloatingPointError(f"PCG breakdown at iteration {k}: p^T A p = {denom}")
        alpha = rho / denom
        u += alpha * p
        r -= alpha * q
        rel = float(torch.linalg.vector_norm(fd - A(u))) / norm_f
        if not np.isfinite(rel):
            raise FloatingPointError(f"non-finite residual at iteration {k}")
        history.append(rel)
        if rel <= tol:
            converged = True
            break
        if k >= STAGNATION_WINDOW and rel > (1.0 - STAGNATION_FACTOR) * history[k - STAGNATION_WINDOW]:
            stagnated = True
            break
        tp = time.perf_counter()
        z = T(r)
        torch.cuda.synchronize()
        t_prec += time.perf_counter() - tp
        n_prec += 1
        rho_next = float(torch.dot(r, z))
        p = z + (rho_next / rho) * p
        rho = rho_next
    rep = PcgReport(n_it=k, achieved_residual=history[-1], t_pcg=time.perf_counter() - t0,
                    t_s=t_prec / max(n_prec, 1), residual_history=history, stagnated=stagnated,
                    converged=converged)
    return to_host(u, was_np), rep
