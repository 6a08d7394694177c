"""Extremal eigenvalue of T^{-1}A by Lanczos in the A-inner product
(mirrors /root/reference/pkg/src/iedd/spectrum.py:133-190).

With a native operator and a native or identity preconditioner the loop
runs in libiedd_b200.so (ie_lanczos_f64): basis and A-basis stay on the
device, the two-pass A-orthogonalisation is done as two classical
Gram-Schmidt sweeps (GEMV pairs), and the Ritz value comes from a device
Sturm-multisection on the tridiagonal.  Any other operator the reference
accepts (a callable or an object with .matvec, spectrum.py:147; any object
with .apply, :161) runs the reference's loop on device vectors with host
callbacks (_lanczos_generic).  The stopping rule is the reference's (5
consecutive steps with |change| <= rtol*max(|lambda|,1), beta^2 <= 0,
beta < 1e-14, max_iters).

The dense-spectrum analysis (spectrum.py:37-130: preconditioned_spectrum,
extremal_eigenvector, jacobi_pairing_check) materialises A and T^{-1} on the
device (K1's entry formula, K3 applied to the unit columns) and solves the
symmetric congruence G^T A G, T^{-1} = G G^T, with the device's dense
Cholesky / symmetric eigensolver (torch.linalg, cuSOLVER): a utility around
the path, not a hot kernel."""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .precond import Preconditioner
from .toeplitz import KernelMatvec

DENSE_LIMIT_SPECTRUM = 4096
MULTIPLICITY_TOL = 1e-8


def extremal_eigenvalue_lanczos(matvec, precond, n: int, which: str = "min", max_iters: int = 400,
                                rtol: float = 1e-9, seed: int = 0, return_steps: bool = False):
    if which not in ("min", "max"):
        raise ValueError(f"which must be 'min' or 'max', got {which!r}")
    if not hasattr(precond, "apply"):  # spectrum.py:161 calls precond.apply
        raise TypeError(f"precond of type {type(precond).__name__} has no .apply")
    native = (isinstance(matvec, KernelMatvec) and isinstance(precond, Preconditioner)
              and matvec.N == n == precond.n)
    if not native:
        return _lanczos_generic(matvec, precond, n, which, max_iters, rtol, seed, return_steps)
    torch = _lib.torch_cuda()
    v0 = torch.from_numpy(np.random.default_rng(seed).standard_normal(n)).cuda()
    lam = ctypes.c_double(0.0)
    steps = ctypes.c_int64(0)
    rc = _lib.lib().ie_lanczos_f64(matvec.handle, precond.handle, _lib.ptr(v0), 0 if which == "min" else 1,  # NULL: identity
                                   max_iters, rtol, ctypes.byref(lam), ctypes.byref(steps), _lib.stream_ptr())
    if rc == _lib.IE_ERR_NO_RITZ:
        raise RuntimeError("Lanczos produced no Ritz values")
    _lib.check(rc, "extremal_eigenvalue_lanczos")
    return (lam.value, steps.value) if return_steps else lam.value


def _lanczos_generic(matvec, precond, n, which, max_iters, rtol, seed, return_steps):
    """spectrum.py:133-190 for operators without a native handle: the
    reference's loop (two-pass modified Gram-Schmidt in the A-inner product,
    Ritz values of the tridiagonal by scipy) on device vectors; the user's
    callables see numpy arrays, as in the reference."""
    from scipy.linalg import eigvalsh_tridiagonal

    from .pcg import _device_op
    torch = _lib.torch_cuda()
    A = _device_op(matvec, n)
    T = _device_op(precond, n)
    v = torch.from_numpy(np.random.default_rng(seed).standard_normal(n)).cuda()
    av = A(v)
    nrm = float(torch.dot(v, av)) ** 0.5
    V, AV = [v / nrm], [av / nrm]
    alphas, betas = [], []
    estimate, stable, steps = None, 0, 1
    for j in range(max_iters):
        w = T(AV[j])
        alphas.append(float(torch.dot(w, AV[j])))
        for _ in range(2):
            for vi, avi in zip(V, AV):
                w -= float(torch.dot(w, avi)) * vi
        aw = A(w)
        steps += 1
        beta2 = float(torch.dot(w, aw))
        if beta2 <= 0 or not np.isfinite(beta2):
            break
        beta = beta2 ** 0.5
        ritz = eigvalsh_tridiagonal(np.array(alphas), np.array(betas))
        current = float(ritz[0] if which == "min" else ritz[-1])
        if estimate is not None and abs(current - estimate) <= rtol * max(abs(current), 1.0):
            stable += 1
            if stable >= 5:
                estimate = current
                break
        else:
            stable = 0
        estimate = current
        if beta < 1e-14:
            break
        betas.append(beta)
        V.append(w / beta)
        AV.append(aw / beta)
    if estimate is None:
        raise RuntimeError("Lanczos produced no Ritz values")
    return (estimate, steps) if return_steps else estimate


# --------------------------------------------------------------------------
# dense spectra (spectrum.py:29-130)
# --------------------------------------------------------------------------
from dataclasses import dataclass, field  # noqa: E402


@dataclass(frozen=True)
class SpectrumReport:
    lambda_min: float
    lambda_max: float
    eigenvalues: np.ndarray = field(repr=False)
    multiplicity_at_max: int
    config: dict


def _congruence(op, precond):
    """(G, G^T A G) on the device, T^{-1} = G G^T (spectrum.py:37-45)."""
    torch = _lib.torch_cuda()
    tinv = precond.apply_dense_device()
    g, info = torch.linalg.cholesky_ex(tinv)
    if int(info.item()) != 0:
        raise RuntimeError("materialized preconditioner is not numerically SPD")
    idx = np.arange(op.n, dtype=np.int64)
    a = op.assemble_block_device(idx, idx)
    return g, g.T @ (a @ g)


def preconditioned_spectrum(op, precond, dense_limit: int = DENSE_LIMIT_SPECTRUM, config: dict | None = None):
    """All eigenvalues of T^{-1}A (spectrum.py:48-73)."""
    if op.n > dense_limit:
        raise ValueError(f"N={op.n} exceeds dense_limit={dense_limit}; raise the limit "
                         "explicitly for larger dense spectra")
    torch = _lib.torch_cuda()
    _, sym = _congruence(op, precond)
    w = torch.linalg.eigvalsh(sym).cpu().numpy()
    lam_max = float(w[-1])
    return SpectrumReport(lambda_min=float(w[0]), lambda_max=lam_max, eigenvalues=w,
                          multiplicity_at_max=int(np.sum(np.abs(w - lam_max) <= MULTIPLICITY_TOL)),
                          config=dict(config or {}, N=op.n, kind=precond.kind, D=precond.n_subdomains))


def multiplicity_at(report: SpectrumReport, value: float, tol: float) -> int:
    return int(np.sum(np.abs(report.eigenvalues - value) <= tol))


def extremal_eigenvector(op, precond, which: str, dense_limit: int = DENSE_LIMIT_SPECTRUM):
    """Extremal eigenpair of T^{-1}A (spectrum.py:80-102): unit-norm vector,
    largest-magnitude entry positive."""
    if which not in ("min", "max"):
        raise ValueError(f"which must be 'min' or 'max', got {which!r}")
    if op.n > dense_limit:
        raise ValueError(f"N={op.n} exceeds dense_limit={dense_limit}")
    torch = _lib.torch_cuda()
    g, sym = _congruence(op, precond)
    w, vecs = torch.linalg.eigh(sym)
    col = 0 if which == "min" else -1
    vec = (g @ vecs[:, col]).cpu().numpy()
    vec /= np.linalg.norm(vec)
    if vec[np.argmax(np.abs(vec))] < 0:
        vec = -vec
    return float(w[col].item()), vec


def jacobi_pairing_check(op, decomposition) -> float:
    """max_k |lambda_k + lambda_{N+1-k} - 2| for a two-subdomain Jacobi split
    (spectrum.py:105-114)."""
    from .precond import from_decomposition
    if decomposition.kind != "jacobi" or decomposition.n_subdomains != 2:
        raise ValueError("pairing check needs a two-subdomain Jacobi decomposition")
    pre = from_decomposition(op, decomposition, dense_limit=op.n)
    w = preconditioned_spectrum(op, pre, dense_limit=op.n).eigenvalues
    return float(np.max(np.abs(w + w[::-1] - 2.0)))
