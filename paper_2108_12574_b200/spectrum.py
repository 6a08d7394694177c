"""Extremal eigenvalue of T^{-1}A by Lanczos in the A-inner product
(mirrors /root/reference/pkg/src/iedd/spectrum.py:133-190).

With native operator and preconditioner the loop runs in libiedd_b200.so
(ie_lanczos_f64): basis and A-basis stay on the device, the two-pass
A-orthogonalisation is done as two classical Gram-Schmidt sweeps (GEMV
pairs), and the Ritz value comes from a device Sturm-multisection on the
tridiagonal.  The stopping rule is the reference's (5 consecutive steps with
|change| <= rtol*max(|lambda|,1), beta^2 <= 0, beta < 1e-14, max_iters).

The dense-spectrum analysis (spectrum.py:37-130) is out of scope."""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .precond import Preconditioner
from .toeplitz import KernelMatvec

DENSE_LIMIT_SPECTRUM = 4096


def extremal_eigenvalue_lanczos(matvec, precond, n: int, which: str = "min", max_iters: int = 400,
                                rtol: float = 1e-9, seed: int = 0, return_steps: bool = False):
    if which not in ("min", "max"):
        raise ValueError(f"which must be 'min' or 'max', got {which!r}")
    if not (isinstance(matvec, KernelMatvec) and isinstance(precond, Preconditioner)
            and precond.handle is not None and matvec.N == n == precond.n):
        raise TypeError("extremal_eigenvalue_lanczos needs a KernelMatvec and a device Preconditioner "
                        "built by from_decomposition for the same N")
    torch = _lib.torch_cuda()
    v0 = torch.from_numpy(np.random.default_rng(seed).standard_normal(n)).cuda()
    lam = ctypes.c_double(0.0)
    steps = ctypes.c_int64(0)
    rc = _lib.lib().ie_lanczos_f64(matvec.handle, precond.handle, _lib.ptr(v0), 0 if which == "min" else 1,
                                   max_iters, rtol, ctypes.byref(lam), ctypes.byref(steps), _lib.stream_ptr())
    if rc == _lib.IE_ERR_NO_RITZ:
        raise RuntimeError("Lanczos produced no Ritz values")
    _lib.check(rc, "extremal_eigenvalue_lanczos")
    return (lam.value, steps.value) if return_steps else lam.value
