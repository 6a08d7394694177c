"""Additive Schwarz / block-Jacobi preconditioners on the GPU.

Mirrors /root/reference/pkg/src/iedd/precond.py:81-215 (Preconditioner,
identity, from_decomposition with backend="exact").  The D subdomain blocks
are extracted and factorised on the device in one batched launch (K2) and
applied as gather -> per-block solve -> deterministic ascending-id sum (K3);
see csrc/precond.cu.

Recursive skeletonisation (backend="rskel", rs_global) is out of scope for
the B200 hot path and raises ValueError.
"""

from __future__ import annotations

import ctypes
import time

import numpy as np

from . import _lib
from .geometry import Decomposition, Partitioning
from .kernel import KernelOperator
from .linalg import NotPositiveDefinite
from .toeplitz import to_device_vector, to_host

NONE = "none"
RS_GLOBAL = "rs-global"
EXACT = "exact"
RSKEL = "rskel"
DENSE_LIMIT_DEFAULT = 4096


class Preconditioner:
    """Applies T^{-1}; build through from_decomposition / identity."""

    def __init__(self, kind: str, n: int, handle, backend: str, t_factor: float, stats=None):
        self.kind = kind
        self.n = n
        self.backend = backend
        self.t_factor = t_factor
        self._handle = handle
        self._stats = stats or {"S": 0, "memory_bytes": 0, "device_bytes": 0, "factored": 0, "D": 0}
        self._lib = _lib.lib() if handle is not None else None

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and h.value:
            self._lib.ie_precond_destroy(h)
            self._handle = None

    @property
    def handle(self):
        return self._handle

    def apply_device(self, r, z):
        """z = T^{-1} r for torch CUDA float64 tensors (no host sync)."""
        if self._handle is None:
            z.copy_(r)
            return z
        rc = self._lib.ie_precond_apply_f64(self._handle, _lib.ptr(r), _lib.ptr(z), _lib.stream_ptr())
        _lib.check(rc, "Preconditioner.apply")
        return z

    def apply(self, f):
        if self._handle is None:
            a = np.asarray(f, dtype=float) if not _is_tensor(f) else f
            if tuple(a.shape) != (self.n,):
                raise ValueError(f"expected vector of length {self.n}, got {tuple(a.shape)}")
            return a.copy() if isinstance(a, np.ndarray) else a.clone()
        r, was_np = to_device_vector(f, self.n)
        z = r.new_empty(r.shape)
        self.apply_device(r, z)
        return to_host(z, was_np)

    def apply_dense(self) -> np.ndarray:
        """Materialise T^{-1} (precond.py:102-116): apply to the unit columns."""
        return self.apply_dense_device().cpu().numpy()

    def apply_dense_device(self):
        """T^{-1} as a symmetrised dense device tensor."""
        torch = _lib.torch_cuda()
        if self._handle is None:
            return torch.eye(self.n, dtype=torch.float64, device="cuda")
        eye = torch.eye(self.n, dtype=torch.float64, device="cuda")
        out = torch.empty_like(eye)
        for j in range(self.n):
            self.apply_device(eye[j], out[j])
        return 0.5 * (out + out.T)

    def block(self, k: int):
        """Subdomain k's stored factor, read back from the device: ("cholesky",
        G) with A_k = G^T G (the reference's CholeskyFactor.g, linalg.py:36-45;
        variant "subst", blocks of <= 160 points) or ("inverse", A_k^{-1})
        otherwise -- s x s numpy arrays in the block's point order."""
        if self._handle is None:
            raise ValueError("the identity preconditioner has no blocks")
        import ctypes
        s, kind = ctypes.c_int64(0), ctypes.c_int32(0)
        _lib.check(self._lib.ie_precond_block_f64(self._handle, int(k), None, ctypes.byref(s), ctypes.byref(kind)),
                   "Preconditioner.block")
        out = np.empty((s.value, s.value), dtype=np.float64)
        _lib.check(self._lib.ie_precond_block_f64(self._handle, int(k), _lib.np_ptr(out), ctypes.byref(s),
                                                  ctypes.byref(kind)), "Preconditioner.block")
        return ("cholesky" if kind.value == 1 else "inverse"), out

    @property
    def n_subdomains(self) -> int:
        return max(self._stats["D"], 1)

    def stats(self) -> dict:
        return {"S": self._stats["S"], "memory_bytes": self._stats["memory_bytes"],
                "t_factor": self.t_factor, "device_bytes": self._stats["device_bytes"],
                "factored_blocks": self._stats["factored"]}


def _is_tensor(x) -> bool:
    try:
        import torch
        return isinstance(x, torch.Tensor)
    except ImportError:  # pragma: no cover
        return False


def identity(n: int) -> Preconditioner:
    return Preconditioner(kind=NONE, n=n, handle=None, backend=EXACT, t_factor=0.0)


def from_decomposition(op: KernelOperator, decomposition: Decomposition, backend: str = EXACT,
                       eps: float = 1e-3, proxy=None, dense_limit: int = DENSE_LIMIT_DEFAULT,
                       share_mirrored_subdomains: bool = False, *, variant: str = "packed_inverse",
                       share_translated: bool = True) -> Preconditioner:
    """Factorise every block A_k = A(I_k, I_k) on the device.

    variant: "packed_inverse" (apply = packed symmetric A_k^{-1} matvec) or
    "subst" (forward/back substitution with the Cholesky factor).
    share_translated: factorise one block per translation class (exact: such
    blocks are bitwise identical here); share_mirrored_subdomains: classes
    under translations and grid reflections (each block in a canonical point
    order), which covers the reference's mirrored CBD subdomains
    (precond.py:137-154) and reports its memory accounting.
    """
    if backend not in (EXACT, RSKEL):
        raise ValueError(f"backend must be 'exact' or 'rskel', got {backend!r}")
    if backend == RSKEL:
        raise ValueError("backend='rskel' (recursive skeletonisation) is outside the B200 hot path; "
                         "use backend='exact'")
    if variant not in _lib.VARIANTS:
        raise ValueError(f"variant must be one of {tuple(_lib.VARIANTS)}, got {variant!r}")
    subs = decomposition.subdomains
    for i, idx in enumerate(subs):
        if idx.size > dense_limit:
            raise ValueError(f"subdomain {i} has {idx.size} points > dense_limit={dense_limit}; "
                             "use backend='rskel'")
    t0 = time.perf_counter()
    sizes = np.array([s.size for s in subs], dtype=np.int64)
    offsets = np.zeros(len(subs) + 1, dtype=np.int64)
    np.cumsum(sizes, out=offsets[1:])
    indices = np.ascontiguousarray(np.concatenate([np.asarray(s, dtype=np.int64) for s in subs]))
    # bit 0: translation classes; bit 1: translations + grid reflections (the
    # reference's mirrored sharing, precond.py:137-154, generalised)
    share_mask = (1 if share_translated else 0) | (2 if share_mirrored_subdomains else 0)
    L = _lib.lib()
    h = ctypes.c_void_p()
    bad = ctypes.c_int64(-1)
    rc = L.ie_precond_create(op.geom(), _lib.np_ptr(offsets), _lib.np_ptr(indices), len(subs),
                             _lib.VARIANTS[variant], share_mask, ctypes.byref(h),
                             ctypes.byref(bad), _lib.stream_ptr())
    if rc == _lib.IE_ERR_NOT_SPD:
        i = bad.value
        raise NotPositiveDefinite(f"subdomain {i}: matrix is not positive definite (subdomain {i})")
    _lib.check(rc, "from_decomposition")
    st = np.zeros(5, dtype=np.int64)
    _lib.check(L.ie_precond_stats(h, _lib.np_ptr(st)), "stats")
    memory_bytes = int(st[1])
    if share_mirrored_subdomains and decomposition.kind == "cbd" and decomposition.m_per_dim % 2 == 0:
        # the reference's accounting (precond.py:38-39, 60-61): one factor, 8 s bytes per mirrored solver
        memory_bytes = 8 * (int(sizes[0]) ** 2 + int(sizes[0])) + 8 * int(sizes[1:].sum())
    stats = {"S": int(st[0]), "memory_bytes": memory_bytes, "device_bytes": int(st[2]),
             "factored": int(st[3]), "D": int(st[4])}
    return Preconditioner(kind=decomposition.kind, n=op.n, handle=h, backend=EXACT,
                          t_factor=time.perf_counter() - t0, stats=stats)


def rs_global(op: KernelOperator, partitioning: Partitioning, eps: float = 1e-3, proxy=None):
    raise ValueError("rs_global (recursive skeletonisation) is outside the B200 hot path")
