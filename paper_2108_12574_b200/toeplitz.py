"""Matrix-free operator application y = A x on the GPU.

Drop-in for the reference's ToeplitzMatvec (/root/reference/pkg/src/iedd/
toeplitz.py:11-57): same constructor argument, ``shape``, ``matvec`` (1-D
float64 array of length N in, fresh array out, ValueError mentioning
"length" otherwise) and ``@``.  The reference evaluates A x by circulant
FFT; here K1 (csrc/matvec.cu) evaluates the log-r / 1/r kernel on the fly
for every pair (BASELINE.json north star, component (1)); ToeplitzMatvec
defaults to K1b, the same circulant-FFT algorithm as the reference, on the
device.

Device API: ``matvec_device(X, Y, nrhs, row_begin, row_end)`` takes torch
CUDA float64 tensors and enqueues on the current stream without a host sync.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .kernel import KernelOperator


def to_device_vector(v, n: int):
    """(torch CUDA float64 tensor, was_numpy).  Validates length n.  A numpy
    input backed by pinned (page-locked) memory is copied by DMA directly."""
    torch = _lib.torch_cuda()
    if isinstance(v, torch.Tensor):
        if v.shape != (n,):
            raise ValueError(f"expected vector of length {n}, got shape {tuple(v.shape)}")
        t = v.to(device="cuda", dtype=torch.float64).contiguous()
        return t, False
    a = np.asarray(v, dtype=float)
    if a.shape != (n,):
        raise ValueError(f"expected vector of length {n}, got shape {a.shape}")
    # (non_blocking: from page-locked memory the copy is stream-ordered and the host
    # goes on to enqueue the kernels behind it; from pageable memory it is staged
    # synchronously either way)
    return torch.from_numpy(np.ascontiguousarray(a)).to("cuda", non_blocking=True), True


def to_host(t, was_numpy: bool):
    """Device result -> fresh numpy array (the reference returns fresh arrays).
    The copy lands in page-locked memory from torch's caching host allocator
    (DMA at full PCIe/C2C rate instead of a staged pageable copy); the array
    keeps its buffer alive and returns it to the cache when released."""
    if not was_numpy:
        return t
    torch = _lib.torch_cuda()
    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
    h.copy_(t)
    return h.numpy()


FFT_MAX_N = 4096  # circulant lines of up to 8192 points (csrc/fft.cu kFftMaxPoints)


def fft_size(n: int) -> int:
    """Circulant embedding size per axis: the smallest power of two >= 2n - 1
    (at least 4).  The reference embeds in exactly 2n (toeplitz.py:19-30,
    pocketfft handles any length); any size >= 2n - 1 gives the same Toeplitz
    product, and a power of two keeps every line transform radix-2^k -- for
    power-of-two n the two coincide."""
    m = 4
    while m < 2 * n - 1:
        m *= 2
    return m


def fft_supported(n: int, dim: int = 2) -> bool:
    """The FFT path covers every 2 <= n <= 4096; in 3D the setup's M^3
    complex embedding is kept under 4 GiB (n <= 128)."""
    if not 2 <= n <= FFT_MAX_N:
        return False
    return dim < 3 or fft_size(n) ** 3 * 16 <= 4 << 30


class KernelMatvec:
    """Device matvec y = A x.

    method="direct" (default here): K1, the O(N^2) matrix-free sum with the
    log-r / 1/r kernel evaluated for every pair (csrc/matvec.cu).
    method="fft": K1b, the reference's circulant-embedding FFT algorithm in
    hand-written FP64 Stockham kernels (csrc/fft.cu).
    """

    def __init__(self, op: KernelOperator, method: str = "direct"):
        if method == "auto":
            method = "fft" if fft_supported(op.grid.n_per_dim, op.grid.dim) else "direct"
        if method not in _lib.MATVEC_METHODS:
            raise ValueError(f"method must be one of {tuple(_lib.MATVEC_METHODS)} or 'auto', got {method!r}")
        if method == "fft" and not fft_supported(op.grid.n_per_dim, op.grid.dim):
            raise ValueError(f"method='fft' needs 2 <= n_per_dim <= {FFT_MAX_N} (3D: <= 128), "
                             f"got {op.grid.n_per_dim}")
        self.op = op
        self.method = method
        self.dim = op.grid.dim
        self.n = op.grid.n_per_dim
        self.N = op.n
        self.M = fft_size(self.n) if method == "fft" else 0  # circulant size per axis (FFT method)
        self._lib = _lib.lib()
        h = ctypes.c_void_p()
        _lib.check(self._lib.ie_matvec_create_method(op.geom(), _lib.MATVEC_METHODS[method], ctypes.byref(h)),
                   "ToeplitzMatvec")
        self._handle = h

    def __del__(self):
        h = getattr(self, "_handle", None)
        if h is not None and h.value:
            self._lib.ie_matvec_destroy(h)
            self._handle = None

    @property
    def handle(self):
        return self._handle

    @property
    def shape(self) -> tuple:
        return (self.N, self.N)

    def matvec_device(self, X, Y, nrhs: int = 1, row_begin: int = 0, row_end: int | None = None,
                      ldx: int | None = None, ldy: int | None = None):
        """Y[:, c] = A[row_begin:row_end] X[:, c] for c < nrhs, columns at
        stride ldx / ldy (default N / row count).  No host synchronisation."""
        row_end = self.N if row_end is None else row_end
        ldx = self.N if ldx is None else ldx
        ldy = (row_end - row_begin) if ldy is None else ldy
        rc = self._lib.ie_matvec_f64(self._handle, _lib.ptr(X), ldx, nrhs, _lib.ptr(Y), ldy,
                                     row_begin, row_end, _lib.stream_ptr())
        _lib.check(rc, "matvec")
        return Y

    def matvec(self, v):
        x, was_np = to_device_vector(v, self.N)
        torch = _lib.torch_cuda()
        y = torch.empty_like(x)
        self.matvec_device(x, y)
        return to_host(y, was_np)

    def __matmul__(self, v):
        return self.matvec(v)


class ToeplitzMatvec(KernelMatvec):
    """Drop-in for the reference's ToeplitzMatvec: method="auto" picks the
    FFT algorithm the reference uses (any n up to 4096; 3D up to 128), else
    the direct sum."""

    def __init__(self, op: KernelOperator, method: str = "auto"):
        super().__init__(op, method=method)


def build_matvec(op: KernelOperator, method: str = "auto") -> KernelMatvec:
    return ToeplitzMatvec(op, method=method)
