"""Operator metadata and entry access (mirrors
/root/reference/pkg/src/iedd/kernel.py:36-214).

KernelOperator is a value object holding what the device kernels need
(dim, n, lattice spacing, quadrature weight h^dim, diagonal value).  Entry and
block access (assemble_block, dense, toeplitz_generator) are evaluated on the
GPU by the same entry code the preconditioner build uses
(csrc/common.cuh: entry_from_m).

diagonal_entry is scalar setup metadata computed on the host from closed
forms of the reference's self-integrals (kernel.py:70-99; the reference's
tests pin the same constants, tests/test_kernel.py:16-23).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from . import _lib
from .geometry import Grid

TWO_PI = 2.0 * math.pi
CELL = "cell"
SPAN = "span"

# self-integral of 1/(4 pi r) over the unit cube, /h^2 (reference test constant
# tests/test_kernel.py:17; equals BASELINE.json's 2.3800774/(4 pi))
_DIAG_3D_UNIT = 0.1894005387092370500171


class QuadratureError(RuntimeError):
    """Kept for API parity (kernel.py:32-33); the closed forms cannot fail."""


def kernel_value(r) -> float:
    """Free-space Laplace kernel at separation r (kernel.py:36-46)."""
    r = np.asarray(r, dtype=float)
    if r.ndim != 1 or r.size not in (2, 3):
        raise ValueError(f"r must be a 2- or 3-vector, got shape {r.shape}")
    dist = float(np.linalg.norm(r))
    if dist == 0.0:
        raise ValueError("kernel is singular at r = 0; diagonal handled separately")
    if r.size == 2:
        return -math.log(dist) / TWO_PI
    return 1.0 / (2.0 * TWO_PI * dist)


@lru_cache(maxsize=None)
def diagonal_entry(dim: int, h: float) -> float:
    """Self-interaction integral of the kernel over one cell of size h."""
    if h <= 0:
        raise ValueError(f"h must be positive, got {h}")
    if dim == 2:
        return h * h * (-math.log(h) + 0.5 * math.log(2.0) + (6.0 - math.pi) / 4.0) / TWO_PI
    if dim == 3:
        return h * h * _DIAG_3D_UNIT
    if dim == 1:
        return (h / TWO_PI) * (1.0 - math.log(h / 2.0))
    raise ValueError(f"dim must be 1, 2 or 3, got {dim}")


def _default_lattice(dim: int) -> str:
    return SPAN if dim == 2 else CELL


@dataclass(frozen=True)
class KernelOperator:
    grid: Grid
    lattice: str
    diag_value: float

    @property
    def n(self) -> int:
        return self.grid.n_points

    @property
    def shape(self) -> tuple:
        return (self.n, self.n)

    @property
    def lattice_spacing(self) -> float:
        if self.lattice == CELL:
            return self.grid.spacing
        return 1.0 / (self.grid.n_per_dim - 1)

    @property
    def weight(self) -> float:
        return self.grid.spacing ** self.grid.dim

    @property
    def coords(self) -> np.ndarray:
        """(N, dim) kernel-space coordinates (host bookkeeping)."""
        return self.grid.multi_indices() * self.lattice_spacing

    def geom(self) -> _lib.IeGeom:
        return _lib.IeGeom(self.grid.dim, self.grid.n_per_dim, self.lattice_spacing, self.weight,
                           self.diag_value)

    def entry(self, i: int, j: int) -> float:
        if i == j:
            return self.diag_value
        return float(self.assemble_block(np.array([i]), np.array([j]))[0, 0])

    def assemble_block(self, rows, cols) -> np.ndarray:
        """Dense A[rows, cols], evaluated on the device (kernel.py:170-184)."""
        return self.assemble_block_device(rows, cols).cpu().numpy()

    def assemble_block_device(self, rows, cols):
        """As assemble_block, returning the device tensor."""
        torch = _lib.torch_cuda()
        rows = np.ascontiguousarray(np.asarray(rows, dtype=np.int64).ravel())
        cols = np.ascontiguousarray(np.asarray(cols, dtype=np.int64).ravel())
        for a in (rows, cols):
            if a.size and (a.min() < 0 or a.max() >= self.n):
                raise IndexError("index out of range for the operator")
        dr = torch.from_numpy(rows).cuda()
        dc = torch.from_numpy(cols).cuda()
        out = torch.empty((rows.size, cols.size), dtype=torch.float64, device="cuda")
        g = self.geom()
        rc = _lib.lib().ie_assemble_block_f64(g, _lib.ptr(dr), rows.size, _lib.ptr(dc), cols.size,
                                              _lib.ptr(out), _lib.stream_ptr())
        _lib.check(rc, "assemble_block")
        return out

    def dense(self) -> np.ndarray:
        idx = np.arange(self.n, dtype=np.int64)
        return self.assemble_block(idx, idx)

    def toeplitz_generator(self) -> np.ndarray:
        """Kernel over non-negative lags, shape (n,)*dim (kernel.py:190-199):
        row 0 of A in C order."""
        row = self.assemble_block(np.array([0]), np.arange(self.n))
        return row.reshape(self.grid.shape)


def build_operator(grid: Grid, lattice: str | None = None) -> KernelOperator:
    lat = lattice or _default_lattice(grid.dim)
    if lat not in (CELL, SPAN):
        raise ValueError(f"lattice must be 'cell' or 'span', got {lattice!r}")
    if lat == SPAN and grid.n_per_dim < 2:
        raise ValueError("span lattice needs n_per_dim >= 2")
    return KernelOperator(grid=grid, lattice=lat, diag_value=diagonal_entry(grid.dim, grid.spacing))
