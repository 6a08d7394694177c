"""CPU ORACLE for the Schwarz-PCG hot path -- TEST INFRASTRUCTURE ONLY.

This module is a numpy/scipy restatement of the reference package's algorithm
(iedd 0.1.0, /root/reference/pkg/src/iedd) for the functions on the hot path
(SURVEY.md section 8(a), rows a1-a11).  It exists to CHECK the CUDA product:
only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference leg may import it.  The product package never imports it and has no
CPU fallback.

Pinning: tests/test_oracle.py checks this restatement against
  * the reference's own known-answer constants (tests/test_kernel.py:16-18,
    :91-99 of the reference),
  * the reference's golden suites (goldens.json iterations-2d/3d, spectrum-2d/3d,
    schwarz-scaling-2d, pairing) shipped as paper_2108_12574_b200/data/goldens.json, and
  * golden vectors produced by running the unmodified reference in the build
    container (tools/gen_goldens.py -> tests/golden/ref_*.npz).

Line citations are to the reference's own files, e.g. kernel.py:170-184 means
/root/reference/pkg/src/iedd/kernel.py lines 170-184.
"""

from __future__ import annotations

import itertools
import math
import time
from dataclasses import dataclass, field

import numpy as np
import scipy.linalg as sla

TWO_PI = 2.0 * np.pi
STAGNATION_WINDOW = 30          # pcg.py:11
STAGNATION_FACTOR = 1e-3        # pcg.py:12
DENSE_LIMIT_DEFAULT = 4096      # precond.py:23


class NotPositiveDefinite(RuntimeError):
    """linalg.py:17-18."""


# --------------------------------------------------------------------------
# geometry (geometry.py:23-244): C-order grid, uniform boxes, dilation
# --------------------------------------------------------------------------
@dataclass(frozen=True)
class Grid:
    dim: int
    n_per_dim: int

    @property
    def spacing(self) -> float:
        return 1.0 / self.n_per_dim

    @property
    def n_points(self) -> int:
        return self.n_per_dim ** self.dim

    @property
    def shape(self):
        return (self.n_per_dim,) * self.dim

    def multi_indices(self) -> np.ndarray:
        # geometry.py:42-44: (N, dim) in C order, last axis fastest
        grids = np.meshgrid(*[np.arange(self.n_per_dim)] * self.dim, indexing="ij")
        return np.stack([g.ravel() for g in grids], axis=1).astype(np.int64)


def build_grid(dim: int, n: int) -> Grid:
    # geometry.py:58-68
    if dim not in (1, 2, 3):
        raise ValueError(f"dim must be 1, 2 or 3, got {dim}")
    if n < 2:
        raise ValueError(f"n_per_dim must be >= 2, got {n}")
    return Grid(dim, n)


def box_indices(grid: Grid, lo, hi) -> np.ndarray:
    """geometry.py:71-82: sorted indices of the inclusive box, clipped."""
    lo = np.maximum(np.asarray(lo), 0)
    hi = np.minimum(np.asarray(hi), grid.n_per_dim - 1)
    if np.any(hi < lo):
        return np.zeros(0, dtype=np.int64)
    axes = [np.arange(a, b + 1, dtype=np.int64) for a, b in zip(lo, hi)]
    flat = np.zeros(1, dtype=np.int64)
    for ax in axes:  # C order: previous axes are slower
        flat = (flat[:, None] * grid.n_per_dim + ax[None, :]).ravel()
    return np.sort(flat)


@dataclass(frozen=True)
class Decomposition:
    kind: str
    grid: Grid
    m_per_dim: int
    overlap_width: int
    subdomains: list = field(repr=False)


def build_decomposition(grid: Grid, m: int, w: int, kind: str) -> Decomposition:
    """geometry.py:108-148, 164-176, 209-244.  jacobi: the m^dim boxes of q^dim
    points; schwarz: boxes grown by w (clipped); cbd: per parity colour
    c = 1 + sum_d (cell_d mod 2) 2^d, the sorted union of its grown boxes."""
    kind = kind.lower()
    if kind not in ("jacobi", "schwarz", "cbd"):
        raise ValueError(f"kind must be 'jacobi', 'schwarz' or 'cbd', got {kind!r}")
    if m < 1:
        raise ValueError(f"m_per_dim must be >= 1, got {m}")
    if grid.n_per_dim % m:
        raise ValueError(f"m_per_dim={m} does not divide n_per_dim={grid.n_per_dim}")
    if w < 0:
        raise ValueError(f"overlap_width must be >= 0, got {w}")
    q = grid.n_per_dim // m
    ww = 0 if kind == "jacobi" else w
    boxes, colours = [], []
    for cell in itertools.product(range(m), repeat=grid.dim):
        lo = np.array(cell, dtype=np.int64) * q
        boxes.append(box_indices(grid, lo - ww, lo + q - 1 + ww))
        colours.append(1 + sum((c % 2) << d for d, c in enumerate(cell)))
    if kind != "cbd":
        return Decomposition(kind, grid, m, ww, boxes)
    subs = []
    for col in range(1, 2 ** grid.dim + 1):
        members = [b for b, c in zip(boxes, colours) if c == col]
        subs.append(np.unique(np.concatenate(members)))
    return Decomposition(kind, grid, m, ww, subs)


# --------------------------------------------------------------------------
# operator entries (kernel.py:36-214)
# --------------------------------------------------------------------------
_GLX, _GLW = np.polynomial.legendre.leggauss(20)


def _panel_quadrature(fn, a, b, rtol=1e-13):
    """kernel.py:53-67: composite 20-point Gauss-Legendre, panels doubled
    until two successive levels agree to rtol."""
    last = None
    for level in range(13):
        npan = 2 ** level
        edges = a + (b - a) * np.arange(npan + 1) / npan
        c = 0.5 * (edges[1:] + edges[:-1])
        r = 0.5 * (edges[1:] - edges[:-1])
        pts = (c[:, None] + r[:, None] * _GLX[None, :]).ravel()
        wts = (r[:, None] * _GLW[None, :]).ravel()
        val = float(wts @ fn(pts))
        if last is not None and abs(val - last) <= rtol * max(abs(val), 1e-300):
            return val
        last = val
    raise RuntimeError("quadrature did not converge")


def diagonal_entry(dim: int, h: float) -> float:
    """kernel.py:70-99: singular self-integral of the kernel over one cell."""
    if h <= 0:
        raise ValueError(f"h must be positive, got {h}")
    half = 0.5 * h
    if dim == 2:
        def g(t):
            rr = half / np.cos(t)
            return rr * rr * (0.5 * np.log(rr) - 0.25)
        return -8.0 * _panel_quadrature(g, 0.0, np.pi / 4) / TWO_PI
    if dim == 3:
        def g(v):
            return 2.0 * np.arcsinh(1.0 / np.sqrt(1.0 + v * v))
        return 3.0 * half * half * _panel_quadrature(g, -1.0, 1.0) / (2.0 * TWO_PI)
    if dim == 1:
        return (h / TWO_PI) * (1.0 - np.log(half))
    raise ValueError(f"dim must be 1, 2 or 3, got {dim}")


@dataclass(frozen=True)
class Operator:
    grid: Grid
    lattice: str
    diag_value: float

    @property
    def n(self):
        return self.grid.n_points

    @property
    def lattice_spacing(self):
        # kernel.py:131-135
        return self.grid.spacing if self.lattice == "cell" else 1.0 / (self.grid.n_per_dim - 1)

    @property
    def weight(self):
        return self.grid.spacing ** self.grid.dim

    def coords(self):
        # kernel.py:141-144 (computed once here; the reference rebuilds it per call)
        return self.grid.multi_indices() * self.lattice_spacing

    def kernel_of_dist(self, dist):
        # kernel.py:146-149: 3D 1/(4 pi r); 1D and 2D -log(r)/(2 pi)
        if self.grid.dim == 3:
            return 1.0 / (2.0 * TWO_PI * dist)
        return -np.log(dist) / TWO_PI

    def assemble_block(self, rows, cols, coords=None):
        """kernel.py:170-184: weight*K(|c_i-c_j|), diag_value where d2 == 0."""
        c = self.coords() if coords is None else coords
        ri, rj = c[np.asarray(rows, dtype=np.int64)], c[np.asarray(cols, dtype=np.int64)]
        d2 = np.zeros((ri.shape[0], rj.shape[0]))
        for ax in range(self.grid.dim):
            dd = ri[:, ax][:, None] - rj[:, ax][None, :]
            d2 += dd * dd
        zero = d2 == 0.0
        out = self.weight * self.kernel_of_dist(np.sqrt(np.where(zero, 1.0, d2)))
        out[zero] = self.diag_value
        return out

    def dense(self):
        idx = np.arange(self.n)
        return self.assemble_block(idx, idx)

    def generator(self):
        """kernel.py:190-199: kernel over non-negative lags; lag 0 = diagonal."""
        n = self.grid.n_per_dim
        lag = np.indices((n,) * self.grid.dim).astype(float) * self.lattice_spacing
        d2 = (lag * lag).sum(axis=0)
        gen = self.weight * self.kernel_of_dist(np.sqrt(np.where(d2 == 0.0, 1.0, d2)))
        gen[(0,) * self.grid.dim] = self.diag_value
        return gen


def build_operator(grid: Grid, lattice: str | None = None) -> Operator:
    """kernel.py:202-214; default lattice is span in 2D, cell otherwise."""
    lat = lattice or ("span" if grid.dim == 2 else "cell")
    if lat not in ("cell", "span"):
        raise ValueError(f"lattice must be 'cell' or 'span', got {lattice!r}")
    return Operator(grid, lat, diagonal_entry(grid.dim, grid.spacing))


class FFTMatvec:
    """toeplitz.py:11-53: (2n)^d circulant embedding of the multilevel
    Toeplitz operator, applied with real FFTs.  workers > 1 (bench.py's CPU
    reference arm only): the same pocketfft transforms through scipy.fft on
    that many host threads."""

    def __init__(self, op: Operator, workers: int = 1):
        self.workers = workers
        self.dim, self.n = op.grid.dim, op.grid.n_per_dim
        n, d = self.n, self.dim
        emb = np.zeros((2 * n,) * d)
        emb[(slice(0, n),) * d] = op.generator()
        for ax in range(d):
            src = [slice(None)] * d
            dst = [slice(None)] * d
            src[ax] = slice(1, n)
            dst[ax] = slice(2 * n - 1, n, -1)
            emb[tuple(dst)] = emb[tuple(src)]
        self.shape_emb = emb.shape
        self.symbol = np.fft.rfftn(emb)

    def matvec(self, v):
        v = np.asarray(v, dtype=float)
        N = self.n ** self.dim
        if v.shape != (N,):
            raise ValueError(f"expected vector of length {N}, got shape {v.shape}")
        pad = np.zeros(self.shape_emb)
        pad[(slice(0, self.n),) * self.dim] = v.reshape((self.n,) * self.dim)
        if self.workers > 1:
            import scipy.fft as sfft
            out = sfft.irfftn(sfft.rfftn(pad, workers=self.workers) * self.symbol, s=self.shape_emb,
                              axes=tuple(range(self.dim)), workers=self.workers)
        else:
            out = np.fft.irfftn(np.fft.rfftn(pad) * self.symbol, s=self.shape_emb,
                                axes=tuple(range(self.dim)))
        return out[(slice(0, self.n),) * self.dim].reshape(N)

    __call__ = matvec


# --------------------------------------------------------------------------
# preconditioner (precond.py:91-100, 157-215; linalg.py:31-58)
# --------------------------------------------------------------------------
class SchwarzPrecond:
    """T^{-1} = sum_k R_k^T (G_k^T G_k)^{-1} R_k with upper Cholesky G_k,
    accumulated in ascending k from zeros (precond.py:97-99)."""

    def __init__(self, op: Operator, dec: Decomposition, dense_limit=DENSE_LIMIT_DEFAULT):
        t0 = time.perf_counter()
        coords = op.coords()
        self.n = op.n
        self.kind = dec.kind
        self.indices = []
        self.factors = []
        for k, idx in enumerate(dec.subdomains):
            if idx.size > dense_limit:
                raise ValueError(f"subdomain {k} has {idx.size} points > dense_limit="
                                 f"{dense_limit}; use backend='rskel'")
            a = op.assemble_block(idx, idx, coords)
            try:
                g = sla.cholesky(a, lower=False, check_finite=False)
            except sla.LinAlgError as exc:
                raise NotPositiveDefinite(f"subdomain {k}: matrix is not positive definite") from exc
            self.indices.append(idx)
            self.factors.append(g)
        self.t_factor = time.perf_counter() - t0

    def apply(self, f):
        f = np.asarray(f, dtype=float)
        if f.shape != (self.n,):
            raise ValueError(f"expected vector of length {self.n}, got {f.shape}")
        out = np.zeros_like(f)
        for idx, g in zip(self.indices, self.factors):
            y = sla.solve_triangular(g, f[idx], trans="T", lower=False, check_finite=False)
            out[idx] += sla.solve_triangular(g, y, trans="N", lower=False, check_finite=False)
        return out

    __call__ = apply

    def apply_dense(self):
        out = np.zeros((self.n, self.n))
        for idx, g in zip(self.indices, self.factors):
            inv = sla.cho_solve((g, False), np.eye(idx.size))
            out[np.ix_(idx, idx)] += inv
        return 0.5 * (out + out.T)


class PooledApply:
    """SchwarzPrecond.apply on all host cores (bench.py's CPU reference arm
    only): worker processes forked after the factorisation (the factors are
    shared copy-on-write) each solve a contiguous range of blocks with the
    same two solve_triangular calls into a shared staging buffer; the parent
    accumulates out[idx_k] += z_k in ascending k (np.add.at applies the updates
    in order), exactly the reference's sum.  Threads do not help here: the
    per-block scipy call overhead holds the GIL (measured, c3: 61 ms at 1 and
    at 8 threads)."""

    def __init__(self, pre: "SchwarzPrecond", nproc: int):
        import multiprocessing as mp
        from multiprocessing import shared_memory
        self.pre = pre
        self.n = pre.n
        sizes = np.array([i.size for i in pre.indices])
        self.off = np.concatenate([[0], np.cumsum(sizes)])
        self.cat = np.concatenate(pre.indices)
        self._f = shared_memory.SharedMemory(create=True, size=8 * pre.n)
        self._z = shared_memory.SharedMemory(create=True, size=8 * int(self.off[-1]))
        D = len(pre.indices)
        self.ranges = [(D * t // nproc, D * (t + 1) // nproc) for t in range(nproc)]
        global _POOL_STATE
        _POOL_STATE = (pre, self.off, self._f.name, self._z.name)
        self.pool = mp.get_context("fork").Pool(nproc)
        self.fbuf = np.ndarray((pre.n,), dtype=np.float64, buffer=self._f.buf)
        self.zbuf = np.ndarray((int(self.off[-1]),), dtype=np.float64, buffer=self._z.buf)

    def apply(self, f):
        self.fbuf[:] = np.asarray(f, dtype=float)
        self.pool.map(_pooled_solve, self.ranges)
        out = np.zeros(self.n)
        np.add.at(out, self.cat, self.zbuf)
        return out

    __call__ = apply

    def close(self):
        self.pool.terminate()
        self._f.close()
        self._f.unlink()
        self._z.close()
        self._z.unlink()


_POOL_STATE = None


def _pooled_solve(rng):
    from multiprocessing import shared_memory
    pre, off, fname, zname = _POOL_STATE
    fs = shared_memory.SharedMemory(name=fname)
    zs = shared_memory.SharedMemory(name=zname)
    f = np.ndarray((pre.n,), dtype=np.float64, buffer=fs.buf)
    z = np.ndarray((int(off[-1]),), dtype=np.float64, buffer=zs.buf)
    for k in range(*rng):
        g = pre.factors[k]
        y = sla.solve_triangular(g, f[pre.indices[k]], trans="T", lower=False, check_finite=False)
        z[off[k]:off[k + 1]] = sla.solve_triangular(g, y, trans="N", lower=False, check_finite=False)
    del f, z
    fs.close()
    zs.close()
    return 0


# --------------------------------------------------------------------------
# PCG (pcg.py:36-136)
# --------------------------------------------------------------------------
@dataclass
class PcgResult:
    n_it: int
    achieved_residual: float
    t_pcg: float
    t_s: float
    residual_history: list
    stagnated: bool = False
    converged: bool = False


def _callable(op):
    if callable(op):
        return op
    if hasattr(op, "matvec"):
        return op.matvec
    return op.apply


def make_rhs(matvec, n, mode="random", seed=0):
    """pcg.py:36-51."""
    if mode == "random":
        ue = np.random.default_rng(seed).standard_normal(n)
        return _callable(matvec)(ue), ue
    if mode == "noise":
        return np.random.default_rng(seed).standard_normal(n), None
    if mode == "ones":
        return np.ones(n), None
    raise ValueError(f"rhs mode must be 'random', 'noise' or 'ones', got {mode!r}")


def pcg(matvec, precond, f, tol=1e-12, max_iters=None):
    """pcg.py:54-136: PCG from u0 = 0 with the TRUE residual ||f - A u|| as
    the stopping quantity, 30-iteration / 1e-3 stagnation window, breakdown
    on non-positive or non-finite p^T A p."""
    if not 0.0 < tol < 1.0:
        raise ValueError(f"tol must be in (0, 1), got {tol}")
    A = _callable(matvec)
    T = _callable(precond) if precond is not None else (lambda x: x.copy())
    f = np.asarray(f, dtype=float)
    n = f.size
    if max_iters is None:
        max_iters = max(2 * n, 100)
    nf = float(np.linalg.norm(f))
    u = np.zeros(n)
    if nf == 0.0:
        return u, PcgResult(0, 0.0, 0.0, 0.0, [0.0], converged=True)
    t0 = time.perf_counter()
    tprec, nprec = 0.0, 0
    r = f.copy()
    ts = time.perf_counter()
    z = T(r)
    tprec += time.perf_counter() - ts
    nprec += 1
    p = z.copy()
    rho = float(r @ z)
    hist = [1.0]
    stag = conv = False
    k = 0
    while k < max_iters:
        k += 1
        q = A(p)
        den = float(p @ q)
        if not np.isfinite(den) or den <= 0.0:
            raise FloatingPointError(f"PCG breakdown at iteration {k}: p^T A p = {den}")
        alpha = rho / den
        u += alpha * p
        r -= alpha * q
        rel = float(np.linalg.norm(f - A(u))) / nf
        if not np.isfinite(rel):
            raise FloatingPointError(f"non-finite residual at iteration {k}")
        hist.append(rel)
        if rel <= tol:
            conv = True
            break
        if k >= STAGNATION_WINDOW and rel > (1.0 - STAGNATION_FACTOR) * hist[k - STAGNATION_WINDOW]:
            stag = True
            break
        ts = time.perf_counter()
        z = T(r)
        tprec += time.perf_counter() - ts
        nprec += 1
        rho_new = float(r @ z)
        p = z + (rho_new / rho) * p
        rho = rho_new
    return u, PcgResult(k, hist[-1], time.perf_counter() - t0, tprec / max(nprec, 1),
                        hist, stag, conv)


# --------------------------------------------------------------------------
# Lanczos (spectrum.py:133-190) and the dense spectrum used to pin it
# --------------------------------------------------------------------------
def lanczos_extremal(matvec, precond, n, which="min", max_iters=400, rtol=1e-9, seed=0):
    """A-inner-product Lanczos on T^{-1}A with two-pass MGS
    reorthogonalisation; stop after 5 consecutive stable Ritz values."""
    if which not in ("min", "max"):
        raise ValueError(f"which must be 'min' or 'max', got {which!r}")
    A = matvec.matvec if hasattr(matvec, "matvec") else matvec
    v = np.random.default_rng(seed).standard_normal(n)
    av = A(v)
    s = np.sqrt(v @ av)
    v, av = v / s, av / s
    V, AV = [v], [av]
    al, be = [], []
    est, stable = None, 0
    for j in range(max_iters):
        w = precond.apply(AV[j])
        al.append(float(w @ AV[j]))
        for _ in range(2):
            for vi, avi in zip(V, AV):
                w -= (w @ avi) * vi
        aw = A(w)
        b2 = float(w @ aw)
        if b2 <= 0 or not np.isfinite(b2):
            break
        b = math.sqrt(b2)
        ritz = sla.eigvalsh_tridiagonal(np.array(al), np.array(be))
        cur = float(ritz[0] if which == "min" else ritz[-1])
        if est is not None and abs(cur - est) <= rtol * max(abs(cur), 1.0):
            stable += 1
            if stable >= 5:
                return cur
        else:
            stable = 0
        est = cur
        if b < 1e-14:
            break
        be.append(b)
        V.append(w / b)
        AV.append(aw / b)
    if est is None:
        raise RuntimeError("Lanczos produced no Ritz values")
    return est


def dense_spectrum(op: Operator, pre: SchwarzPrecond):
    """spectrum.py:47-69: eigenvalues of G^T A G with T^{-1} = G G^T."""
    g = sla.cholesky(pre.apply_dense(), lower=True, check_finite=False)
    return sla.eigh(g.T @ (op.dense() @ g), eigvals_only=True, check_finite=False)
