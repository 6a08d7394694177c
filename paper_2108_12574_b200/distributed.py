"""Sharded Schwarz-PCG across the ranks of a torch.distributed group
(one process per GPU, NCCL over NVLink).

Partitioning.  Rank g owns a contiguous band [b_g, e_g) of the C-ordered
unknowns: the first lattice axis is split at subdomain-row boundaries and the
cut points are rounded to the dot-product chunk (2048) so that every
fixed-chunk partial lives on exactly one rank.  Per iteration:

  * the fused 2-RHS A-pass [p, u] -> [q, w] for the band's rows:
      - FFT method, 2D (BandFFT): row FFTs of the band, an all-to-all
        transpose to column slabs, column FFT * symbol * inverse, the reverse
        all-to-all, inverse row FFTs -- no rank ever holds the whole iterate;
      - otherwise (K1 direct sum, 3D FFT): all-gather of [p, u], then the
        band's rows (K1 rows are summed in the same order for any row range;
        the replicated FFT computes all rows and keeps the band),
  * all-gather of the fixed-chunk dot partials, reduced on every rank by the
    same device kernel and order as the single-GPU solver,
  * r-halo exchange for the apply (one all-to-all in which only neighbouring
    bands send): each rank applies the subdomains that intersect its band
    (neighbours' overlap blocks are recomputed), so the z values of its band
    are summed in ascending global block id -- the reference's order.

Every scalar and every owned vector entry is therefore bitwise identical for
any number of ranks, and identical to ie_pcg_f64 on one GPU.

The compute backend is pluggable: CudaBackend (C-ABI kernels) in production;
the CPU tests inject a numpy backend and run the same driver over gloo.
"""

from __future__ import annotations

import ctypes
import math
import time
from dataclasses import dataclass, field

import numpy as np

CHUNK = 2048
STAGNATION_WINDOW = 30
STAGNATION_FACTOR = 1e-3


def dist_fft_disabled() -> bool:
    """IEDD_B200_NO_DIST_FFT=1: replicate the FFT on every rank (all-gather of
    the iterate) instead of the band decomposition (comparison runs)."""
    import os
    return bool(os.environ.get("IEDD_B200_NO_DIST_FFT"))


# --------------------------------------------------------------------------
# plan
# --------------------------------------------------------------------------
def band_bounds(grid, m_per_dim: int, world: int, chunk: int = CHUNK) -> tuple:
    """Cut points (world+1) of the rank bands: subdomain-row boundaries of the
    first lattice axis, rounded to multiples of `chunk`, monotone."""
    N = grid.n_points
    n = grid.n_per_dim
    m = max(1, min(m_per_dim, n))
    line = n ** (grid.dim - 1)
    cuts = []
    for g in range(world + 1):
        first_line = (m * g // world) * (n // m)
        idx = first_line * line
        idx = min(N, int(round(idx / chunk)) * chunk)
        cuts.append(idx)
    cuts[0], cuts[-1] = 0, N
    for i in range(1, len(cuts)):
        cuts[i] = max(cuts[i], cuts[i - 1])
    return tuple(cuts)


@dataclass(frozen=True)
class ShardPlan:
    world: int
    rank: int
    N: int
    bounds: tuple
    blocks: np.ndarray = field(repr=False)  # global subdomain ids applied on this rank (ascending)
    need: tuple = ()  # per rank: [lo, hi) of the points its blocks touch (band + halo)

    @property
    def begin(self) -> int:
        return self.bounds[self.rank]

    @property
    def end(self) -> int:
        return self.bounds[self.rank + 1]

    @property
    def size(self) -> int:
        return self.end - self.begin

    def chunks(self, r: int | None = None) -> tuple:
        r = self.rank if r is None else r
        b, e = self.bounds[r], self.bounds[r + 1]
        return (b // CHUNK, -(-e // CHUNK)) if e > b else (b // CHUNK, b // CHUNK)


def blocks_intersecting(subdomains, begin: int, end: int) -> np.ndarray:
    out = []
    for k, idx in enumerate(subdomains):
        j = np.searchsorted(idx, begin)
        if j < idx.size and idx[j] < end:
            out.append(k)
    return np.array(out, dtype=np.int64)


def make_plan(grid, decomposition, world: int, rank: int) -> ShardPlan:
    bounds = band_bounds(grid, getattr(decomposition, "m_per_dim", 1), world)
    subs = decomposition.subdomains
    lo_k = np.array([int(s[0]) if s.size else 0 for s in subs])     # index sets are sorted
    hi_k = np.array([int(s[-1]) + 1 if s.size else 0 for s in subs])
    need, blocks = [], None
    for g in range(world):
        bg = blocks_intersecting(subs, bounds[g], bounds[g + 1])
        if g == rank:
            blocks = bg
        lo = min([bounds[g]] + [int(lo_k[k]) for k in bg])
        hi = max([bounds[g + 1]] + [int(hi_k[k]) for k in bg])
        need.append((lo, hi))
    return ShardPlan(world=world, rank=rank, N=grid.n_points, bounds=bounds, blocks=blocks, need=tuple(need))


@dataclass(frozen=True)
class SubDecomposition:
    """The subset of a decomposition a rank applies (ascending global ids)."""

    kind: str
    subdomains: list
    global_ids: np.ndarray

    @property
    def n_subdomains(self) -> int:
        return len(self.subdomains)


# --------------------------------------------------------------------------
# communication
# --------------------------------------------------------------------------
class Comm:
    """Band all-gathers over torch.distributed (NCCL for CUDA tensors, gloo
    for CPU tensors).  Bands are padded to the longest one."""

    def __init__(self, plan: ShardPlan, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.plan = plan
        self.maxlen = max(plan.bounds[i + 1] - plan.bounds[i] for i in range(plan.world))
        self.maxch = max(plan.chunks(i)[1] - plan.chunks(i)[0] for i in range(plan.world))

    def _gather(self, x, length_of):
        import torch
        world = self.plan.world
        ncol, L = x.shape
        pad = self.maxlen if length_of == "band" else self.maxch
        buf = x.new_zeros((ncol, pad))
        buf[:, :L] = x
        outs = [torch.empty_like(buf) for _ in range(world)]
        if world == 1:
            outs[0].copy_(buf)
        else:
            self.dist.all_gather(outs, buf, group=self.group)
        pieces = []
        for r in range(world):
            if length_of == "band":
                n = self.plan.bounds[r + 1] - self.plan.bounds[r]
            else:
                c0, c1 = self.plan.chunks(r)
                n = c1 - c0
            pieces.append(outs[r][:, :n])
        return torch.cat(pieces, dim=1)

    def alltoall(self, send, send_counts, recv_counts):
        """Flat variable-size all-to-all: block h of `send` (send_counts[h]
        elements, rank order) goes to rank h; the blocks received are
        concatenated in rank order."""
        out = send.new_empty(int(sum(recv_counts)))
        if self.plan.world == 1:
            out.copy_(send)
        else:
            self.dist.all_to_all_single(out, send.contiguous(), [int(c) for c in recv_counts],
                                        [int(c) for c in send_counts], group=self.group)
        return out

    def halo(self, x, out):
        """Band vector x -> out (length N) holding every entry this rank's
        blocks read: its band plus the halo [need_lo, begin) and [end,
        need_hi) from the neighbouring bands (one all-to-all; only
        neighbours exchange non-empty blocks).  Entries outside stay stale."""
        p = self.plan
        g = p.rank
        lo_g, hi_g = p.need[g] if p.need else (0, p.N)

        def inter(a0, a1, b0, b1):
            return max(a0, b0), min(a1, b1)

        sends, scount, rcount, rpos = [], [], [], []
        for h in range(p.world):
            lo_h, hi_h = p.need[h] if p.need else (0, p.N)
            a, b = inter(p.begin, p.end, lo_h, hi_h)
            n_s = max(0, b - a) if h != g else 0
            sends.append(x[a - p.begin: a - p.begin + n_s])
            scount.append(n_s)
            a2, b2 = inter(p.bounds[h], p.bounds[h + 1], lo_g, hi_g)
            n_r = max(0, b2 - a2) if h != g else 0
            rcount.append(n_r)
            rpos.append(a2)
        out[p.begin: p.end] = x
        if p.world > 1:
            import torch
            recv = self.alltoall(torch.cat(sends), scount, rcount)
            off = 0
            for h in range(p.world):
                if rcount[h]:
                    out[rpos[h]: rpos[h] + rcount[h]] = recv[off: off + rcount[h]]
                    off += rcount[h]
        return out

    def allgather_band(self, x):
        """(ncol, band) -> (ncol, N) in global order."""
        return self._gather(x, "band")

    def allgather_partials(self, x):
        """(ncol, band chunks) -> (ncol, all chunks) in chunk order."""
        return self._gather(x, "chunks")


# --------------------------------------------------------------------------
# distributed FFT matvec (2D): row bands, two all-to-all transposes
# --------------------------------------------------------------------------
class BandFFT:
    """ToeplitzMatvec.matvec (toeplitz.py:39-50) across the rank bands without
    gathering the iterate.  Rank g holds grid rows [a_g, b_g); the 2n spectrum
    columns are split into G slabs of Mc = 2n / G.

      1. row FFTs of the band, written destination-major (slab h contiguous);
      2. all-to-all: rank g receives every grid row of its column slab;
      3. column FFT * symbol * inverse FFT of the slab;
      4. reverse all-to-all: rank g receives its rows of every slab;
      5. inverse row FFTs -> the band of A x.

    With two right-hand sides the exact power-of-two column scaling uses the
    all-gathered per-chunk maxima, so every rank scales identically.  The
    per-line arithmetic is that of the single-GPU pass (same kernels, same
    data), so the result does not depend on G.  Per iteration and rank this
    moves 2 x 16 * n * (2n) / G bytes instead of all-gathering [p, u]."""

    def __init__(self, stages, plan: ShardPlan, n: int):
        self.st = stages
        self.plan = plan
        self.n = n
        self.G = plan.world
        self.M = 2 * n
        self.Mc = self.M // self.G
        self.rows = [((plan.bounds[h + 1] - plan.bounds[h]) // n) for h in range(self.G)]
        self.row0 = sum(self.rows[: plan.rank])

    @staticmethod
    def supported(grid, plan: ShardPlan) -> bool:
        n, G = grid.n_per_dim, plan.world
        M = 2 * n
        return (grid.dim == 2 and M % G == 0 and (M // G) & (M // G - 1) == 0
                and all(b % n == 0 for b in plan.bounds))

    def matvec(self, comm, Xb):
        """Xb: (ncol, band) -> (ncol, band) = rows [begin, end) of A x."""
        ncol = Xb.shape[0]
        amax = None
        if ncol == 2:
            part = self.st.absmax(Xb)                                    # (nch_band, 2)
            amax = comm.allgather_partials(part.T.contiguous()).T.contiguous().reshape(-1)
        g, G, Mc = self.plan.rank, self.G, self.Mc
        mine = self.rows[g]
        b1 = self.st.band_fwd(Xb, mine, G, amax)                          # (G, mine, Mc) complex
        b2 = comm.alltoall(b1, [2 * mine * Mc] * G, [2 * r * Mc for r in self.rows])
        self.st.band_cols(b2, g * Mc, Mc)                                 # (n, Mc) complex
        b3 = comm.alltoall(b2, [2 * r * Mc for r in self.rows], [2 * mine * Mc] * G)
        return self.st.band_inv(b3, mine, G, ncol, amax)


class CudaBandStages:
    """The band passes through the C-ABI (ie_matvec_band_*)."""

    def __init__(self, mv, plan: ShardPlan):
        import torch

        from . import _lib
        self.torch, self._lib, self.L = torch, _lib, _lib.lib()
        self.mv, self.plan = mv, plan
        self.namax = -(-plan.N // CHUNK)

    def absmax(self, Xb):
        n = Xb.shape[1]
        out = self.torch.empty(max(1, -(-n // CHUNK)), 2, dtype=self.torch.float64, device=Xb.device)
        self._lib.check(self.L.ie_absmax_partials_f64(self._lib.ptr(Xb), Xb.stride(0), n, self._lib.ptr(out),
                                                      self._lib.stream_ptr()), "absmax")
        return out[: -(-n // CHUNK)]

    def band_fwd(self, Xb, nrows, parts, amax):
        out = self.torch.empty(2 * nrows * self.mv.n * 2, dtype=self.torch.float64, device=Xb.device)
        self._lib.check(self.L.ie_matvec_band_fwd_f64(
            self.mv.handle, self._lib.ptr(Xb), Xb.stride(0), Xb.shape[0], self.plan.begin, self.plan.end, parts,
            self._lib.ptr(out), self._lib.ptr(amax) if amax is not None else None, self.namax,
            self._lib.stream_ptr()), "band_fwd")
        return out

    def band_cols(self, buf, c0, ncols):
        self._lib.check(self.L.ie_matvec_band_cols_f64(self.mv.handle, self._lib.ptr(buf), c0, c0 + ncols,
                                                       self._lib.stream_ptr()), "band_cols")

    def band_inv(self, buf, nrows, parts, ncol, amax):
        Y = self.torch.empty(ncol, self.plan.size, dtype=self.torch.float64, device=buf.device)
        self._lib.check(self.L.ie_matvec_band_inv_f64(
            self.mv.handle, self._lib.ptr(buf), self.plan.begin, self.plan.end, parts, self._lib.ptr(Y),
            self.plan.size, ncol, self._lib.ptr(amax) if amax is not None else None, self.namax,
            self._lib.stream_ptr()), "band_inv")
        return Y


# --------------------------------------------------------------------------
# CUDA backend (production)
# --------------------------------------------------------------------------
class CudaBackend:
    """Per-rank device work through the C-ABI (same kernels as ie_pcg_f64)."""

    def __init__(self, op, decomposition, plan: ShardPlan, method: str = "auto",
                 variant: str = "packed_inverse", share_translated: bool = True):
        import torch

        from . import _lib
        from .precond import from_decomposition
        from .toeplitz import KernelMatvec
        self.torch = torch
        self._lib = _lib
        self.L = _lib.lib()
        self.plan = plan
        self.N = plan.N
        if method == "auto":
            from .toeplitz import fft_supported
            method = "fft" if fft_supported(op.grid.n_per_dim) else "direct"
        self.mv = KernelMatvec(op, method=method)
        self.method = method
        self.band = (BandFFT(CudaBandStages(self.mv, plan), plan, op.grid.n_per_dim)
                     if method == "fft" and BandFFT.supported(op.grid, plan) and not dist_fft_disabled() else None)
        sub = SubDecomposition(decomposition.kind, [decomposition.subdomains[k] for k in plan.blocks],
                               plan.blocks)
        self.pre = (from_decomposition(op, sub, variant=variant, share_translated=share_translated)
                    if plan.blocks.size else None)
        self.dev = torch.device("cuda", torch.cuda.current_device())
        self._full = torch.empty(2, self.N, dtype=torch.float64, device=self.dev)
        self._scal = torch.empty(1, dtype=torch.float64, device=self.dev)

    def tensor(self, a):
        return self.torch.as_tensor(np.asarray(a, dtype=np.float64)).to(self.dev)

    def zeros(self, n):
        return self.torch.zeros(n, dtype=self.torch.float64, device=self.dev)

    def matvec_band(self, X):
        """X: (nrhs, N) full columns -> (nrhs, band) rows [begin, end)."""
        nrhs = X.shape[0]
        Y = self.torch.empty(nrhs, max(self.plan.size, 1), dtype=self.torch.float64, device=self.dev)
        if self.plan.size:
            X = X.contiguous()
            self.mv.matvec_device(X, Y, nrhs=nrhs, row_begin=self.plan.begin, row_end=self.plan.end,
                                  ldx=self.N, ldy=Y.shape[1])
        return Y[:, : self.plan.size]

    def matvec_cols(self, comm, Xb):
        """Band columns in, band rows of A x out (distributed FFT, or
        all-gather + the band rows of the full-range pass)."""
        if self.band is not None:
            return self.band.matvec(comm, Xb.contiguous())
        return self.matvec_band(comm.allgather_band(Xb))

    def apply_band(self, r_full):
        if self.pre is None:
            return self.zeros(0)
        z = self._full[0]
        self.pre.apply_device(r_full.contiguous(), z)
        return z[self.plan.begin: self.plan.end].clone()

    def dot_partials(self, x, y, mode: int):
        n = x.numel()
        out = self.torch.empty(max(1, -(-n // CHUNK)), dtype=self.torch.float64, device=self.dev)
        if n:
            self._lib.check(self.L.ie_dot_partials_f64(self._lib.ptr(x), self._lib.ptr(y), n, mode,
                                                       self._lib.ptr(out), self._lib.stream_ptr()), "dot")
        return out[: -(-n // CHUNK)] if n else out[:0]

    def sum_partials(self, parts) -> float:
        parts = parts.contiguous()
        self._lib.check(self.L.ie_sum_partials_f64(self._lib.ptr(parts), parts.numel(), self._lib.ptr(self._scal),
                                                   self._lib.stream_ptr()), "sum")
        return float(self._scal.item())

    def update(self, op: int, a, b, s: float):
        if a.numel():
            self._lib.check(self.L.ie_update_f64(op, self._lib.ptr(a), self._lib.ptr(b), float(s), a.numel(),
                                                 self._lib.stream_ptr()), "update")

    def sync(self):
        self.torch.cuda.synchronize()


# --------------------------------------------------------------------------
# the sharded solver (control flow of pcg.py:54-136, fused 2-RHS schedule)
# --------------------------------------------------------------------------
@dataclass
class ShardedReport:
    n_it: int
    achieved_residual: float
    t_pcg: float
    t_s: float
    residual_history: list
    stagnated: bool = False
    converged: bool = False


def solve_sharded(backend, comm: Comm, plan: ShardPlan, f_band, tol: float = 1e-12,
                  max_iters: int | None = None, gather_solution: bool = True):
    """PCG on the band decomposition; every rank returns the same report and
    (if gather_solution) the full solution."""
    if not 0.0 < tol < 1.0:
        raise ValueError(f"tol must be in (0, 1), got {tol}")
    N = plan.N
    if max_iters is None:
        max_iters = max(2 * N, 100)
    t0 = time.perf_counter()
    nf = math.sqrt(backend.sum_partials(comm.allgather_partials(backend.dot_partials(f_band, f_band, 0)[None])[0]))
    u = backend.zeros(plan.size)
    if nf == 0.0:
        full = comm.allgather_band(u[None])[0] if gather_solution else u
        return full, ShardedReport(0, 0.0, 0.0, 0.0, [0.0], converged=True)
    t_prec, n_prec = 0.0, 0
    r_buf = backend.zeros(N)

    def apply(r_band):
        nonlocal t_prec, n_prec
        ts = time.perf_counter()
        r_full = comm.halo(r_band, r_buf)
        z = backend.apply_band(r_full)
        backend.sync()
        t_prec += time.perf_counter() - ts
        n_prec += 1
        return z

    r = f_band.clone()
    z = apply(r)
    p = z.clone()
    rho = backend.sum_partials(comm.allgather_partials(backend.dot_partials(r, z, 0)[None])[0])
    hist = [1.0]
    k = 0
    pending = False
    conv = stag = False
    while True:
        it = k + 1
        do_p = it <= max_iters
        if not pending and not do_p:
            break
        cols = ([p] if do_p else []) + ([u] if pending else [])
        Y = backend.matvec_cols(comm, _stack(cols))
        q = Y[0] if do_p else None
        w = Y[-1] if pending else None
        parts = []
        if do_p:
            parts.append(backend.dot_partials(p, q, 0))
        if pending:
            parts.append(backend.dot_partials(f_band, w, 1))
        G = comm.allgather_partials(_stack(parts))
        row = 0
        denom = res2 = None
        if do_p:
            denom = backend.sum_partials(G[row])
            row += 1
        if pending:
            res2 = backend.sum_partials(G[row])
            rel = math.sqrt(res2) / nf
            if not math.isfinite(rel):
                raise FloatingPointError(f"non-finite residual at iteration {k}")
            hist.append(rel)
            if rel <= tol:
                conv = True
                break
            if k >= STAGNATION_WINDOW and rel > (1.0 - STAGNATION_FACTOR) * hist[k - STAGNATION_WINDOW]:
                stag = True
                break
            if not do_p:
                break
        if not math.isfinite(denom) or denom <= 0.0:
            raise FloatingPointError(f"PCG breakdown at iteration {it}: p^T A p = {denom}")
        alpha = rho / denom
        backend.update(0, u, p, alpha)
        backend.update(1, r, q, alpha)
        k = it
        pending = True
        if k < max_iters:
            z = apply(r)
            rz = backend.sum_partials(comm.allgather_partials(backend.dot_partials(r, z, 0)[None])[0])
            beta = rz / rho
            rho = rz
            backend.update(2, p, z, beta)
    full = comm.allgather_band(u[None])[0] if gather_solution else u
    rep = ShardedReport(n_it=k, achieved_residual=hist[-1], t_pcg=time.perf_counter() - t0,
                        t_s=t_prec / max(n_prec, 1), residual_history=hist, stagnated=stag, converged=conv)
    return full, rep


class NcclComm:
    """The library's own NCCL communicator over the ranks of the torch
    process group (the unique id travels by torch.distributed broadcast)."""

    def __init__(self, plan: ShardPlan, group=None):
        import torch.distributed as dist

        from . import _lib
        self._lib = _lib
        L = _lib.lib()
        nb = int(L.ie_comm_id_bytes())
        buf = ctypes.create_string_buffer(nb)
        if plan.rank == 0:
            _lib.check(L.ie_comm_unique_id(buf), "ie_comm_unique_id")
        obj = [buf.raw if plan.rank == 0 else None]
        if plan.world > 1:
            dist.broadcast_object_list(obj, src=0, group=group)
        idb = ctypes.create_string_buffer(obj[0], nb)
        h = ctypes.c_void_p()
        _lib.check(L.ie_comm_create(idb, plan.world, plan.rank, ctypes.byref(h)), "ie_comm_create")
        self.handle = h

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            self._lib.lib().ie_comm_destroy(h)
            self.handle = None


def native_supported(backend, plan: ShardPlan) -> bool:
    """ie_pcg_sharded_f64's domain: the band FFT and equal, chunk-aligned bands."""
    sizes = {plan.bounds[h + 1] - plan.bounds[h] for h in range(plan.world)}
    return backend.band is not None and len(sizes) == 1 and all(b % CHUNK == 0 for b in plan.bounds)


def solve_sharded_native(backend, ncomm: NcclComm, plan: ShardPlan, f_band, tol: float = 1e-12,
                         max_iters: int | None = None):
    """pcg.solve on the band decomposition through the native NCCL driver
    (ie_pcg_sharded_f64): device-side control, the iteration (collectives
    included) captured in a CUDA graph.  Returns (u_band, ShardedReport)."""
    from . import _lib
    if not 0.0 < tol < 1.0:
        raise ValueError(f"tol must be in (0, 1), got {tol}")
    if not native_supported(backend, plan):
        raise ValueError("native sharded PCG needs the 2D band FFT and equal chunk-aligned bands")
    if max_iters is None:
        max_iters = max(2 * plan.N, 100)
    u = backend.zeros(plan.size)
    hist = np.zeros(max_iters + 2, dtype=np.float64)
    n_it = ctypes.c_int64(0)
    flags = np.zeros(2, dtype=np.int32)
    times = np.zeros(2, dtype=np.float64)
    fail_it = ctypes.c_int64(0)
    fail_val = ctypes.c_double(0.0)
    bounds = np.ascontiguousarray(plan.bounds, dtype=np.int64)
    need = np.ascontiguousarray(np.array(plan.need, dtype=np.int64).reshape(-1)) if plan.need else None
    th = backend.pre.handle if backend.pre is not None else None
    f_band = f_band.contiguous()
    rc = _lib.lib().ie_pcg_sharded_f64(
        backend.mv.handle, th, ncomm.handle, _lib.np_ptr(bounds), _lib.np_ptr(need) if need is not None else None,
        _lib.ptr(f_band), _lib.ptr(u), tol, max_iters, _lib.np_ptr(hist), ctypes.byref(n_it), _lib.np_ptr(flags),
        _lib.np_ptr(times), ctypes.byref(fail_it), ctypes.byref(fail_val), _lib.stream_ptr())
    if rc == _lib.IE_ERR_BREAKDOWN:
        raise FloatingPointError(f"PCG breakdown at iteration {fail_it.value}: p^T A p = {fail_val.value}")
    if rc == _lib.IE_ERR_NONFINITE:
        raise FloatingPointError(f"non-finite residual at iteration {fail_it.value}")
    _lib.check(rc, "ie_pcg_sharded_f64")
    k = n_it.value
    h = [float(x) for x in hist[: k + 1]]
    return u, ShardedReport(n_it=k, achieved_residual=h[-1], t_pcg=float(times[0]), t_s=float(times[1]),
                            residual_history=h, stagnated=bool(flags[1]), converged=bool(flags[0]))


def lanczos_sharded(backend, comm: Comm, plan: ShardPlan, which: str = "min", max_iters: int = 400,
                    rtol: float = 1e-9, seed: int = 0, return_steps: bool = False):
    """Extremal eigenvalue of T^{-1}A by Lanczos in the A-inner product
    (spectrum.py:133-190) on the band decomposition: the basis V and A V are
    kept as band rows; every inner product is a fixed-chunk partial all-gather
    summed in global chunk order (so alphas, betas and the Ritz value are
    identical on every rank and for every G); the full reorthogonalisation is
    classical Gram-Schmidt applied twice (one partial all-gather per pass for
    all coefficients), the update w -= c_i v_i applied in ascending i."""
    import numpy as np
    from scipy.linalg import eigvalsh_tridiagonal

    if which not in ("min", "max"):
        raise ValueError(f"which must be 'min' or 'max', got {which!r}")

    def dot(x, y):
        return backend.sum_partials(comm.allgather_partials(backend.dot_partials(x, y, 0)[None])[0])

    r_buf = backend.zeros(plan.N)
    v = backend.tensor(np.random.default_rng(seed).standard_normal(plan.N)[plan.begin: plan.end])
    av = backend.matvec_cols(comm, v[None])[0]
    nrm = math.sqrt(dot(v, av))
    V = [v / nrm]
    AV = [av / nrm]
    alphas, betas = [], []
    estimate = None
    stable = 0
    steps = 1
    for j in range(max_iters):
        w = backend.apply_band(comm.halo(AV[j], r_buf))
        alphas.append(dot(w, AV[j]))
        for _ in range(2):
            parts = _stack([backend.dot_partials(w, avi, 0) for avi in AV])
            G = comm.allgather_partials(parts)
            coef = [backend.sum_partials(G[i]) for i in range(len(AV))]
            for c, vi in zip(coef, V):
                backend.update(0, w, vi, -c)
        aw = backend.matvec_cols(comm, w[None])[0]
        steps += 1
        beta2 = dot(w, aw)
        if beta2 <= 0 or not math.isfinite(beta2):
            break
        beta = math.sqrt(beta2)
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


def _stack(cols):
    import torch
    if isinstance(cols[0], torch.Tensor):
        return torch.stack(cols)
    return np.stack(cols)


# --------------------------------------------------------------------------
# bench entry for torchrun (bench.py --gpus N)
# --------------------------------------------------------------------------
def bench_sharded(args, metric, cfg, workload):
    """bench.py --gpus N under torchrun: config 5 on N ranks (bands of rows and
    subdomains).  Prints the contract JSON line on rank 0; time = max over ranks
    of the CUDA-event time of exactly `steps` iterations."""
    import json
    import os
    import statistics

    import torch
    import torch.distributed as dist

    import paper_2108_12574_b200 as ie

    from . import _lib
    ws, rank = dist.get_world_size(), dist.get_rank()
    grid = ie.build_grid(cfg["dim"], cfg["n"])
    op = ie.build_operator(grid, lattice="cell")
    dec = ie.build_decomposition(grid, cfg["m"], cfg["w"], "schwarz")
    plan = make_plan(grid, dec, ws, rank)
    backend = CudaBackend(op, dec, plan, method=getattr(args, "matvec", "auto"))
    comm = Comm(plan)
    f = np.random.default_rng(cfg["seed"]).standard_normal(op.n)
    f_band = backend.tensor(f[plan.begin: plan.end])
    native = native_supported(backend, plan) and not os.environ.get("IEDD_B200_PY_SHARDED")
    if native:
        ncomm = NcclComm(plan)

        def run(fb, iters, gather):
            u, rep = solve_sharded_native(backend, ncomm, plan, fb, tol=1e-10, max_iters=iters)
            return (comm.allgather_band(u[None])[0] if gather else u), rep
    else:
        def run(fb, iters, gather):
            return solve_sharded(backend, comm, plan, fb, tol=1e-10, max_iters=iters, gather_solution=gather)
    run(f_band, max(args.warmup, 1), False)
    dev = torch.device("cuda", torch.cuda.current_device())
    st = torch.cuda.current_stream()
    clocks = None
    if rank == 0:
        from bench import ClockSampler  # noqa: WPS433 (bench.py is the caller)
        clocks = ClockSampler(int(os.environ.get("LOCAL_RANK", "0")))
        clocks.start()
    dist.barrier()
    torch.cuda.synchronize()
    n0 = _lib.launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    _, rep = run(f_band, args.steps, False)
    e1.record(st)
    torch.cuda.synchronize()
    dist.barrier()
    launches = _lib.launch_count() - n0
    ms = torch.tensor([e0.elapsed_time(e1)], device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    # end to end: host f in (each rank copies its band), gathered host u out
    e2e = []
    for _ in range(3):
        dist.barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        import time as _t
        w0 = _t.perf_counter()
        fb = backend.tensor(f[plan.begin: plan.end])
        u, _ = run(fb, args.steps, True)
        u.cpu()
        dt = torch.tensor([_t.perf_counter() - w0], device=dev)
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        e2e.append(float(dt.item()))
    # K1 direct sum on this rank's band rows (the north-star kernel matvec:
    # compute-bound, N^2 / G pairs per rank): aggregate pair-evals/s
    from .toeplitz import KernelMatvec
    k1 = KernelMatvec(op, method="direct")
    Xk = torch.from_numpy(np.random.default_rng(9).standard_normal((2, op.n))).to(dev)
    Yk = torch.empty(2, max(plan.size, 1), dtype=torch.float64, device=dev)
    k1.matvec_device(Xk, Yk, nrhs=2, row_begin=plan.begin, row_end=plan.end, ldy=Yk.shape[1])
    torch.cuda.synchronize()
    dist.barrier()
    e0.record(st)
    k1.matvec_device(Xk, Yk, nrhs=2, row_begin=plan.begin, row_end=plan.end, ldy=Yk.shape[1])
    e1.record(st)
    torch.cuda.synchronize()
    k1_ms = torch.tensor([e0.elapsed_time(e1)], device=dev)
    dist.all_reduce(k1_ms, op=dist.ReduceOp.MAX)
    k1_ms = float(k1_ms.item())
    if rank == 0:
        clk = clocks.stop()
        out = {"metric": metric, "value": args.steps / (ms * 1e-3), "unit": "iter/s", "n_gpus": ws,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
               "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
               "data": "synthetic (BASELINE.json config 5, seeded)",
               "config": {"workload": workload, "N": op.n, "parallelism": f"row/subdomain bands x{ws} (NCCL)",
                          "driver": "native ie_pcg_sharded_f64" if native else "python solve_sharded",
                          "matvec": backend.method, "bands": list(plan.bounds),
                          "l2": "not flushed"},
               "n_it": rep.n_it,
               "e2e": {"value": args.steps / statistics.median(e2e), "unit": "iter/s",
                       "h2d_bytes_per_step": 8 * plan.size / args.steps,
                       "d2h_bytes_per_step": 8 * op.n / args.steps,
                       "note": "per solve of K steps: H2D of each rank's f band, D2H of the gathered u"},
               "gpu_launches": launches, "clocks": clk,
               "kernel_matvec": {"kernel": "k_matvec<2,2,2> on each rank's band rows (sources all-gathered)",
                                 "pass_ms": k1_ms, "pair_evals_per_s": float(op.n) ** 2 / (k1_ms * 1e-3),
                                 "note": "max over ranks of one 2-RHS pass; N^2 pairs in total"},
               "roofline": {"bound": "n/a", "note": "see the N=1 line for the kernel rooflines"}}
        print(json.dumps(out))
    return None
