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


def pow2_scale(mx: float) -> float:
    """2^-e with 2^e > mx >= 2^(e-1) (C frexp), 1.0 for 0 / non-finite: the
    exact power-of-two column multiplier of the 2-RHS FFT packing
    (pcg_pow2_scale in csrc/pcg_state.cuh)."""
    if not (mx > 0.0) or not math.isfinite(mx):
        return 1.0
    return math.ldexp(1.0, -math.frexp(mx)[1])


def pcg_scales(max_z: float, beta: float, max_p_old: float, max_u: float) -> tuple:
    """The 2-RHS multipliers [p_new, u] of the next A-pass, the rule k_iter_b
    applies on the device: max|p_new| <= max|z| + |beta| max|p_old| (products
    rounded as written), so no rank needs max|p_new| before its row
    transforms.  All inputs are global maxima (exact; order-independent)."""
    return pow2_scale(max_z + abs(beta) * max_p_old), pow2_scale(max_u)


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
    for CPU tensors).  Bands are padded to the longest one.  host_staged:
    device tensors go through host copies (gloo between processes that share
    one GPU, where NCCL cannot run)."""

    def __init__(self, plan: ShardPlan, group=None, host_staged: bool = False):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.plan = plan
        self.host_staged = host_staged
        self.maxlen = max(plan.bounds[i + 1] - plan.bounds[i] for i in range(plan.world))
        self.maxch = max(plan.chunks(i)[1] - plan.chunks(i)[0] for i in range(plan.world))

    def _gather(self, x, length_of):
        import torch
        world = self.plan.world
        ncol, L = x.shape
        pad = self.maxlen if length_of == "band" else self.maxch
        buf = x.new_zeros((ncol, pad))
        buf[:, :L] = x
        dev = buf.device
        if self.host_staged and world > 1:
            buf = buf.cpu()
        outs = [torch.empty_like(buf) for _ in range(world)]
        if world == 1:
            outs[0].copy_(buf)
        else:
            self.dist.all_gather(outs, buf, group=self.group)
        outs = [o.to(dev) for o in outs]
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
        elif self.host_staged:  # gloo has no all_to_all: pairwise exchanges on host copies
            src = send.contiguous().cpu()
            so = np.concatenate([[0], np.cumsum(send_counts)]).astype(int)
            ro = np.concatenate([[0], np.cumsum(recv_counts)]).astype(int)
            host = src.new_empty(int(ro[-1]))
            me = self.plan.rank
            host[ro[me]: ro[me + 1]] = src[so[me]: so[me + 1]]
            ops = []
            for h in range(self.plan.world):
                if h == me:
                    continue
                if send_counts[h]:
                    ops.append(self.dist.P2POp(self.dist.isend, src[so[h]: so[h + 1]].clone(), h, group=self.group))
                if recv_counts[h]:
                    ops.append(self.dist.P2POp(self.dist.irecv, host[ro[h]: ro[h + 1]], h, group=self.group))
            if ops:
                for req in self.dist.batch_isend_irecv(ops):
                    req.wait()
            out.copy_(host)
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

    def allgather_var(self, x, counts):
        """(ncol, counts[rank]) -> (ncol, sum(counts)) in rank order."""
        import torch
        world = self.plan.world
        ncol, L = x.shape
        pad = max(counts)
        buf = x.new_zeros((ncol, pad))
        buf[:, :L] = x
        dev = buf.device
        if self.host_staged and world > 1:
            buf = buf.cpu()
        outs = [torch.empty_like(buf) for _ in range(world)]
        if world == 1:
            outs[0].copy_(buf)
        else:
            self.dist.all_gather(outs, buf, group=self.group)
        return torch.cat([outs[r][:, :counts[r]].to(dev) for r in range(world)], dim=1)

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

    With two right-hand sides the exact power-of-two column multipliers come
    from the caller (pcg_scales: global quantities), so every rank scales
    identically.  The per-line arithmetic is that of the single-GPU pass
    (same kernels, same data), so the result does not depend on G.  Per
    iteration and rank this moves 2 x 16 * n * (2n) / G bytes instead of
    all-gathering [p, u]."""

    def __init__(self, stages, plan: ShardPlan, n: int):
        self.st = stages
        self.plan = plan
        self.n = n
        self.G = plan.world
        from .toeplitz import fft_size
        self.M = fft_size(n)
        self.Mc = self.M // self.G
        self.rows = [((plan.bounds[h + 1] - plan.bounds[h]) // n) for h in range(self.G)]
        self.row0 = sum(self.rows[: plan.rank])

    @staticmethod
    def supported(grid, plan: ShardPlan) -> bool:
        from .toeplitz import fft_size
        n, G = grid.n_per_dim, plan.world
        M = fft_size(n)
        return (grid.dim == 2 and M % G == 0 and (M // G) & (M // G - 1) == 0
                and all(b % n == 0 for b in plan.bounds))

    def matvec(self, comm, Xb, scales=None):
        """Xb: (ncol, band) -> (ncol, band) = rows [begin, end) of A x.  Two
        columns need `scales` (the 2-RHS multipliers, pcg_scales)."""
        ncol = Xb.shape[0]
        if ncol == 2 and scales is None:
            raise ValueError("BandFFT.matvec: two columns need the 2-RHS scales (pcg_scales)")
        g, G, Mc = self.plan.rank, self.G, self.Mc
        mine = self.rows[g]
        sc = scales if ncol == 2 else None
        b1 = self.st.band_fwd(Xb, mine, G, sc)                            # (G, mine, Mc) complex
        b2 = comm.alltoall(b1, [2 * mine * Mc] * G, [2 * r * Mc for r in self.rows])
        self.st.band_cols(b2, g * Mc, Mc)                                 # (n, Mc) complex
        b3 = comm.alltoall(b2, [2 * r * Mc for r in self.rows], [2 * mine * Mc] * G)
        return self.st.band_inv(b3, mine, G, ncol, sc)


class CudaBandStages:
    """The band passes through the C-ABI (ie_matvec_band_*)."""

    def __init__(self, mv, plan: ShardPlan):
        import torch

        from . import _lib
        self.torch, self._lib, self.L = torch, _lib, _lib.lib()
        self.mv, self.plan = mv, plan
        self.namax = -(-plan.N // CHUNK)

    def _sc(self, scales, dev):
        return None if scales is None else self.torch.tensor(list(scales), dtype=self.torch.float64, device=dev)

    def band_fwd(self, Xb, nrows, parts, scales):
        out = self.torch.empty(nrows * self.mv.M * 2, dtype=self.torch.float64, device=Xb.device)
        sc = self._sc(scales, Xb.device)
        self._lib.check(self.L.ie_matvec_band_fwd_f64(
            self.mv.handle, self._lib.ptr(Xb), Xb.stride(0), Xb.shape[0], self.plan.begin, self.plan.end, parts,
            self._lib.ptr(out), self._lib.ptr(sc) if sc is not None else None, self._lib.stream_ptr()), "band_fwd")
        return out

    def band_cols(self, buf, c0, ncols):
        self._lib.check(self.L.ie_matvec_band_cols_f64(self.mv.handle, self._lib.ptr(buf), c0, c0 + ncols,
                                                       self._lib.stream_ptr()), "band_cols")

    def band_inv(self, buf, nrows, parts, ncol, scales):
        Y = self.torch.empty(ncol, self.plan.size, dtype=self.torch.float64, device=buf.device)
        sc = self._sc(scales, buf.device)
        self._lib.check(self.L.ie_matvec_band_inv_f64(
            self.mv.handle, self._lib.ptr(buf), self.plan.begin, self.plan.end, parts, self._lib.ptr(Y),
            self.plan.size, ncol, self._lib.ptr(sc) if sc is not None else None, self._lib.stream_ptr()),
            "band_inv")
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
            method = "fft" if fft_supported(op.grid.n_per_dim, op.grid.dim) else "direct"
        self.mv = KernelMatvec(op, method=method)
        self.method = method
        self.band = (BandFFT(CudaBandStages(self.mv, plan), plan, op.grid.n_per_dim)
                     if method == "fft" and BandFFT.supported(op.grid, plan) and not dist_fft_disabled() else None)
        sub = SubDecomposition(decomposition.kind, [decomposition.subdomains[k] for k in plan.blocks],
                               plan.blocks)
        self.pre = (from_decomposition(op, sub, variant=variant, share_translated=share_translated)
                    if plan.blocks.size else None)
        self.dev = torch.device("cuda", torch.cuda.current_device())
        # dot products of the A-pass per grid line (n points along the last
        # axis) with the association ie_pcg_f64 uses when the post pass rides
        # in the FFT's last line transform -- bitwise the single-GPU values;
        # needs every band cut on a line boundary
        import os
        n = op.grid.n_per_dim
        self.line_post = (method == "fft" and op.grid.dim >= 2 and self.mv.M >= 64
                          and not os.environ.get("IEDD_B200_NO_FUSE") and not os.environ.get("IEDD_B200_NO_FUSE_POST")
                          and all(b % n == 0 for b in plan.bounds))
        self.line_len = n
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

    def matvec_cols(self, comm, Xb, scales=None):
        """Band columns in, band rows of A x out (distributed FFT, or
        all-gather + the band rows of the full-range pass)."""
        if self.band is not None:
            return self.band.matvec(comm, Xb.contiguous(), scales)
        return self.matvec_band(comm.allgather_band(Xb))

    def chunk_max(self, x):
        """Per-2048-chunk max|x| of a band vector."""
        n = x.numel()
        out = self.torch.empty(max(1, -(-n // CHUNK)), 2, dtype=self.torch.float64, device=self.dev)
        if n:
            self._lib.check(self.L.ie_absmax_partials_f64(self._lib.ptr(x), 0, n, self._lib.ptr(out),
                                                          self._lib.stream_ptr()), "absmax")
        return out[: -(-n // CHUNK), 0].contiguous() if n else out[:0, 0]

    def apply_band(self, r_full):
        if self.pre is None:
            return self.zeros(0)
        z = self._full[0]
        self.pre.apply_device(r_full.contiguous(), z)
        return z[self.plan.begin: self.plan.end].clone()

    def post_partials(self, p, q, f, w, do_p: bool, pending: bool):
        """The A-pass partials [p.q if do_p, |f - w|^2 if pending] of the band:
        per grid line (line_post) or per dot chunk."""
        if not self.line_post:
            rows = ([self.dot_partials(p, q, 0)] if do_p else []) + ([self.dot_partials(f, w, 1)] if pending else [])
            return _stack(rows)
        n = self.line_len
        nl = self.plan.size // n
        out = self.torch.empty(int(do_p) + int(pending), max(nl, 1), dtype=self.torch.float64, device=self.dev)
        row = 0
        for on, (x, y, mode) in ((do_p, (p, q, 0)), (pending, (f, w, 1))):
            if on:
                if nl:
                    self._lib.check(self.L.ie_line_partials_f64(self._lib.ptr(x), self._lib.ptr(y), nl, n, self.mv.M,
                                                                mode, self._lib.ptr(out[row]), self._lib.stream_ptr()),
                                    "line partials")
                row += 1
        return out[:, :nl]

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

    def gmax(x):  # global max|x| (exact: the maximum does not depend on the order)
        return float(comm.allgather_partials(backend.chunk_max(x)[None])[0].max().item())

    r = f_band.clone()
    z = apply(r)
    p = z.clone()
    max_p = gmax(p)
    scales = None
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
        Y = backend.matvec_cols(comm, _stack(cols), scales if len(cols) == 2 else None)
        q = Y[0] if do_p else None
        w = Y[-1] if pending else None
        if hasattr(backend, "post_partials"):
            parts = backend.post_partials(p, q, f_band, w, do_p, pending)
        else:
            parts = _stack(([backend.dot_partials(p, q, 0)] if do_p else []) +
                           ([backend.dot_partials(f_band, w, 1)] if pending else []))
        if getattr(backend, "line_post", False):
            G = comm.allgather_var(parts, [(plan.bounds[r + 1] - plan.bounds[r]) // backend.line_len
                                           for r in range(plan.world)])
        else:
            G = comm.allgather_partials(parts)
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
            scales = pcg_scales(gmax(z), beta, max_p, gmax(u))
            backend.update(2, p, z, beta)
            max_p = gmax(p)
    full = comm.allgather_band(u[None])[0] if gather_solution else u
    rep = ShardedReport(n_it=k, achieved_residual=hist[-1], t_pcg=time.perf_counter() - t0,
                        t_s=t_prec / max(n_prec, 1), residual_history=hist, stagnated=stag, converged=conv)
    return full, rep


class NativeShard:
    """This rank's part of the native sharded solver (ie_pcg_sharded_f64):
    the exchange heap every peer stores into over NVLink.  Multi-process:
    the CUDA IPC handles travel by torch.distributed all_gather_object, then
    every rank opens its peers' heaps (ie_shard_connect)."""

    def __init__(self, backend, plan: ShardPlan, group=None, connect: bool = True):
        from . import _lib
        self._lib = _lib
        self.L = _lib.lib()
        self.plan = plan
        self.backend = backend
        bounds = np.ascontiguousarray(plan.bounds, dtype=np.int64)
        need = np.ascontiguousarray(np.array(plan.need, dtype=np.int64).reshape(-1)) if plan.need else None
        th = backend.pre.handle if backend.pre is not None else None
        h = ctypes.c_void_p()
        _lib.check(self.L.ie_shard_create(backend.mv.handle, th, plan.world, plan.rank, _lib.np_ptr(bounds),
                                          _lib.np_ptr(need) if need is not None else None, ctypes.byref(h)),
                   "ie_shard_create")
        self.handle = h
        rows = np.zeros(2, dtype=np.int64)
        _lib.check(self.L.ie_shard_need_rows(h, _lib.np_ptr(rows)), "ie_shard_need_rows")
        self.need_lo, self.need_hi = int(rows[0]), int(rows[1])
        if connect and plan.world > 1:
            import torch.distributed as dist
            nb = int(self.L.ie_shard_handle_bytes())
            buf = ctypes.create_string_buffer(nb)
            _lib.check(self.L.ie_shard_export(h, buf), "ie_shard_export")
            blobs = [None] * plan.world
            dist.all_gather_object(blobs, buf.raw, group=group)
            allb = ctypes.create_string_buffer(b"".join(blobs), nb * plan.world)
            _lib.check(self.L.ie_shard_connect(h, allb), "ie_shard_connect")

    def __del__(self):
        h = getattr(self, "handle", None)
        if h is not None and h.value:
            self._lib.lib().ie_shard_destroy(h)
            self.handle = None


def native_supported(backend, plan: ShardPlan) -> bool:
    """ie_pcg_sharded_f64's domain: the band FFT and equal, chunk-aligned bands."""
    sizes = {plan.bounds[h + 1] - plan.bounds[h] for h in range(plan.world)}
    return backend.band is not None and len(sizes) == 1 and all(b % CHUNK == 0 for b in plan.bounds)


def _report(hist, n_it, flags, times):
    k = n_it.value
    h = [float(x) for x in hist[: k + 1]]
    return ShardedReport(n_it=k, achieved_residual=h[-1], t_pcg=float(times[0]), t_s=float(times[1]),
                         residual_history=h, stagnated=bool(flags[1]), converged=bool(flags[0]))


def _raise_pcg(_lib, rc, fail_it, fail_val, what):
    if rc == _lib.IE_ERR_BREAKDOWN:
        raise FloatingPointError(f"PCG breakdown at iteration {fail_it.value}: p^T A p = {fail_val.value}")
    if rc == _lib.IE_ERR_NONFINITE:
        raise FloatingPointError(f"non-finite residual at iteration {fail_it.value}")
    _lib.check(rc, what)


def solve_sharded_native(shard: NativeShard, f_need, tol: float = 1e-12, max_iters: int | None = None):
    """pcg.solve on the band decomposition through the native driver
    (ie_pcg_sharded_f64; every rank calls it).  f_need = f on the rank's need
    rows [shard.need_lo, shard.need_hi).  Returns (u_band, ShardedReport)."""
    from . import _lib
    if not 0.0 < tol < 1.0:
        raise ValueError(f"tol must be in (0, 1), got {tol}")
    plan = shard.plan
    if max_iters is None:
        max_iters = max(2 * plan.N, 100)
    u = shard.backend.zeros(plan.size)
    hist = np.zeros(max_iters + 2, dtype=np.float64)
    n_it, fail_it, fail_val = ctypes.c_int64(0), ctypes.c_int64(0), ctypes.c_double(0.0)
    flags = np.zeros(2, dtype=np.int32)
    times = np.zeros(2, dtype=np.float64)
    f_need = f_need.contiguous()
    if f_need.numel() != shard.need_hi - shard.need_lo:
        raise ValueError(f"f_need has length {f_need.numel()}, the need rows hold {shard.need_hi - shard.need_lo}")
    rc = _lib.lib().ie_pcg_sharded_f64(shard.handle, _lib.ptr(f_need), _lib.ptr(u), tol, max_iters,
                                       _lib.np_ptr(hist), ctypes.byref(n_it), _lib.np_ptr(flags), _lib.np_ptr(times),
                                       ctypes.byref(fail_it), ctypes.byref(fail_val), _lib.stream_ptr())
    _raise_pcg(_lib, rc, fail_it, fail_val, "ie_pcg_sharded_f64")
    return u, _report(hist, n_it, flags, times)


class LocalShards:
    """All G ranks of the native sharded solver inside one process on one
    device (ie_pcg_sharded_local_f64): the peers are plain device pointers
    and every exchange phase runs for all ranks before the next starts.  It
    runs the multi-GPU code path -- plans, halo rows, pushes, mailbox
    counters, the captured iteration -- on a single GPU, so the G > 1 paths
    are testable (tests/test_gpu_parity.py::TestShardedP2P)."""

    def __init__(self, op, decomposition, world: int, method: str = "fft", variant: str = "packed_inverse",
                 share_translated: bool = True, identity: bool = False):
        from . import _lib
        self._lib = _lib
        self.L = _lib.lib()
        grid = op.grid
        self.world = world
        self.plans = [make_plan(grid, decomposition, world, g) for g in range(world)]
        self.backends = [CudaBackend(op, decomposition, pl, method=method, variant=variant,
                                     share_translated=share_translated) for pl in self.plans]
        if identity:  # precond=None (pcg.py:68): the identity on every rank, no halo
            for b in self.backends:
                b.pre = None
        if not all(native_supported(b, pl) for b, pl in zip(self.backends, self.plans)):
            raise ValueError("native sharded PCG needs the 2D band FFT and equal chunk-aligned bands")
        self.shards = [NativeShard(b, pl, connect=False) for b, pl in zip(self.backends, self.plans)]
        arr = (ctypes.c_void_p * world)(*[sh.handle.value for sh in self.shards])
        _lib.check(self.L.ie_shard_connect_local(arr, world), "ie_shard_connect_local")
        self._arr = arr

    def solve(self, f, tol: float = 1e-12, max_iters: int | None = None):
        """Full-length f (numpy or device tensor) -> (u (N,) device tensor, ShardedReport)."""
        torch = self.backends[0].torch
        dev = self.backends[0].dev
        f = torch.as_tensor(f, dtype=torch.float64).to(dev)
        if not 0.0 < tol < 1.0:
            raise ValueError(f"tol must be in (0, 1), got {tol}")
        N = self.plans[0].N
        if max_iters is None:
            max_iters = max(2 * N, 100)
        fs = [f[sh.need_lo: sh.need_hi].contiguous() for sh in self.shards]
        us = [torch.empty(pl.size, dtype=torch.float64, device=dev) for pl in self.plans]
        fp = (ctypes.c_void_p * self.world)(*[t.data_ptr() for t in fs])
        up = (ctypes.c_void_p * self.world)(*[t.data_ptr() for t in us])
        hist = np.zeros(max_iters + 2, dtype=np.float64)
        n_it, fail_it, fail_val = ctypes.c_int64(0), ctypes.c_int64(0), ctypes.c_double(0.0)
        flags = np.zeros(2, dtype=np.int32)
        times = np.zeros(2, dtype=np.float64)
        rc = self.L.ie_pcg_sharded_local_f64(self._arr, self.world, fp, up, tol, max_iters, self._lib.np_ptr(hist),
                                             ctypes.byref(n_it), self._lib.np_ptr(flags), self._lib.np_ptr(times),
                                             ctypes.byref(fail_it), ctypes.byref(fail_val), self._lib.stream_ptr())
        _raise_pcg(self._lib, rc, fail_it, fail_val, "ie_pcg_sharded_local_f64")
        return torch.cat(us), _report(hist, n_it, flags, times)


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
def _band_fft_flops(n: int, rows: int, need_rows: int, cols: int) -> float:
    """Conventional complex-FFT flops (5 M log2 M per line, M = the circulant
    size, 2n for power-of-two n) of one rank's 2-RHS band pass: `rows` forward
    row lines, `cols` column lines forward and inverse, `need_rows` inverse
    row lines."""
    from .toeplitz import fft_size
    M = fft_size(n)
    return (rows + 2 * cols + need_rows) * 5.0 * M * math.log2(M)


def bench_sharded(args, metric, cfg, workload, config_keys=None, cpu_baseline=None):
    """bench.py --gpus N under torchrun: config 5 on N ranks (bands of rows and
    subdomains) through the native P2P driver.  Before timing it checks itself:
    a 12-iteration solve on all ranks is compared BITWISE (history and the
    gathered u) against ie_pcg_f64 on rank 0's device.  Prints the contract
    JSON line on rank 0; time = max over ranks of the CUDA-event time of
    exactly `steps` iterations."""
    import json
    import os
    import statistics
    import time as _t

    import torch
    import torch.distributed as dist

    import paper_2108_12574_b200 as ie

    from . import _lib
    ws, rank = dist.get_world_size(), dist.get_rank()
    dev = torch.device("cuda", torch.cuda.current_device())
    st = torch.cuda.current_stream()
    grid = ie.build_grid(cfg["dim"], cfg["n"])
    op = ie.build_operator(grid, lattice="cell")
    dec = ie.build_decomposition(grid, cfg["m"], cfg["w"], "schwarz")
    plan = make_plan(grid, dec, ws, rank)
    backend = CudaBackend(op, dec, plan, method=getattr(args, "matvec", "auto"))
    comm = Comm(plan)
    f = np.random.default_rng(cfg["seed"]).standard_normal(op.n)
    native = native_supported(backend, plan) and not os.environ.get("IEDD_B200_PY_SHARDED")
    why = None
    shard = None
    if native:
        try:
            shard = NativeShard(backend, plan)
        except (RuntimeError, ValueError) as e:  # no P2P path between the GPUs
            native, why = False, str(e)
    ok = torch.tensor([1 if native else 0], device=dev)
    dist.all_reduce(ok, op=dist.ReduceOp.MIN)
    native = bool(ok.item())
    f_pin = torch.empty(op.n, dtype=torch.float64, pin_memory=True)
    f_pin.numpy()[:] = f
    if native:
        f_need = f_pin[shard.need_lo: shard.need_hi].to(dev)

        def run(iters):
            return solve_sharded_native(shard, f_need, tol=1e-10, max_iters=iters)
    else:
        f_band = f_pin[plan.begin: plan.end].to(dev)

        def run(iters):
            return solve_sharded(backend, comm, plan, f_band, tol=1e-10, max_iters=iters, gather_solution=False)

    # ---- self-check before timing: bitwise against the single-GPU solver
    pit = 12
    if native:
        # a native solve that fails at run time (peer mapping refused, a mailbox
        # wait timing out: status 6) must not take the job down: every rank
        # reports, and all fall back to the torch.distributed driver together
        try:
            u_b, rep_b = run(pit)
            okn = 1
        except RuntimeError as e:
            okn, why = 0, str(e)
        okt = torch.tensor([okn], device=dev)
        dist.all_reduce(okt, op=dist.ReduceOp.MIN)
        if not bool(okt.item()):
            native = False
            why = why or "native driver failed on another rank"
            f_band = f_pin[plan.begin: plan.end].to(dev)

            def run(iters):  # noqa: F811
                return solve_sharded(backend, comm, plan, f_band, tol=1e-10, max_iters=iters, gather_solution=False)
            u_b, rep_b = run(pit)
    else:
        u_b, rep_b = run(pit)
    u_all = comm.allgather_band(u_b[None])[0]
    parity = None
    if rank == 0:
        pre_full = ie.from_decomposition(op, dec)
        u1, rep1 = ie.solve(backend.mv, pre_full, torch.from_numpy(f).to(dev), tol=1e-10, max_iters=pit)
        parity = {"iterations": pit, "n_it": [rep_b.n_it, rep1.n_it],
                  "history_bitwise": rep_b.residual_history == rep1.residual_history,
                  "u_bitwise": bool(torch.equal(u_all, u1)),
                  "reference": "ie_pcg_f64 on rank 0's device (config 5, same f)"}
        parity["ok"] = parity["history_bitwise"] and parity["u_bitwise"] and rep_b.n_it == rep1.n_it
        del pre_full
    run(max(args.warmup, 1))
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
    _, rep = run(args.steps)
    e1.record(st)
    torch.cuda.synchronize()
    dist.barrier()
    launches = _lib.launch_count() - n0
    ms = torch.tensor([e0.elapsed_time(e1)], device=dev)
    dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    # end to end: each rank copies its rows of f from pinned host memory and
    # its band of u back to pinned host memory, inside the timed region
    u_host = torch.empty(plan.size, dtype=torch.float64, pin_memory=True)
    e2e = []
    for _ in range(3):
        dist.barrier()
        w0 = _t.perf_counter()
        if native:
            fn = f_pin[shard.need_lo: shard.need_hi].to(dev, non_blocking=True)
            u, _ = solve_sharded_native(shard, fn, tol=1e-10, max_iters=args.steps)
        else:
            fb = f_pin[plan.begin: plan.end].to(dev, non_blocking=True)
            u, _ = solve_sharded(backend, comm, plan, fb, tol=1e-10, max_iters=args.steps, gather_solution=False)
        u_host.copy_(u)
        dt = torch.tensor([_t.perf_counter() - w0], device=dev)
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        e2e.append(float(dt.item()))
    # dominant kernel: the rank's band FFT pass (row fwd, column fwd*sym*inv,
    # inverse need rows), timed on this stream without the exchanges
    n, G = cfg["n"], ws
    Mc = backend.mv.M // G
    rows = plan.size // n
    need_rows = (shard.need_hi - shard.need_lo) // n if native else rows
    X = torch.from_numpy(np.random.default_rng(9).standard_normal((2, plan.size))).to(dev)
    buf = torch.empty(max(rows, need_rows) * backend.mv.M * 2, dtype=torch.float64, device=dev)
    col = torch.empty(n * Mc * 2, dtype=torch.float64, device=dev)
    Yb = torch.empty(2, max(need_rows, rows) * n, dtype=torch.float64, device=dev)
    sc = torch.tensor([1.0, 1.0], dtype=torch.float64, device=dev)
    L = _lib.lib()

    def band_pass():
        _lib.check(L.ie_matvec_band_fwd_f64(backend.mv.handle, _lib.ptr(X), X.stride(0), 2, plan.begin, plan.end, G,
                                            _lib.ptr(buf), _lib.ptr(sc), _lib.stream_ptr()), "band_fwd")
        _lib.check(L.ie_matvec_band_cols_f64(backend.mv.handle, _lib.ptr(col), rank * Mc, rank * Mc + Mc,
                                             _lib.stream_ptr()), "band_cols")
        _lib.check(L.ie_matvec_band_inv_f64(backend.mv.handle, _lib.ptr(buf), 0, need_rows * n, G, _lib.ptr(Yb),
                                            Yb.stride(0), 2, _lib.ptr(sc), _lib.stream_ptr()), "band_inv")
    band_pass()
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(10):
        band_pass()
    e1.record(st)
    torch.cuda.synchronize()
    fft_ms = torch.tensor([e0.elapsed_time(e1) / 10], device=dev)
    dist.all_reduce(fft_ms, op=dist.ReduceOp.MAX)
    fft_ms = float(fft_ms.item())
    fl = torch.tensor([_band_fft_flops(n, rows, need_rows, Mc)], dtype=torch.float64, device=dev)
    dist.all_reduce(fl, op=dist.ReduceOp.SUM)
    peak = ctypes.c_double(0.0)
    _lib.check(L.ie_fp64_peak(ctypes.byref(peak), _lib.stream_ptr()), "fp64 peak")
    peak_tf = 2.0 * peak.value / 1e12 * ws
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
        config = dict(config_keys or {"workload": workload})
        config.update({"parallelism": f"row/subdomain bands x{ws}",
                       "driver": "native ie_pcg_sharded_f64 (NVLink P2P pushes)" if native
                       else f"python solve_sharded over torch.distributed ({why or 'forced'})",
                       "matvec": backend.method, "bands": list(plan.bounds)})
        achieved = float(fl.item()) / (fft_ms * 1e-3) / 1e12
        out = {"metric": metric, "value": args.steps / (ms * 1e-3), "unit": "iter/s", "n_gpus": ws,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
               "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
               "data": "synthetic (BASELINE.json config 5, seeded)", "config": config,
               "n_it": rep.n_it, "parity": parity,
               "exchange": ({"points_per_iteration": 4,
                             "bytes_out_per_rank_per_iteration": int(
                                 rows * backend.mv.M * 16                               # FWD: row spectra
                                 + need_rows * backend.mv.M * 16                        # BACK: need rows of the slab
                                 + ws * (rows * 16 + (plan.size // CHUNK) * 32)),       # POST, RZ slabs
                             "transport": "NVLink peer stores (CUDA IPC) + mailbox counters"}
                            if native else {"transport": "torch.distributed collectives"}),
               "e2e": {"value": args.steps / statistics.median(e2e), "unit": "iter/s",
                       "h2d_bytes_per_step": 8 * op.n / args.steps, "d2h_bytes_per_step": 8 * op.n / args.steps,
                       "note": "per solve of K steps: every rank's H2D of its f rows and D2H of its u band "
                               "(pinned), max over ranks of the wall time"},
               "gpu_launches": launches, "clocks": clk,
               "roofline": {"bound": "fp64", "kernel": "k_fft8 band passes (row fwd, column fwd*sym*inv, "
                                                       "inverse need rows), all ranks",
                            "achieved": achieved, "unit": "TFLOP/s", "peak": peak_tf,
                            "frac": achieved / peak_tf, "traffic": None,
                            "note": "flops = 5 M log2 M per line FFT summed over the ranks' lines; time = max "
                                    "over ranks of one band pass without its exchanges; peak = live DFMA "
                                    "microbenchmark x ranks"},
               "kernel_matvec": {"kernel": "k_matvec<2,2,16,ADJ> on each rank's band rows",
                                 "pass_ms": k1_ms, "pair_evals_per_s": float(op.n) ** 2 / (k1_ms * 1e-3),
                                 "note": "max over ranks of one 2-RHS pass; N^2 pairs in total"}}
        if cpu_baseline is not None:
            out["cpu_baseline"] = cpu_baseline()
        print(json.dumps(out))
    return None
