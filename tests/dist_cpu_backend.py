"""CPU backend for the sharded-driver tests (test infrastructure): the same
interface as distributed.CudaBackend, computed with the oracle on torch CPU
tensors so the driver's plan / gather / ordering logic runs over gloo."""

import numpy as np
import torch

from oracle import iedd_oracle as O
from paper_2108_12574_b200.distributed import CHUNK, BandFFT


class NumpyBandStages:
    """The four band passes of BandFFT in numpy (pocketfft per line), on the
    same buffer layouts as the CUDA passes (complex as interleaved float64)."""

    def __init__(self, op, plan):
        self.plan = plan
        from paper_2108_12574_b200.toeplitz import fft_size
        n = op.grid.n_per_dim
        self.n, self.M = n, fft_size(n)
        M = self.M
        emb = np.zeros((M, M))
        emb[:n, :n] = op.generator()
        emb[M - n + 1:, :] = emb[n - 1:0:-1, :]
        emb[:, M - n + 1:] = emb[:, n - 1:0:-1]
        self.sym = np.fft.fft2(emb).real

    def band_fwd(self, Xb, nrows, parts, scales):
        x = Xb.numpy().reshape(Xb.shape[0], nrows, self.n)
        z = x[0].astype(complex)
        if Xb.shape[0] == 2:
            s0, s1 = scales
            z = x[0] * s0 + 1j * (x[1] * s1)
        f = np.fft.fft(z, n=self.M, axis=1)                      # (nrows, M)
        out = f.reshape(nrows, parts, self.M // parts).transpose(1, 0, 2)
        return torch.from_numpy(np.ascontiguousarray(out).view(np.float64).reshape(-1).copy())

    def band_cols(self, buf, c0, ncols):
        b = buf.numpy().view(complex).reshape(self.n, ncols)
        f = np.fft.fft(b, n=self.M, axis=0) * self.sym[:, c0:c0 + ncols]
        b[:] = np.fft.ifft(f, axis=0)[: self.n]

    def band_inv(self, buf, nrows, parts, ncol, scales):
        b = buf.numpy().view(complex).reshape(parts, nrows, self.M // parts).transpose(1, 0, 2)
        y = np.fft.ifft(b.reshape(nrows, self.M), axis=1)[:, : self.n].reshape(-1)
        if ncol == 2:
            s0, s1 = scales
            return torch.from_numpy(np.stack([y.real / s0, y.imag / s1]))
        return torch.from_numpy(y.real[None].copy())


class OracleBackend:
    def __init__(self, dim, n, m, w, kind, lattice, plan, dist_fft=False):
        self.plan = plan
        grid = O.build_grid(dim, n)
        self.op = O.build_operator(grid, lattice)
        self.mv = O.FFTMatvec(self.op)
        self.band = (BandFFT(NumpyBandStages(self.op, plan), plan, n)
                     if dist_fft and BandFFT.supported(grid, plan) else None)
        dec = O.build_decomposition(grid, m, w, kind)
        sub = O.Decomposition(kind, grid, m, w, [dec.subdomains[k] for k in plan.blocks])
        self.pre = O.SchwarzPrecond(self.op, sub) if plan.blocks.size else None
        self.N = self.op.n

    def tensor(self, a):
        return torch.as_tensor(np.asarray(a, dtype=np.float64))

    def zeros(self, n):
        return torch.zeros(n, dtype=torch.float64)

    def matvec_band(self, X):
        Y = np.stack([self.mv.matvec(X[c].numpy())[self.plan.begin: self.plan.end] for c in range(X.shape[0])])
        return torch.from_numpy(Y)

    def matvec_cols(self, comm, Xb, scales=None):
        if self.band is not None:
            return self.band.matvec(comm, Xb.contiguous(), scales)
        return self.matvec_band(comm.allgather_band(Xb))

    def chunk_max(self, x):
        xa = np.abs(x.numpy())
        return torch.tensor([float(xa[c: c + CHUNK].max()) for c in range(0, xa.size, CHUNK)],
                            dtype=torch.float64)

    def apply_band(self, r_full):
        if self.pre is None:
            return self.zeros(0)
        return torch.from_numpy(self.pre.apply(r_full.numpy())[self.plan.begin: self.plan.end].copy())

    def dot_partials(self, x, y, mode):
        xa, ya = x.numpy(), y.numpy()
        out = []
        for c0 in range(0, xa.size, CHUNK):
            a, b = xa[c0: c0 + CHUNK], ya[c0: c0 + CHUNK]
            out.append(float(a @ b) if mode == 0 else float((a - b) @ (a - b)))
        return torch.tensor(out, dtype=torch.float64)

    def sum_partials(self, parts):
        s = 0.0
        for v in parts.tolist():
            s += v
        return s

    def update(self, op, a, b, s):
        if op == 0:
            a += s * b
        elif op == 1:
            a -= s * b
        else:
            a.copy_(b + s * a)

    def sync(self):
        pass
