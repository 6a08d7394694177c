"""CPU backend for the sharded-driver tests (test infrastructure): the same
interface as distributed.CudaBackend, computed with the oracle on torch CPU
tensors so the driver's plan / gather / ordering logic runs over gloo."""

import numpy as np
import torch

from oracle import iedd_oracle as O
from paper_2108_12574_b200.distributed import CHUNK


class OracleBackend:
    def __init__(self, dim, n, m, w, kind, lattice, plan):
        self.plan = plan
        grid = O.build_grid(dim, n)
        self.op = O.build_operator(grid, lattice)
        self.mv = O.FFTMatvec(self.op)
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
