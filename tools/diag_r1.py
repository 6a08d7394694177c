"""Diagnostics: (1) K1/K1b row accuracy at config 3 against an
extended-precision (np.longdouble) direct sum for sampled rows; (2) solve()
timing split (device tensors vs numpy in/out)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_12574_b200 as ie  # noqa: E402
from oracle import iedd_oracle as O  # noqa: E402

n = 256
op = ie.build_operator(ie.build_grid(2, n), lattice="cell")
x = np.random.default_rng(1).standard_normal(op.n)
yd = ie.KernelMatvec(op, method="direct").matvec(x)
yf = ie.KernelMatvec(op, method="fft").matvec(x)
oop = O.build_operator(O.build_grid(2, n), "cell")
yo = O.FFTMatvec(oop).matvec(x)
mi = oop.grid.multi_indices().astype(np.longdouble)
h = np.longdouble(1) / n
xl = x.astype(np.longdouble)
rows = np.random.default_rng(0).choice(op.n, 24, replace=False)
err = {"direct": [], "fft": [], "oracle_fft": []}
for i in rows:
    d2 = ((mi - mi[i]) ** 2).sum(axis=1) * h * h
    d2[i] = 1
    k = -(h * h) * np.log(d2) / (4 * np.pi)   # -(h^2/2pi) log d
    k[i] = np.longdouble(op.diag_value)
    yr = (k * xl).sum()
    for name, y in (("direct", yd), ("fft", yf), ("oracle_fft", yo)):
        err[name].append(float(abs(np.longdouble(y[i]) - yr) / abs(yr)))
for name, e in err.items():
    print(f"row rel err {name:10s}: median {np.median(e):.2e}  max {np.max(e):.2e}")
print("||direct-fft||/||fft|| =", np.linalg.norm(yd - yf) / np.linalg.norm(yf))
print("||direct-oracle||/||.|| =", np.linalg.norm(yd - yo) / np.linalg.norm(yo),
      " ||fft-oracle|| =", np.linalg.norm(yf - yo) / np.linalg.norm(yo))

# timing split at config 5
grid = ie.build_grid(2, 1024)
op5 = ie.build_operator(grid, lattice="cell")
mv = ie.ToeplitzMatvec(op5)
pre = ie.from_decomposition(op5, ie.build_decomposition(grid, 128, 2, "schwarz"))
f = np.random.default_rng(3).standard_normal(op5.n)
fd = torch.from_numpy(f).cuda()
for K in (10, 10, 50):
    torch.cuda.synchronize(); t = time.perf_counter(); u, rep = ie.solve(mv, pre, fd, tol=1e-10, max_iters=K)
    torch.cuda.synchronize(); t1 = time.perf_counter() - t
    t = time.perf_counter(); u, rep = ie.solve(mv, pre, f, tol=1e-10, max_iters=K); t2 = time.perf_counter() - t
    print(f"K={K}: device-f solve {1e3*t1:.2f} ms ({1e3*t1/K:.3f} ms/it, t_pcg {1e3*rep.t_pcg:.2f}), numpy-f solve {1e3*t2:.2f} ms")
t = time.perf_counter(); a = torch.from_numpy(f).cuda(); torch.cuda.synchronize(); t3 = time.perf_counter() - t
t = time.perf_counter(); b = a.cpu().numpy(); t4 = time.perf_counter() - t
print(f"H2D 8MB {1e3*t3:.2f} ms, D2H 8MB {1e3*t4:.2f} ms")
X = torch.from_numpy(np.random.default_rng(9).standard_normal((2, op5.n))).cuda(); Y = torch.empty_like(X)
r = X[0].clone(); z = torch.empty_like(r)
for name, fn in (("fft 2rhs", lambda: mv.matvec_device(X, Y, nrhs=2)), ("fft 1rhs", lambda: mv.matvec_device(X[0], Y[0])),
                 ("apply", lambda: pre.apply_device(r, z))):
    fn(); torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(20): fn()
    torch.cuda.synchronize(); print(f"{name}: {1e3*(time.perf_counter()-t)/20:.3f} ms (host timed)")
