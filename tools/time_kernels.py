"""Device-event timing of the hot kernels at config 5 (and FFT at configs 3/4)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_12574_b200 as ie  # noqa: E402


def t(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for dim, n in ((2, 1024), (2, 256), (3, 32)):
    op = ie.build_operator(ie.build_grid(dim, n), lattice="cell")
    mv = ie.KernelMatvec(op, method="fft")
    X = torch.from_numpy(np.random.default_rng(0).standard_normal((2, op.n))).cuda()
    Y = torch.empty_like(X)
    print(f"fft {dim}D n={n}: 2-RHS {t(lambda: mv.matvec_device(X, Y, nrhs=2)):.4f} ms, "
          f"1-RHS {t(lambda: mv.matvec_device(X[0], Y[0])):.4f} ms")
grid = ie.build_grid(2, 1024)
op = ie.build_operator(grid, lattice="cell")
dec = ie.build_decomposition(grid, 128, 2, "schwarz")
pre = ie.from_decomposition(op, dec)
r = torch.from_numpy(np.random.default_rng(1).standard_normal(op.n)).cuda()
z = torch.empty_like(r)
print(f"apply c5 shared (gemm): {t(lambda: pre.apply_device(r, z), 50):.4f} ms")
mv = ie.ToeplitzMatvec(op)
f = torch.from_numpy(np.random.default_rng(3).standard_normal(op.n)).cuda()
ie.solve(mv, pre, f, tol=1e-10, max_iters=3)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
u, rep = ie.solve(mv, pre, f, tol=1e-10, max_iters=20)
e1.record()
torch.cuda.synchronize()
print(f"pcg c5: {e0.elapsed_time(e1) / 20:.4f} ms/iteration ({rep.n_it} it)")
for name, cfg in (("c2", (2, 64, 8, 1)),):
    dim, n, m, w = cfg
    g = ie.build_grid(dim, n)
    o = ie.build_operator(g, lattice="cell")
    p = ie.from_decomposition(o, ie.build_decomposition(g, m, w, "schwarz"))
    import time
    mvv = ie.ToeplitzMatvec(o)
    t0 = time.perf_counter()
    lam, steps = ie.extremal_eigenvalue_lanczos(mvv, p, o.n, which="min", max_iters=300, return_steps=True)
    print(f"lanczos {name} min: {1e3*(time.perf_counter()-t0):.1f} ms, {steps} steps, lambda {lam}")
