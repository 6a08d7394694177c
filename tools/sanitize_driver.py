"""Small workload for compute-sanitizer (racecheck / synccheck / memcheck):
every kernel family of the hot path at config-3 size (2D n=256, Schwarz
w=2) -- the FFT passes incl. the fused PCG modes and the TMA column pass, the
DMMA class apply + scatter with its decider tail, the vector kernels, a few
graph-replayed iterations, the packed apply without sharing, a large-block
sweep build, Lanczos steps, and the native sharded driver with two ranks on
the one device (pushes and mailbox waits).

  compute-sanitizer --tool racecheck python tools/sanitize_driver.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_12574_b200 as ie  # noqa: E402
from paper_2108_12574_b200 import distributed as D  # noqa: E402

grid = ie.build_grid(2, 256)
op = ie.build_operator(grid, lattice="cell")
dec = ie.build_decomposition(grid, 32, 2, "schwarz")
f = np.random.default_rng(1).standard_normal(op.n)
mv = ie.ToeplitzMatvec(op)
pre = ie.from_decomposition(op, dec)
u, rep = ie.solve(mv, pre, f, tol=1e-10, max_iters=6)
print("pcg fft/shared", rep.n_it, rep.residual_history[-1])
u, rep = ie.solve(ie.KernelMatvec(op, method="direct"), ie.from_decomposition(op, dec, share_translated=False),
                  f, tol=1e-10, max_iters=3)
print("pcg direct/unshared", rep.n_it)
big = ie.from_decomposition(ie.build_operator(ie.build_grid(2, 32)), ie.build_decomposition(ie.build_grid(2, 32), 2, 1,
                                                                                            "schwarz"))
print("sweep build", big.stats()["S"])
small = ie.build_grid(2, 32)
sop = ie.build_operator(small)
lam = ie.extremal_eigenvalue_lanczos(ie.ToeplitzMatvec(sop), ie.from_decomposition(sop, ie.build_decomposition(small, 4, 1,
                                                                                                              "schwarz")),
                                     sop.n, which="max", max_iters=20)
print("lanczos", lam)
u2, rep2 = D.LocalShards(op, dec, 2).solve(f, tol=1e-10, max_iters=4)
print("sharded G=2", rep2.n_it)
