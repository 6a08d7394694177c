import os, sys, time
import torch
sys.path.insert(0, "/root/repo")
import paper_2108_12574_b200 as ie
grid = ie.build_grid(2, 64); op = ie.build_operator(grid, lattice="cell")
mv = ie.ToeplitzMatvec(op)
for kind in ("schwarz", "jacobi"):
    pre = ie.from_decomposition(op, ie.build_decomposition(grid, 8, 1, kind))
    for which in ("min", "max"):
        ts = []
        for rep in range(4):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            lam, st = ie.extremal_eigenvalue_lanczos(mv, pre, op.n, which=which, max_iters=300, return_steps=True)
            torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
        print(kind, which, st, ["%.2f" % (1e3 * t) for t in ts])
