import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import numpy as np
import paper_2108_12574_b200 as ie
n = 32
grid = ie.build_grid(2, n); op = ie.build_operator(grid, lattice="cell")
mv = ie.KernelMatvec(op, method="fft")
pre = ie.from_decomposition(op, ie.build_decomposition(grid, 4, 1, "schwarz"))
f = np.random.default_rng(0).standard_normal(op.n)
z0 = pre.apply(f)
print("max|z0|", np.abs(z0).max(), "rz0", f @ z0)
try:
    u, rep = ie.solve(mv, pre, f, tol=1e-10, max_iters=3)
    print(rep.residual_history)
except Exception as e:
    print("ERR", e)
