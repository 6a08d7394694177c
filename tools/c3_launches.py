"""Config-3 (2D n=256) Schwarz PCG for an ncu launch list."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_12574_b200 as ie  # noqa: E402

grid = ie.build_grid(2, 256)
op = ie.build_operator(grid, lattice="cell")
mv = ie.ToeplitzMatvec(op)
pre = ie.from_decomposition(op, ie.build_decomposition(grid, 32, 2, "schwarz"))
f = torch.from_numpy(np.random.default_rng(1).standard_normal(op.n)).cuda()
ie.solve(mv, pre, f, tol=1e-10, max_iters=5)
torch.cuda.synchronize()
u, rep = ie.solve(mv, pre, f, tol=1e-10, max_iters=12)
torch.cuda.synchronize()
print("done", rep.n_it)
