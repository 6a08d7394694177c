"""Run 10 config-5 PCG iterations (after warm-up) for an ncu launch list."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_12574_b200 as ie  # noqa: E402

grid = ie.build_grid(2, 1024)
op = ie.build_operator(grid, lattice="cell")
mv = ie.ToeplitzMatvec(op)
pre = ie.from_decomposition(op, ie.build_decomposition(grid, 128, 2, "schwarz"))
f = torch.from_numpy(np.random.default_rng(3).standard_normal(op.n)).cuda()
ie.solve(mv, pre, f, tol=1e-10, max_iters=3)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
u, rep = ie.solve(mv, pre, f, tol=1e-10, max_iters=10)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print("done", rep.n_it)
