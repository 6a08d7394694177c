"""Config-2 Jacobi lambda_min Lanczos for an ncu launch list."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_12574_b200 as ie  # noqa: E402

grid = ie.build_grid(2, 64)
op = ie.build_operator(grid, lattice="cell")
pre = ie.from_decomposition(op, ie.build_decomposition(grid, 8, 1, "jacobi"))
mv = ie.ToeplitzMatvec(op)
ie.extremal_eigenvalue_lanczos(mv, pre, op.n, which="max", max_iters=300)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
print(ie.extremal_eigenvalue_lanczos(mv, pre, op.n, which="min", max_iters=300, return_steps=True))
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
