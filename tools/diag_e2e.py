"""Time the end-to-end solve call (numpy in/out) piece by piece at config 5."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_12574_b200 as ie  # noqa: E402

grid = ie.build_grid(2, 1024)
op = ie.build_operator(grid, lattice="cell")
mv = ie.ToeplitzMatvec(op)
pre = ie.from_decomposition(op, ie.build_decomposition(grid, 128, 2, "schwarz"))
fp = torch.empty(op.n, dtype=torch.float64, pin_memory=True)
f = fp.numpy()
f[:] = np.random.default_rng(3).standard_normal(op.n)
fd = torch.from_numpy(f).cuda()
for K in (3, 10):
    ie.solve(mv, pre, fd, tol=1e-10, max_iters=K)
torch.cuda.synchronize()
for trial in range(4):
    t0 = time.perf_counter()
    u, rep = ie.solve(mv, pre, fd, tol=1e-10, max_iters=10)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    u, rep = ie.solve(mv, pre, f, tol=1e-10, max_iters=10)
    t2 = time.perf_counter()
    x = torch.from_numpy(f).to("cuda")
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    y = x.cpu().numpy()
    t4 = time.perf_counter()
    print(f"device solve {1e3*(t1-t0):.2f} ms | numpy solve {1e3*(t2-t1):.2f} ms | H2D {1e3*(t3-t2):.2f} ms | "
          f"D2H {1e3*(t4-t3):.2f} ms | t_pcg {1e3*rep.t_pcg:.2f}")
