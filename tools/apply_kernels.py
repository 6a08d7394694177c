"""Config-5 translation-shared apply (for ncu captures of k_apply_dmma / k_scatter_fixed)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_12574_b200 as ie  # noqa: E402

grid = ie.build_grid(2, 1024)
op = ie.build_operator(grid, lattice="cell")
pre = ie.from_decomposition(op, ie.build_decomposition(grid, 128, 2, "schwarz"))
r = torch.from_numpy(np.random.default_rng(0).standard_normal(op.n)).cuda()
z = torch.empty_like(r)
for _ in range(3):
    pre.apply_device(r, z)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50):
    pre.apply_device(r, z)
e1.record()
torch.cuda.synchronize()
print(f"apply: {e0.elapsed_time(e1) / 50 * 1e3:.1f} us")
