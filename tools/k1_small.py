"""K1 direct-sum 2-RHS pass timings at the small configs (c1-c4 sizes)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_12574_b200 as ie  # noqa: E402

for dim, n, reps in ((2, 32, 50), (2, 64, 50), (2, 256, 20), (3, 32, 20)):
    op = ie.build_operator(ie.build_grid(dim, n), lattice="cell")
    mv = ie.KernelMatvec(op, method="direct")
    X = torch.from_numpy(np.random.default_rng(0).standard_normal((2, op.n))).cuda()
    Y = torch.empty_like(X)
    mv.matvec_device(X, Y, nrhs=2)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        mv.matvec_device(X, Y, nrhs=2)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"dim={dim} n={n}: {ms:.4f} ms per 2-RHS pass, {op.n ** 2 / (ms * 1e-3):.3e} pair-evals/s")
