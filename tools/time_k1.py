"""K1 direct-sum timing at configs 3 and 5 (2-RHS pass), pair-evals/s."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_12574_b200 as ie  # noqa: E402

for n, reps in ((256, 20), (1024, 2)):
    op = ie.build_operator(ie.build_grid(2, n), lattice="cell")
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
    print(f"K1 n={n}: {ms:.3f} ms per 2-RHS pass, {op.n**2 / (ms * 1e-3):.4e} pair-evals/s")
