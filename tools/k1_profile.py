"""One K1 direct-sum 2-RHS pass at config 5 (for ncu --set full)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_12574_b200 as ie  # noqa: E402

op = ie.build_operator(ie.build_grid(2, 1024), lattice="cell")
mv = ie.KernelMatvec(op, method="direct")
X = torch.from_numpy(np.random.default_rng(0).standard_normal((2, op.n))).cuda()
Y = torch.empty_like(X)
mv.matvec_device(X, Y, nrhs=2)
torch.cuda.synchronize()
print("done")
