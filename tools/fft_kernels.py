"""Per-kernel times of one config-5 2-RHS FFT pass (for the ncu launch list:
ncu --metrics gpu__time_duration.sum -k regex:k_fft python tools/fft_kernels.py)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_12574_b200 as ie  # noqa: E402

op = ie.build_operator(ie.build_grid(2, int(os.environ.get("N1D", "1024"))), lattice="cell")
mv = ie.KernelMatvec(op, method="fft")
X = torch.from_numpy(np.random.default_rng(0).standard_normal((2, op.n))).cuda()
Y = torch.empty_like(X)
for _ in range(3):
    mv.matvec_device(X, Y, nrhs=2)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    mv.matvec_device(X, Y, nrhs=2)
e1.record()
torch.cuda.synchronize()
print(f"2-RHS pass: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us")
