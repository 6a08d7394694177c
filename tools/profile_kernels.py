"""Small driver for ncu captures (one GPU): K1 2-RHS pass at config-3 size,
K3 apply at config-5 size without translation sharing (factors streamed from
HBM), then the same apply with sharing."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_12574_b200 as ie  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
if which in ("all", "k1"):
    op = ie.build_operator(ie.build_grid(2, 256), lattice="cell")
    mv = ie.ToeplitzMatvec(op)
    X = torch.from_numpy(np.random.default_rng(0).standard_normal((2, op.n))).cuda()
    Y = torch.empty_like(X)
    for _ in range(3):
        mv.matvec_device(X, Y, nrhs=2)
if which in ("all", "k3"):
    grid = ie.build_grid(2, 1024)
    op = ie.build_operator(grid, lattice="cell")
    dec = ie.build_decomposition(grid, 128, 2, "schwarz")
    r = torch.from_numpy(np.random.default_rng(1).standard_normal(op.n)).cuda()
    z = torch.empty_like(r)
    for share in (False, True):
        pre = ie.from_decomposition(op, dec, share_translated=share)
        for _ in range(3):
            pre.apply_device(r, z)
torch.cuda.synchronize()
print("profile driver done")
if which == "fft":
    op = ie.build_operator(ie.build_grid(2, 1024), lattice="cell")
    mv = ie.KernelMatvec(op, method="fft")
    X = torch.from_numpy(np.random.default_rng(0).standard_normal((2, op.n))).cuda()
    Y = torch.empty_like(X)
    for _ in range(3):
        mv.matvec_device(X, Y, nrhs=2)
    torch.cuda.synchronize()
    print("fft driver done")
if which == "k1c5":
    op = ie.build_operator(ie.build_grid(2, 1024), lattice="cell")
    mv = ie.KernelMatvec(op, method="direct")
    X = torch.from_numpy(np.random.default_rng(0).standard_normal((2, op.n))).cuda()
    Y = torch.empty_like(X)
    mv.matvec_device(X, Y, nrhs=2)
    torch.cuda.synchronize()
    print("k1c5 driver done")
if which == "gemm":
    grid = ie.build_grid(2, 1024)
    op = ie.build_operator(grid, lattice="cell")
    pre = ie.from_decomposition(op, ie.build_decomposition(grid, 128, 2, "schwarz"))
    r = torch.from_numpy(np.random.default_rng(1).standard_normal(op.n)).cuda()
    z = torch.empty_like(r)
    for _ in range(3):
        pre.apply_device(r, z)
    torch.cuda.synchronize()
    print("gemm driver done")
if which == "k1n512":
    op = ie.build_operator(ie.build_grid(2, 512), lattice="cell")
    mv = ie.KernelMatvec(op, method="direct")
    X = torch.from_numpy(np.random.default_rng(0).standard_normal((2, op.n))).cuda()
    Y = torch.empty_like(X)
    mv.matvec_device(X, Y, nrhs=2)
    torch.cuda.synchronize()
    print("k1n512 done")
