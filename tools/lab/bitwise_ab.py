"""Bitwise fingerprint of the FFT matvec and PCG outputs of the loaded library
build (IEDD_B200_LIB selects another build): a refactor of addressing or
scaling code must leave every output bit unchanged.

  python tools/lab/bitwise_ab.py            # in-tree build
  IEDD_B200_LIB=tools/lab/lib_base.so python tools/lab/bitwise_ab.py
"""
import hashlib
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2108_12574_b200 as ie  # noqa: E402


def h(t):
    a = t.detach().cpu().numpy() if isinstance(t, torch.Tensor) else np.asarray(t)
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


out = {}
for dim, n in ((2, 1024), (2, 2048), (2, 1000), (2, 256), (3, 32), (3, 64), (1, 4096)):
    op = ie.build_operator(ie.build_grid(dim, n), lattice="cell")
    mv = ie.ToeplitzMatvec(op)
    rng = np.random.default_rng(7)
    X = torch.from_numpy(np.stack([rng.standard_normal(op.n), 1e-9 * rng.standard_normal(op.n)])).cuda()
    Y = torch.empty_like(X)
    mv.matvec_device(X, Y, nrhs=2)
    Y1 = torch.empty_like(X[0])
    mv.matvec_device(X[0].contiguous(), Y1)
    torch.cuda.synchronize()
    out[f"matvec_{dim}d_n{n}"] = [h(Y), h(Y1)]
for dim, n, m, w in ((2, 1024, 128, 2), (2, 256, 32, 2), (3, 32, 4, 1)):
    g = ie.build_grid(dim, n)
    op = ie.build_operator(g, lattice="cell")
    pre = ie.from_decomposition(op, ie.build_decomposition(g, m, w, "schwarz"))
    f = np.random.default_rng(3).standard_normal(op.n)
    u, rep = ie.solve(ie.ToeplitzMatvec(op), pre, f, tol=1e-10, max_iters=40)
    out[f"pcg_{dim}d_n{n}"] = [h(u), h(np.asarray(rep.residual_history)), int(rep.n_it)]
print(json.dumps({"lib": os.environ.get("IEDD_B200_LIB", "in-tree"), "hashes": out}))
