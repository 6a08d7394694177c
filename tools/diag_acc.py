"""Row accuracy of the device matvecs against an extended-precision direct
sum (np.longdouble) on sampled rows, for 1 and 2 RHS."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_12574_b200 as ie  # noqa: E402
from oracle import iedd_oracle as O  # noqa: E402

for n in (32, 256):
    op = ie.build_operator(ie.build_grid(2, n), lattice="cell")
    rng = np.random.default_rng(1)
    X = rng.standard_normal((2, op.n))
    X[1] *= 1e6  # second column much larger: tests the 2-RHS packing isolation
    Xt = torch.from_numpy(X).cuda()
    res = {}
    for method in ("direct", "fft"):
        mv = ie.KernelMatvec(op, method=method)
        Y2 = torch.empty_like(Xt)
        mv.matvec_device(Xt, Y2, nrhs=2)
        y1 = torch.empty(op.n, dtype=torch.float64, device="cuda")
        mv.matvec_device(Xt[0], y1)
        res[method + "_1rhs"] = y1.cpu().numpy()
        res[method + "_2rhs"] = Y2[0].cpu().numpy()
    oop = O.build_operator(O.build_grid(2, n), "cell")
    res["oracle_fft"] = O.FFTMatvec(oop).matvec(X[0])
    mi = oop.grid.multi_indices().astype(np.longdouble)
    h = np.longdouble(1) / n
    xl = X[0].astype(np.longdouble)
    rows = np.random.default_rng(0).choice(op.n, 32, replace=False)
    errs = {k: [] for k in res}
    for i in rows:
        d2 = ((mi - mi[i]) ** 2).sum(axis=1) * h * h
        d2[i] = 1
        k = -(h * h) * np.log(d2) / (4 * np.pi)
        k[i] = np.longdouble(op.diag_value)
        yr = (k * xl).sum()
        for name, y in res.items():
            errs[name].append(float(abs(np.longdouble(y[i]) - yr) / abs(yr)))
    for name, e in errs.items():
        print(f"n={n} {name:12s} row rel err median {np.median(e):.2e} max {np.max(e):.2e}")
