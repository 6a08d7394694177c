"""Isolate which component moves config-1 Jacobi iteration counts: oracle
PCG driven by the device matvec / device apply, vs the native solver."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_12574_b200 as ie  # noqa: E402
from oracle import iedd_oracle as O  # noqa: E402

g = O.build_grid(2, 32)
oop = O.build_operator(g, "cell")
f = np.random.default_rng(0).standard_normal(oop.n)
grid = ie.build_grid(2, 32)
op = ie.build_operator(grid, lattice="cell")
for kind in ("jacobi", "schwarz"):
    opre = O.SchwarzPrecond(oop, O.build_decomposition(g, 4, 1, kind))
    out = {}
    for variant in ("packed_inverse", "subst"):
        pre = ie.from_decomposition(op, ie.build_decomposition(grid, 4, 1, kind), variant=variant)
        out[f"oracle_pcg+dev_apply[{variant}]"] = O.pcg(O.FFTMatvec(oop), pre.apply, f, tol=1e-10)[1].n_it
    for method in ("direct", "fft"):
        mv = ie.KernelMatvec(op, method=method)
        out[f"oracle_pcg+dev_mv[{method}]"] = O.pcg(mv.matvec, opre, f, tol=1e-10)[1].n_it
        pre = ie.from_decomposition(op, ie.build_decomposition(grid, 4, 1, kind))
        out[f"oracle_pcg+dev_mv+dev_apply[{method}]"] = O.pcg(mv.matvec, pre.apply, f, tol=1e-10)[1].n_it
        u, rep = ie.solve(mv, pre, f, tol=1e-10)
        out[f"native[{method}]"] = rep.n_it
        out[f"native[{method}] hist tail"] = [f"{x:.2e}" for x in rep.residual_history[-4:]]
    print(kind, out)
