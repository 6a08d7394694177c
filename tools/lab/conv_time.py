"""Converged config-5 solves (unbounded max_iters) at a few tolerances: wall time and iterations
(the batch-size policy's no-op tail shows here, not in the bounded bench runs)."""
import os, sys, time, json
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2108_12574_b200 as ie
grid = ie.build_grid(2, 1024); op = ie.build_operator(grid, lattice="cell")
mv = ie.ToeplitzMatvec(op)
pre = ie.from_decomposition(op, ie.build_decomposition(grid, 128, 2, "schwarz"))
f = torch.from_numpy(np.random.default_rng(3).standard_normal(op.n)).cuda()
out = {}
for tol in (1e-2, 1e-3, 1e-4, 1e-6):
    ie.solve(mv, pre, f, tol=tol); torch.cuda.synchronize()
    ts = []
    for _ in range(5):
        t0 = time.perf_counter(); u, rep = ie.solve(mv, pre, f, tol=tol); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    out[str(tol)] = {"n_it": rep.n_it, "ms": round(1e3 * float(np.median(ts)), 3), "converged": rep.converged}
print(json.dumps(out))
