import os, sys, time, numpy as np, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import paper_2108_12574_b200 as ie
res = {}
for name, dim, n, m, kind, which in (("c2j min", 2, 64, 8, "jacobi", "min"), ("c2s min", 2, 64, 8, "schwarz", "min"), ("c4 min", 3, 32, 4, "schwarz", "min")):
    grid = ie.build_grid(dim, n); op = ie.build_operator(grid, lattice="cell")
    mv = ie.ToeplitzMatvec(op); pre = ie.from_decomposition(op, ie.build_decomposition(grid, m, 1, kind))
    ie.extremal_eigenvalue_lanczos(mv, pre, op.n, which=which, max_iters=300)
    ts = []
    for _ in range(5):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        lam = ie.extremal_eigenvalue_lanczos(mv, pre, op.n, which=which, max_iters=300)
        torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    res[name] = (round(min(ts) * 1e3, 2), round(float(np.median(ts)) * 1e3, 2))
print(res)
