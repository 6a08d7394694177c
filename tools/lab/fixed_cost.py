"""Device-resident and host-to-host solve wall times at small K (per-solve fixed cost), median of 15."""
import os, sys, time, json
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2108_12574_b200 as ie
grid = ie.build_grid(2, 1024); op = ie.build_operator(grid, lattice="cell")
mv = ie.ToeplitzMatvec(op)
pre = ie.from_decomposition(op, ie.build_decomposition(grid, 128, 2, "schwarz"))
pin = torch.empty(op.n, dtype=torch.float64, pin_memory=True)
f_host = pin.numpy(); f_host[:] = np.random.default_rng(3).standard_normal(op.n)
f_dev = torch.from_numpy(f_host).cuda()
def med(fn, reps=15):
    fn(); torch.cuda.synchronize(); ts = []
    for _ in range(reps):
        t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); ts.append(time.perf_counter() - t0)
    return round(1e3 * float(np.median(ts)), 4)
out = {}
for K in (5, 10, 20, 50):
    out[K] = {"dev": med(lambda: ie.solve(mv, pre, f_dev, tol=1e-10, max_iters=K)),
              "host": med(lambda: ie.solve(mv, pre, f_host, tol=1e-10, max_iters=K))}
print(json.dumps(out))
