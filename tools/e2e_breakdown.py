"""Per-solve fixed cost of the end-to-end path (e2e vs device
iter/s imply ~0.4 ms per solve): wall time of pcg.solve from pinned numpy f
to numpy u for K = 5 .. 50 iterations (linear fit: slope = per iteration,
intercept = per solve), next to the device-resident solve and the bare 8 MB
host<->device copies."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_12574_b200 as ie  # noqa: E402

grid = ie.build_grid(2, 1024)
op = ie.build_operator(grid, lattice="cell")
mv = ie.ToeplitzMatvec(op)
pre = ie.from_decomposition(op, ie.build_decomposition(grid, 128, 2, "schwarz"))
pin = torch.empty(op.n, dtype=torch.float64, pin_memory=True)
f_host = pin.numpy()
f_host[:] = np.random.default_rng(3).standard_normal(op.n)
f_dev = torch.from_numpy(f_host).cuda()


def best(fn, reps=7):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts))


out = {"K": [], "host_ms": [], "device_ms": []}
for K in (5, 10, 20, 50):
    out["K"].append(K)
    out["host_ms"].append(1e3 * best(lambda: ie.solve(mv, pre, f_host, tol=1e-10, max_iters=K)))
    out["device_ms"].append(1e3 * best(lambda: ie.solve(mv, pre, f_dev, tol=1e-10, max_iters=K)))
for key in ("host_ms", "device_ms"):
    slope, icpt = np.polyfit(out["K"], out[key], 1)
    out[key + "_fit"] = {"per_iteration_ms": slope, "per_solve_ms": icpt}
d = torch.empty(op.n, dtype=torch.float64, device="cuda")
out["h2d_8MB_ms"] = 1e3 * best(lambda: d.copy_(pin, non_blocking=True))
out["d2h_8MB_ms"] = 1e3 * best(lambda: pin.copy_(d, non_blocking=True))
print(json.dumps(out, indent=1))
