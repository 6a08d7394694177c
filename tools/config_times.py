"""Per-config wall times of the drop-in API on the GPU (solver / Lanczos after a
warm-up call), for the DESIGN.md table.  The reference timings are those
recorded by tools/gen_goldens.py when the goldens were frozen (t_pcg)."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2108_12574_b200 as ie  # noqa: E402

GOLD = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden")
out = {}


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        r = fn()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return min(ts), r


for name, (dim, n, m, w, seed, kinds) in {"c1": (2, 32, 4, 1, 0, ("schwarz", "jacobi")),
                                          "c3": (2, 256, 32, 2, 1, ("schwarz",)),
                                          "c4": (3, 32, 4, 1, 2, ("schwarz",)),
                                          "c5": (2, 1024, 128, 2, 3, ("schwarz",))}.items():
    grid = ie.build_grid(dim, n)
    op = ie.build_operator(grid, lattice="cell")
    f = np.random.default_rng(seed).standard_normal(op.n)
    g = dict(np.load(os.path.join(GOLD, f"ref_{name}.npz")))
    for kind in kinds:
        dec = ie.build_decomposition(grid, m, w, kind)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pre = ie.from_decomposition(op, dec)
        torch.cuda.synchronize()
        t_f = time.perf_counter() - t0
        for method in ("fft", "direct"):
            if name == "c5" and method == "direct":
                continue
            mv = ie.KernelMatvec(op, method=method)
            mi = 50 if name == "c5" else None
            t, (u, rep) = timed(lambda: ie.solve(mv, pre, f, tol=1e-10, max_iters=mi))
            ref_t = float(g[f"{kind}_times"][1])
            out[f"{name} {kind} pcg [{method}]"] = dict(n_it=rep.n_it, ref_n_it=int(g[f"{kind}_meta"][0]),
                                                       t_s=t, ref_t_pcg_s=ref_t, speedup=ref_t / t,
                                                       t_build_s=t_f, ref_t_f_s=float(g[f"{kind}_times"][0]))
with open(os.path.join(GOLD, "ref_cbd.json")) as fh:
    cbd = {c["key"]: c for c in json.load(fh) if "n_it_ref" in c}
for key in ("2d_n64_m16", "3d_n16_m8"):
    c = cbd[key]
    grid = ie.build_grid(c["dim"], c["n"])
    op = ie.build_operator(grid)
    mv = ie.ToeplitzMatvec(op)
    dec = ie.build_decomposition(grid, c["m"], c["overlap"], "cbd")
    ie.from_decomposition(op, dec)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pre = ie.from_decomposition(op, dec)
    torch.cuda.synchronize()
    t_f = time.perf_counter() - t0
    f, _ = ie.make_rhs(mv, op.n, mode="noise", seed=0)
    t, (u, rep) = timed(lambda: ie.solve(mv, pre, f, tol=1e-12))
    out[f"cbd {key} pcg"] = dict(n_it=rep.n_it, ref_n_it=c["n_it_ref"], t_s=t, ref_t_pcg_s=c["t_pcg_s"],
                                 t_build_s=t_f, ref_t_f_s=c["t_factor_s"], smax=int(max(s.size for s in dec.subdomains)))
for name, (dim, n, m, w, kinds, mi) in {"c2": (2, 64, 8, 1, ("schwarz", "jacobi"), 300),
                                        "c4": (3, 32, 4, 1, ("schwarz",), 200)}.items():
    grid = ie.build_grid(dim, n)
    op = ie.build_operator(grid, lattice="cell")
    mv = ie.ToeplitzMatvec(op)
    for kind in kinds:
        pre = ie.from_decomposition(op, ie.build_decomposition(grid, m, w, kind))
        for which in (("min", "max") if name == "c2" else ("min",)):
            t, (lam, steps) = timed(lambda: ie.extremal_eigenvalue_lanczos(mv, pre, op.n, which=which, max_iters=mi,
                                                                          return_steps=True), reps=2)
            out[f"{name} {kind} lanczos {which}"] = dict(lam=lam, steps=steps, t_s=t)
print(json.dumps(out, indent=1))
