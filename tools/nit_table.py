"""PCG iteration counts of every parity case (native solver, both matvec
methods, both apply variants, shared/unshared factors) against the
reference's recorded counts (goldens) or the oracle's, with the last
residuals: the evidence for the n_it contract."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2108_12574_b200 as ie  # noqa: E402
from oracle import iedd_oracle as O  # noqa: E402

GOLD = os.path.join(ROOT, "tests", "golden")
rows = []


def rec(case, rep, ref):
    rows.append({"case": case, "n_it": rep.n_it, "ref": int(ref), "d": rep.n_it - int(ref),
                 "tail": [float(f"{x:.3e}") for x in rep.residual_history[-3:]]})
    print(json.dumps(rows[-1]), flush=True)


for name, (dim, n, m, w, seed, kinds) in {"c1": (2, 32, 4, 1, 0, ("schwarz", "jacobi")),
                                          "c3": (2, 256, 32, 2, 1, ("schwarz",)),
                                          "c4": (3, 32, 4, 1, 2, ("schwarz",))}.items():
    grid = ie.build_grid(dim, n)
    op = ie.build_operator(grid, lattice="cell")
    f = np.random.default_rng(seed).standard_normal(op.n)
    g = dict(np.load(os.path.join(GOLD, f"ref_{name}.npz")))
    for kind in kinds:
        dec = ie.build_decomposition(grid, m, w, kind)
        for variant in ("packed_inverse", "subst"):
            for share in (True, False):
                pre = ie.from_decomposition(op, dec, variant=variant, share_translated=share)
                for method in ("fft", "direct"):
                    u, rep = ie.solve(ie.KernelMatvec(op, method=method), pre, f, tol=1e-10)
                    rec(f"{name}/{kind}/{variant}/share={share}/{method}", rep, g[f"{kind}_meta"][0])

# TestProperties / TestScatterWidths shapes: oracle PCG with the dense matvec
for seed in range(6):
    rng = np.random.default_rng(100 + seed)
    dim = int(rng.choice([1, 2, 2, 3]))
    n = int(rng.choice({1: [16, 24, 64], 2: [8, 12, 16, 20], 3: [4, 6, 8]}[dim]))
    m = int(rng.choice([d for d in (1, 2, 4) if n % d == 0]))
    w = int(rng.integers(0, 3))
    kind = str(rng.choice(["jacobi", "schwarz"]))
    lat = str(rng.choice(["cell", "span"])) if dim == 2 else "cell"
    grid = ie.build_grid(dim, n)
    op = ie.build_operator(grid, lattice=lat)
    og = O.build_grid(dim, n)
    oop = O.build_operator(og, lat)
    a = oop.dense()
    x = rng.standard_normal(op.n)
    opre = O.SchwarzPrecond(oop, O.build_decomposition(og, m, w, kind))
    pre = ie.from_decomposition(op, ie.build_decomposition(grid, m, w, kind))
    ou, orep = O.pcg(lambda v: a @ v, opre, x, tol=1e-10)
    ou2, orep2 = O.pcg(O.FFTMatvec(oop), opre, x, tol=1e-10)
    for method in ("fft", "direct"):
        u, rep = ie.solve(ie.KernelMatvec(op, method=method) if method == "direct" else ie.ToeplitzMatvec(op),
                          pre, x, tol=1e-10)
        rec(f"prop{seed}/{dim}d n={n} m={m} w={w} {kind} {lat}/{method} (oracle dense)", rep, orep.n_it)
        if orep2 is not None:
            rec(f"prop{seed}/{method} (oracle fft)", rep, orep2.n_it)

for dim, n, m, w, kind in [(1, 3000, 8, 1, "schwarz"), (2, 50, 5, 1, "schwarz"), (2, 50, 5, 2, "schwarz"),
                           (3, 14, 7, 1, "schwarz"), (2, 50, 5, 0, "jacobi")]:
    rng = np.random.default_rng(1234)
    grid = ie.build_grid(dim, n)
    op = ie.build_operator(grid, lattice="cell")
    og = O.build_grid(dim, n)
    oop = O.build_operator(og, "cell")
    opre = O.SchwarzPrecond(oop, O.build_decomposition(og, m, w, kind))
    x = rng.standard_normal(op.n)
    pre = ie.from_decomposition(op, ie.build_decomposition(grid, m, w, kind))
    u, rep = ie.solve(ie.KernelMatvec(op, method="direct"), pre, x, tol=1e-10)
    a = oop.dense()
    ou, orep = O.pcg(lambda v: a @ v, opre, x, tol=1e-10)
    rec(f"scatter {dim}d n={n} m={m} w={w} {kind}/direct (oracle dense)", rep, orep.n_it)

bad = [r for r in rows if abs(r["d"]) > 1]
print(json.dumps({"cases": len(rows), "beyond_pm1": len(bad), "worst": max(abs(r["d"]) for r in rows)}))
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
with open(os.path.join(ROOT, "gpurun_out", "nit_table.json"), "w") as fh:
    json.dump(rows, fh, indent=1)
