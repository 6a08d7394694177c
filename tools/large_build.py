"""Build time + apply agreement of the large-block paths (blocked sweep vs the
unblocked one-CTA Cholesky, IEDD_B200_UNBLOCKED_LARGE=1), config 4 and a
2D case with 1089-point blocks."""
import os
import subprocess
import sys
import time

import numpy as np

if len(sys.argv) > 1:
    import torch
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_2108_12574_b200 as ie
    res = {}
    for name, (dim, n, m, w, kind, share) in {"c4": (3, 32, 4, 1, "schwarz", True),
                                              "c4_noshare": (3, 32, 4, 1, "schwarz", False),
                                              "g64": (2, 64, 2, 1, "schwarz", True),
                                              "c3d48": (3, 48, 4, 1, "schwarz", True)}.items():
        grid = ie.build_grid(dim, n)
        op = ie.build_operator(grid, lattice="cell")
        dec = ie.build_decomposition(grid, m, w, kind)
        ie.from_decomposition(op, dec, share_translated=share)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pre = ie.from_decomposition(op, dec, share_translated=share)
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
        r = np.random.default_rng(0).standard_normal(op.n)
        np.save(f"gpurun_out/lb_{name}_{sys.argv[1]}.npy", pre.apply(r))
        print(name, sys.argv[1], f"build {t*1e3:.1f} ms", "smax", max(len(b) for b in dec.subdomains))
    sys.exit(0)
env = dict(os.environ)
subprocess.run([sys.executable, __file__, "sweep"], check=True)
env["IEDD_B200_UNBLOCKED_LARGE"] = "1"
subprocess.run([sys.executable, __file__, "unblocked"], check=True, env=env)
for name in ("c4", "c4_noshare", "g64", "c3d48"):
    a = np.load(f"gpurun_out/lb_{name}_sweep.npy")
    b = np.load(f"gpurun_out/lb_{name}_unblocked.npy")
    print(name, "rel diff", np.linalg.norm(a - b) / np.linalg.norm(b))
