"""Apply time of the large-block path (k_apply_big) vs the per-block packed
kernel (IEDD_B200_BIG_MIN_S moves the switch-over), CBD and config 4."""
import os
import subprocess
import sys

if len(sys.argv) > 1:
    import numpy as np
    import torch
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_2108_12574_b200 as ie
    for name, (dim, n, m, w, kind) in {"cbd2d_n64": (2, 64, 16, 1, "cbd"), "cbd3d_n16": (3, 16, 8, 1, "cbd"),
                                        "c4": (3, 32, 4, 1, "schwarz"), "g64": (2, 64, 2, 1, "schwarz")}.items():
        grid = ie.build_grid(dim, n)
        op = ie.build_operator(grid)
        pre = ie.from_decomposition(op, ie.build_decomposition(grid, m, w, kind))
        r = torch.from_numpy(np.random.default_rng(0).standard_normal(op.n)).cuda()
        for _ in range(3):
            z = pre.apply(r)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(50):
            z = pre.apply(r)
        e1.record()
        torch.cuda.synchronize()
        print(f"{name:10s} {sys.argv[1]:>6s} apply {e0.elapsed_time(e1) / 50 * 1e3:8.1f} us  |z|={float(z.norm()):.15e}")
    sys.exit(0)
for v in ("1024", "512"):
    subprocess.run([sys.executable, __file__, v], check=True, env=dict(os.environ, IEDD_B200_BIG_MIN_S=v))
