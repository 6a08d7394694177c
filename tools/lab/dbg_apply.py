# debug: apply error pattern for one geometry (share on/off, both variants)
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2108_12574_b200 as ie
from oracle import iedd_oracle as O
dim, n, m, w, kind = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
grid = ie.build_grid(dim, n); op = ie.build_operator(grid)
og = O.build_grid(dim, n); oop = O.build_operator(og, "cell")
odec = O.build_decomposition(og, m, w, kind)
opre = O.SchwarzPrecond(oop, odec)
dec = ie.build_decomposition(grid, m, w, kind)
x = np.random.default_rng(0).standard_normal(op.n)
ref = opre.apply(x)
for share in (True, False):
    for variant in ("packed_inverse", "subst"):
        pre = ie.from_decomposition(op, dec, share_translated=share, variant=variant)
        y = pre.apply(x)
        err = np.abs(y - ref) / np.abs(ref).max()
        bad = np.nonzero(err > 1e-10)[0]
        print(share, variant, "rel", np.linalg.norm(y - ref) / np.linalg.norm(ref), "nbad", len(bad), "first", bad[:12])
        if len(bad) and dim == 2:
            B = np.zeros((n, n), int); B.flat[bad] = 1
            for row in B[:16]: print("".join(".#"[v] for v in row[:50]))
