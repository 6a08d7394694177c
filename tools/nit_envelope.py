"""Iteration-count envelope of the reference PCG under last-bit rounding
changes (evidence for the n_it contract, tests/golden/nit_envelope.json).

The oracle PCG (a restatement of pcg.py:54-136 with the reference's own FFT
matvec, toeplitz.py:39-50, and per-block Cholesky solves, precond.py:91-100)
is run with its matvec output perturbed by independent random relative
errors of one unit in the last place (y_i * (1 + 2^-52 g_i), g ~ N(0,1)) --
the size of the rounding difference between any two correct FP64
implementations of the same matvec.  The set of n_it values this produces is
the reference's own sensitivity: an implementation whose rounding differs
from numpy's pocketfft cannot be expected to land closer than that.

  python tools/nit_envelope.py [samples] [case ...]   # ~10 min on 8 cores
"""
import collections
import json
import multiprocessing as mp
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CASES = {  # name: (dim, n, m, w, kind, seed)
    "c1_schwarz": (2, 32, 4, 1, "schwarz", 0),
    "c1_jacobi": (2, 32, 4, 1, "jacobi", 0),
    "c3_schwarz": (2, 256, 32, 2, "schwarz", 1),
    "c4_schwarz": (3, 32, 4, 1, "schwarz", 2),
    # the sharded-driver CPU test case (tests/test_distributed.py CASE)
    "gloo_n128_m16_w2_seed4": (2, 128, 16, 2, "schwarz", 4),
}
EPS = 2.0 ** -52


def run(args):
    name, s = args
    from oracle import iedd_oracle as O
    dim, n, m, w, kind, seed = CASES[name]
    g = O.build_grid(dim, n)
    op = O.build_operator(g, "cell")
    pre = O.SchwarzPrecond(op, O.build_decomposition(g, m, w, kind))
    mv = O.FFTMatvec(op)
    f = np.random.default_rng(seed).standard_normal(op.n)
    rng = np.random.default_rng(10_000 + s)

    def a(x):
        y = mv.matvec(x)
        return y if s == 0 else y * (1.0 + EPS * rng.standard_normal(y.size))

    _, rep = O.pcg(a, pre, f, tol=1e-10)
    return name, s, rep.n_it


def main():
    samples = int(sys.argv[1]) if len(sys.argv) > 1 else 24
    names = sys.argv[2:] or list(CASES)
    jobs = [(nm, s) for nm in names for s in range(samples + 1)]
    out = {nm: collections.Counter() for nm in names}
    ref = {}
    with mp.Pool(min(8, os.cpu_count() or 1)) as pool:
        for nm, s, k in pool.imap_unordered(run, jobs):
            if s == 0:
                ref[nm] = k
            else:
                out[nm][k] += 1
    path = os.path.join(ROOT, "tests", "golden", "nit_envelope.json")
    try:
        with open(path) as fh:
            res = json.load(fh)
    except OSError:
        res = {}
    res.update({nm: {"reference": ref[nm], "perturbed_n_it": {str(k): v for k, v in sorted(out[nm].items())},
                     "min": min(out[nm]), "max": max(out[nm]), "samples": samples} for nm in names})
    res["_how"] = ("oracle PCG, matvec output times (1 + 2^-52 g), g ~ N(0,1) iid per entry and call; "
                   "tools/nit_envelope.py")
    print(json.dumps(res, indent=1))
    with open(path, "w") as fh:
        json.dump(res, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
