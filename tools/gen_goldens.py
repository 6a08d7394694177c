"""Freeze golden vectors from the UNMODIFIED reference package (iedd).

Runs only in the build container, where the read-only reference lives at
/root/reference/pkg/src.  The GPU box never imports the reference: tests read
the .npz / .json fixtures this script writes under tests/golden/.

Usage:
    python tools/gen_goldens.py                 # small + c1..c4 fixtures
    python tools/gen_goldens.py --only c5       # the 9-minute c5 run
    python tools/gen_goldens.py --only cbd      # CBD rows of goldens.json

Configs follow BASELINE.json / SURVEY.md section 8(d): cell lattice, f from
default_rng(seed).standard_normal(N), tol 1e-10, u0 = 0.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")

# (dim, n, m, overlap, seed) per BASELINE.json config
CONFIGS = {
    "c1": (2, 32, 4, 1, 0),
    "c2": (2, 64, 8, 1, 0),
    "c3": (2, 256, 32, 2, 1),
    "c4": (3, 32, 4, 1, 2),
    "c5": (2, 1024, 128, 2, 3),
}


def _ref():
    if not os.path.isdir(REF_SRC):
        sys.exit("reference not present; fixtures are generated in the build container only")
    sys.path.insert(0, REF_SRC)
    import iedd  # noqa: F401
    from iedd import geometry, kernel, pcg, precond, spectrum, toeplitz

    return geometry, kernel, pcg, precond, spectrum, toeplitz


class _Counted:
    """Wraps a matvec to count calls (gives Lanczos step counts)."""

    def __init__(self, mv):
        self.mv = mv
        self.calls = 0

    def matvec(self, v):
        self.calls += 1
        return self.mv.matvec(v)


def gen_small(out):
    geometry, kernel, pcg, precond, spectrum, toeplitz = _ref()
    data = {}
    rng = np.random.default_rng(20260)
    # matvec cases (reference tests/test_toeplitz.py:68-78 plus the BASELINE lattice)
    for dim, n, lat in [(2, 8, "span"), (2, 32, "span"), (2, 16, "cell"), (3, 8, "cell"),
                        (1, 16, "cell"), (2, 32, "cell"), (3, 4, "cell"), (2, 12, "cell"),
                        (2, 10, "span")]:
        op = kernel.build_operator(geometry.build_grid(dim, n), lattice=lat)
        tm = toeplitz.ToeplitzMatvec(op)
        x = rng.standard_normal(op.n)
        key = f"mv_{dim}_{n}_{lat}"
        data[key + "_x"] = x
        data[key + "_y"] = tm.matvec(x)
        data[key + "_ydense"] = op.dense() @ x
        data[key + "_diag"] = np.array(op.diag_value)
        data[key + "_row0"] = op.dense()[0]
    # diagonal constants
    for dim, h in [(1, 1.0), (2, 1.0), (3, 1.0), (2, 1 / 32), (3, 1 / 32), (2, 1 / 1024), (1, 1 / 32)]:
        data[f"diag_{dim}_{h!r}"] = np.array(kernel.diagonal_entry(dim, h))
    # preconditioner apply cases
    for dim, n, m, w, kind, lat in [(2, 32, 4, 1, "schwarz", "cell"), (2, 32, 4, 1, "jacobi", "cell"),
                                    (2, 16, 2, 1, "schwarz", "span"), (3, 8, 2, 1, "schwarz", "cell"),
                                    (2, 64, 8, 2, "schwarz", "cell"), (2, 12, 3, 1, "schwarz", "cell")]:
        g = geometry.build_grid(dim, n)
        op = kernel.build_operator(g, lattice=lat)
        d = geometry.build_decomposition(g, m, w, kind)
        pre = precond.from_decomposition(op, d)
        r = rng.standard_normal(op.n)
        key = f"ap_{dim}_{n}_{m}_{w}_{kind}_{lat}"
        data[key + "_r"] = r
        data[key + "_z"] = pre.apply(r)
        if (dim, n, kind) == (2, 32, "schwarz"):
            for b in (0, 5):
                data[key + f"_G{b}"] = pre._solvers[b].factor.g
    np.savez_compressed(os.path.join(out, "ref_small.npz"), **data)

    # small PCG runs (reference tests/test_pcg.py and goldens iterations suites)
    pcgd = {}
    cases = [
        ("t16_jacobi_random", 2, 16, 2, 1, "jacobi", None, "random", 0, 1e-12, None),
        ("t16_schwarz_random", 2, 16, 2, 1, "schwarz", None, "random", 0, 1e-12, None),
        ("g16_jacobi_noise", 2, 16, 2, 1, "jacobi", None, "noise", 0, 1e-12, None),
        ("g16_schwarz_noise", 2, 16, 2, 1, "schwarz", None, "noise", 0, 1e-12, None),
        ("g8_3d_jacobi_noise", 3, 8, 2, 1, "jacobi", None, "noise", 0, 1e-12, None),
        ("g8_3d_schwarz_noise", 3, 8, 2, 1, "schwarz", None, "noise", 0, 1e-12, None),
        ("stag8_schwarz", 2, 8, 2, 1, "schwarz", None, "random", 0, 1e-30, 5000),
        ("cap16_jacobi", 2, 16, 2, 1, "jacobi", None, "random", 0, 1e-12, 5),
    ]
    for name, dim, n, m, w, kind, lat, rhs, seed, tol, mi in cases:
        g = geometry.build_grid(dim, n)
        op = kernel.build_operator(g, lattice=lat)
        mv = toeplitz.ToeplitzMatvec(op)
        pre = precond.from_decomposition(op, geometry.build_decomposition(g, m, w, kind))
        f, _ = pcg.make_rhs(mv, op.n, mode=rhs, seed=seed)
        u, rep = pcg.solve(mv, pre, f, tol=tol, max_iters=mi)
        pcgd[name + "_f"] = f
        pcgd[name + "_u"] = u
        pcgd[name + "_hist"] = np.array(rep.residual_history)
        pcgd[name + "_meta"] = np.array([rep.n_it, rep.converged, rep.stagnated], dtype=np.int64)
    np.savez_compressed(os.path.join(out, "ref_pcg_small.npz"), **pcgd)

    # small Lanczos / dense-spectrum cases (reference tests/test_spectrum.py:159-178)
    lz = {}
    for name, dim, n, m, w, kind, which in [("j16max", 2, 16, 2, 1, "jacobi", "max"),
                                            ("s16min", 2, 16, 4, 1, "schwarz", "min"),
                                            ("s8_3dmin", 3, 8, 2, 1, "schwarz", "min")]:
        g = geometry.build_grid(dim, n)
        op = kernel.build_operator(g)
        pre = precond.from_decomposition(op, geometry.build_decomposition(g, m, w, kind))
        mv = _Counted(toeplitz.ToeplitzMatvec(op))
        lam = spectrum.extremal_eigenvalue_lanczos(mv, pre, op.n, which=which)
        rep = spectrum.preconditioned_spectrum(op, pre)
        lz[name] = np.array([lam, mv.calls, rep.lambda_min, rep.lambda_max])
    np.savez_compressed(os.path.join(out, "ref_lanczos_small.npz"), **lz)

    # the reference's own golden suites (paper values), copied as data
    with open(os.path.join(REF_SRC, "iedd", "goldens.json")) as fh:
        suites = json.load(fh)
    keep = {k: v for k, v in suites.items()
            if k in ("spectrum-2d", "spectrum-3d", "schwarz-scaling-2d", "interface-2d", "interface-3d",
                     "iterations-2d", "iterations-3d", "pairing")}
    pkg_data = os.path.join(os.path.dirname(out), "..", "paper_2108_12574_b200", "data", "goldens.json")
    with open(pkg_data, "w") as fh:  # shipped as package data (the golden runner's default suite file)
        json.dump(keep, fh, indent=1)


def _pcg_config(name, max_iters=None, store_u="f64"):
    geometry, kernel, pcg, precond, spectrum, toeplitz = _ref()
    dim, n, m, w, seed = CONFIGS[name]
    g = geometry.build_grid(dim, n)
    op = kernel.build_operator(g, lattice="cell")
    mv = toeplitz.ToeplitzMatvec(op)
    f = np.random.default_rng(seed).standard_normal(op.n)
    res = {}
    kinds = ("schwarz", "jacobi") if name == "c1" else ("schwarz",)
    for kind in kinds:
        t0 = time.perf_counter()
        pre = precond.from_decomposition(op, geometry.build_decomposition(g, m, w, kind))
        t_f = time.perf_counter() - t0
        u, rep = pcg.solve(mv, pre, f, tol=1e-10, max_iters=max_iters)
        res[f"{kind}_hist"] = np.array(rep.residual_history)
        res[f"{kind}_meta"] = np.array([rep.n_it, rep.converged, rep.stagnated], dtype=np.int64)
        res[f"{kind}_times"] = np.array([t_f, rep.t_pcg, rep.t_s])
        res[f"{kind}_u"] = u.astype(np.float32) if store_u == "f32" else u
        res[f"{kind}_unorm"] = np.array(np.linalg.norm(u))
        print(name, kind, rep.n_it, rep.achieved_residual, f"t_f={t_f:.2f}s t_pcg={rep.t_pcg:.2f}s", flush=True)
    return res


def _lanczos(name, kinds, whiches, max_iters):
    geometry, kernel, pcg, precond, spectrum, toeplitz = _ref()
    dim, n, m, w, _ = CONFIGS[name]
    g = geometry.build_grid(dim, n)
    op = kernel.build_operator(g, lattice="cell")
    res = {}
    for kind in kinds:
        pre = precond.from_decomposition(op, geometry.build_decomposition(g, m, w, kind))
        for which in whiches:
            mv = _Counted(toeplitz.ToeplitzMatvec(op))
            lam = spectrum.extremal_eigenvalue_lanczos(mv, pre, op.n, which=which,
                                                       max_iters=max_iters, seed=0)
            res[f"lam_{kind}_{which}"] = np.array([lam, mv.calls])
            print(name, kind, which, lam, mv.calls, flush=True)
    return res


def gen_cbd(out):
    """CBD (colour-block-diagonal) rows of goldens.json run through the
    reference itself (cli.py:266-283 solve path; spectrum.py Lanczos with
    share_mirrored_subdomains as cli.py:249-263).  goldens.json's 3D CBD n_it
    (27) is stale: the reference computes 22 / 21, recorded here."""
    geometry, kernel, pcg, precond, spectrum, toeplitz = _ref()
    suites = json.load(open(os.path.join(os.path.dirname(out), "..", "paper_2108_12574_b200", "data",
                                         "goldens.json")))
    res, meta = {}, []
    for sname in ("iterations-2d", "iterations-3d"):
        s = suites[sname]
        for case in s["cases"]:
            if case["kind"] != "cbd":
                continue
            g = geometry.build_grid(case["dim"], case["n"])
            op = kernel.build_operator(g)
            mv = toeplitz.ToeplitzMatvec(op)
            dec = geometry.build_decomposition(g, case["m"], case["overlap"], "cbd")
            pre = precond.from_decomposition(op, dec, backend="exact", dense_limit=op.n)
            f, _ = pcg.make_rhs(mv, op.n, mode=s["rhs"], seed=s["seed"])
            u, rep = pcg.solve(mv, pre, f, tol=s["tol"])
            key = f"{case['dim']}d_n{case['n']}_m{case['m']}"
            r = np.random.default_rng(7).standard_normal(op.n)
            res[f"z_{key}"] = pre.apply(r)
            res[f"u_{key}"] = u
            res[f"hist_{key}"] = np.array(rep.residual_history)
            meta.append(dict(case, n_it_ref=rep.n_it, converged=bool(rep.converged), key=key,
                             t_factor_s=pre.t_factor, t_pcg_s=rep.t_pcg))
            print("cbd solve", key, rep.n_it, flush=True)
    for sname in ("spectrum-2d", "spectrum-3d"):
        for case in suites[sname]["cases"]:
            if case["kind"] != "cbd":
                continue
            g = geometry.build_grid(case["dim"], case["n"])
            op = kernel.build_operator(g)
            dec = geometry.build_decomposition(g, case["m"], case["overlap"], "cbd")
            pre = precond.from_decomposition(op, dec, backend="exact", dense_limit=op.n,
                                             share_mirrored_subdomains=True)
            key = f"{case['dim']}d_n{case['n']}_m{case['m']}"
            lam = {}
            for which in ("min", "max"):
                mvc = _Counted(toeplitz.ToeplitzMatvec(op))
                lam[which] = (spectrum.extremal_eigenvalue_lanczos(mvc, pre, op.n, which=which), mvc.calls)
            meta.append(dict(case, suite=sname, key=key, lanczos_min=lam["min"][0], steps_min=lam["min"][1],
                             lanczos_max=lam["max"][0], steps_max=lam["max"][1]))
            print("cbd lanczos", key, lam, flush=True)
    np.savez_compressed(os.path.join(out, "ref_cbd.npz"), **res)
    with open(os.path.join(out, "ref_cbd.json"), "w") as fh:
        json.dump(meta, fh, indent=1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=None)
    args = ap.parse_args()
    os.makedirs(OUT, exist_ok=True)
    todo = [args.only] if args.only else ["small", "c1", "c2", "c3", "c4"]
    for item in todo:
        t0 = time.perf_counter()
        if item == "small":
            gen_small(OUT)
        elif item == "c1":
            np.savez_compressed(os.path.join(OUT, "ref_c1.npz"), **_pcg_config("c1"))
        elif item == "c2":
            np.savez_compressed(os.path.join(OUT, "ref_c2.npz"),
                                **_lanczos("c2", ("schwarz", "jacobi"), ("min", "max"), 300))
        elif item == "c3":
            np.savez_compressed(os.path.join(OUT, "ref_c3.npz"), **_pcg_config("c3"))
        elif item == "c4":
            res = _pcg_config("c4")
            res.update(_lanczos("c4", ("schwarz",), ("min",), 200))
            np.savez_compressed(os.path.join(OUT, "ref_c4.npz"), **res)
        elif item == "cbd":
            gen_cbd(OUT)
        elif item == "c5":
            np.savez_compressed(os.path.join(OUT, "ref_c5.npz"),
                                **_pcg_config("c5", max_iters=50, store_u="f32"))
        print(f"[{item}] {time.perf_counter() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main()
