"""The reference's golden-suite runner (cli.py:223-327) on the device path.

    python -m paper_2108_12574_b200 golden all
    python -m paper_2108_12574_b200 golden spectrum-2d iterations-2d

Each case is built exactly as cli.py builds it (default lattice, exact
backend with dense_limit = N) and checked with the suite's tolerance:
dense spectra through preconditioned_spectrum (spectrum.py:48-73),
lambda_min through Lanczos with mirrored sharing (cli.py:249-263), PCG
iteration counts (cli.py:266-283) and the two-halves Jacobi pairing
(cli.py:286-291).  Output lines and exit codes are the reference's.  The
suites ship as package data (data/goldens.json: the reference's own
goldens.json, which it ships the same way, pkg/pyproject.toml:24-25)."""

from __future__ import annotations

import json
import os

from . import geometry, kernel, pcg, precond, spectrum
from .linalg import NotPositiveDefinite
from .toeplitz import ToeplitzMatvec

EXIT_OK = 0
EXIT_CONFIG = 1
EXIT_NUMERICAL = 2
EXIT_GOLDEN = 3

DEFAULT_GOLDENS = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data", "goldens.json")


class ConfigError(ValueError):
    pass


def load_goldens(path: str | None = None) -> dict:
    path = path or os.environ.get("IEDD_GOLDENS", DEFAULT_GOLDENS)
    try:
        with open(path) as fh:
            return json.load(fh)
    except OSError as exc:
        raise ConfigError(f"missing golden file {path}") from exc


def _op(case):
    return kernel.build_operator(geometry.build_grid(case["dim"], case["n"]))


def _spectrum_case(suite, case):
    op = _op(case)
    dec = geometry.build_decomposition(op.grid, case["m"], case["overlap"], case["kind"])
    pre = precond.from_decomposition(op, dec, backend="exact", dense_limit=op.n)
    rep = spectrum.preconditioned_spectrum(op, pre, dense_limit=op.n)
    tol = suite["tol"]
    ok, msgs = True, []
    for key, got in (("lambda_max", rep.lambda_max), ("lambda_min", rep.lambda_min)):
        if key in case:
            err = abs(got - case[key])
            ok &= err <= tol
            msgs.append(f"{key}={got:.4f} (want {case[key]:.4f}, err {err:.1e})")
    return ok, ", ".join(msgs)


def _lanczos_case(suite, case):
    op = _op(case)
    dec = geometry.build_decomposition(op.grid, case["m"], case["overlap"], case["kind"])
    pre = precond.from_decomposition(op, dec, backend="exact", dense_limit=op.n, share_mirrored_subdomains=True)
    lam = spectrum.extremal_eigenvalue_lanczos(ToeplitzMatvec(op), pre, op.n, which="min")
    err = abs(lam - case["lambda_min"])
    return err <= suite["tol"], f"lambda_min={lam:.4f} (want {case['lambda_min']:.4f}, err {err:.1e})"


def _solve_case(suite, case):
    op = _op(case)
    mv = ToeplitzMatvec(op)
    dec = geometry.build_decomposition(op.grid, case["m"], case["overlap"], case["kind"])
    pre = precond.from_decomposition(op, dec, backend="exact", dense_limit=op.n)
    f, _ = pcg.make_rhs(mv, op.n, mode=suite.get("rhs", "random"), seed=suite.get("seed", 0))
    _, rep = pcg.solve(mv, pre, f, tol=suite.get("tol", 1e-12))
    diff = abs(rep.n_it - case["n_it"])
    return diff <= suite["tol_iters"] and rep.converged, f"n_it={rep.n_it} (want {case['n_it']} +-{suite['tol_iters']})"


def _pairing_case(suite, case):
    grid = geometry.build_grid(case["dim"], case["n"])
    op = kernel.build_operator(grid, lattice="cell")
    defect = spectrum.jacobi_pairing_check(op, geometry.two_halves_decomposition(grid))
    return defect <= suite["tol"], f"pairing defect {defect:.2e}"


RUNNERS = {"spectrum": _spectrum_case, "lanczos-min": _lanczos_case, "solve": _solve_case,
           "pairing": _pairing_case}


def run_golden(suite_names, path: str | None = None, out=print) -> int:
    goldens = load_goldens(path)
    suite_names = list(suite_names or [])
    if not suite_names:
        raise ConfigError("no golden suite named; available: " + ", ".join(sorted(goldens)))
    if suite_names == ["all"]:
        suite_names = sorted(goldens)
    failures = 0
    for name in suite_names:
        if name not in goldens:
            raise ConfigError(f"unknown golden suite {name!r}; available: " + ", ".join(sorted(goldens)))
        suite = goldens[name]
        runner = RUNNERS[suite["check"]]
        for case in suite["cases"]:
            try:
                ok, msg = runner(suite, case)
            except (NotPositiveDefinite, RuntimeError, ValueError) as exc:
                ok, msg = False, f"error: {exc}"
            label = " ".join(f"{k}={v}" for k, v in case.items())
            out(f"[{'PASS' if ok else 'FAIL'}] {name}: {label}: {msg}")
            failures += 0 if ok else 1
    out(f"golden: {failures} failure(s)")
    return EXIT_GOLDEN if failures else EXIT_OK
