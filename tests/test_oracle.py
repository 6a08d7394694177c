"""Pins the CPU oracle (oracle/iedd_oracle.py) before anything is checked
against it: the reference's own known-answer constants, its golden suites
(goldens.json) and golden vectors frozen from the unmodified reference by
tools/gen_goldens.py.  CPU only."""

import json
import os

import numpy as np
import pytest

from oracle import iedd_oracle as O

from .conftest import GOLDEN

# reference tests/test_kernel.py:16-18
DIAG_2D_UNIT = 0.1688913146760059020024
DIAG_3D_UNIT = 0.1894005387092370500171
DIAG_1D_UNIT = 0.2694727431682211324671


def _suites():
    with open(os.path.join(GOLDEN, "..", "..", "paper_2108_12574_b200", "data", "goldens.json")) as fh:
        return json.load(fh)


class TestKnownAnswers:
    def test_diagonal_constants(self):
        assert O.diagonal_entry(2, 1.0) == pytest.approx(DIAG_2D_UNIT, abs=1e-13)
        assert O.diagonal_entry(3, 1.0) == pytest.approx(DIAG_3D_UNIT, abs=1e-13)
        assert O.diagonal_entry(1, 1.0) == pytest.approx(DIAG_1D_UNIT, abs=1e-13)

    @pytest.mark.parametrize("h", [1.0, 0.5, 0.125, 1 / 1024])
    def test_2d_closed_form(self, h):
        # reference tests/test_kernel.py:21-23 (== BASELINE.json diagonal rule)
        closed = h * h * (-np.log(h) + np.log(2.0) / 2 + (6 - np.pi) / 4) / (2 * np.pi)
        assert O.diagonal_entry(2, h) == pytest.approx(closed, rel=1e-12)

    def test_3d_baseline_rule(self):
        h = 1 / 32
        assert O.diagonal_entry(3, h) == pytest.approx(h * h * 2.3800774 / (4 * np.pi), rel=1e-7)

    def test_cell_2x2_entry(self):
        # reference tests/test_kernel.py:91-99
        a = O.build_operator(O.build_grid(2, 2), "cell").dense()
        assert a[0, 1] == pytest.approx(0.25 * np.log(2.0) / (2 * np.pi), rel=1e-14)
        assert a[0, 1] == pytest.approx(0.0275794, abs=1e-7)

    def test_baseline_offdiag_formula(self):
        # BASELINE.json config 1: A_ij = -(h^2/2pi) log|x_i - x_j| on the cell lattice
        op = O.build_operator(O.build_grid(2, 32), "cell")
        a = op.dense()
        h = 1 / 32
        pts = (op.grid.multi_indices() + 0.5) * h
        i, j = 5, 700
        d = np.linalg.norm(pts[i] - pts[j])
        assert a[i, j] == pytest.approx(-(h * h / (2 * np.pi)) * np.log(d), rel=1e-13)

    def test_default_lattices(self):
        assert O.build_operator(O.build_grid(2, 8)).lattice == "span"
        assert O.build_operator(O.build_grid(3, 4)).lattice == "cell"


class TestGoldenVectors:
    def test_diagonals(self, golden):
        g = golden("ref_small")
        for key, val in g.items():
            if key.startswith("diag_"):
                _, dim, h = key.split("_")
                assert O.diagonal_entry(int(dim), float(h)) == pytest.approx(float(val), rel=1e-14)

    @pytest.mark.parametrize("case", ["2_8_span", "2_32_span", "2_16_cell", "3_8_cell", "1_16_cell",
                                      "2_32_cell", "3_4_cell", "2_12_cell", "2_10_span"])
    def test_matvec(self, golden, case):
        g = golden("ref_small")
        dim, n, lat = case.split("_")
        op = O.build_operator(O.build_grid(int(dim), int(n)), lat)
        x = g[f"mv_{case}_x"]
        assert np.array_equal(op.dense()[0], g[f"mv_{case}_row0"])
        y = O.FFTMatvec(op).matvec(x)
        ref = g[f"mv_{case}_y"]
        assert np.linalg.norm(y - ref) <= 1e-14 * np.linalg.norm(ref)
        assert np.linalg.norm(op.dense() @ x - g[f"mv_{case}_ydense"]) <= 1e-14 * np.linalg.norm(ref)

    @pytest.mark.parametrize("case", ["2_32_4_1_schwarz_cell", "2_32_4_1_jacobi_cell",
                                      "2_16_2_1_schwarz_span", "3_8_2_1_schwarz_cell",
                                      "2_64_8_2_schwarz_cell", "2_12_3_1_schwarz_cell"])
    def test_apply(self, golden, case):
        g = golden("ref_small")
        dim, n, m, w, kind, lat = case.split("_")
        grid = O.build_grid(int(dim), int(n))
        op = O.build_operator(grid, lat)
        pre = O.SchwarzPrecond(op, O.build_decomposition(grid, int(m), int(w), kind))
        z = pre.apply(g[f"ap_{case}_r"])
        assert np.array_equal(z, g[f"ap_{case}_z"])
        if case.startswith("2_32_4_1_schwarz"):
            for b in (0, 5):
                assert np.array_equal(pre.factors[b], g[f"ap_{case}_G{b}"])

    @pytest.mark.parametrize("name", ["t16_jacobi_random", "t16_schwarz_random", "g16_jacobi_noise",
                                      "g16_schwarz_noise", "g8_3d_jacobi_noise", "g8_3d_schwarz_noise",
                                      "stag8_schwarz", "cap16_jacobi"])
    def test_small_pcg(self, golden, name):
        g = golden("ref_pcg_small")
        spec = {
            "t16_jacobi_random": (2, 16, 2, 1, "jacobi", 1e-12, None),
            "t16_schwarz_random": (2, 16, 2, 1, "schwarz", 1e-12, None),
            "g16_jacobi_noise": (2, 16, 2, 1, "jacobi", 1e-12, None),
            "g16_schwarz_noise": (2, 16, 2, 1, "schwarz", 1e-12, None),
            "g8_3d_jacobi_noise": (3, 8, 2, 1, "jacobi", 1e-12, None),
            "g8_3d_schwarz_noise": (3, 8, 2, 1, "schwarz", 1e-12, None),
            "stag8_schwarz": (2, 8, 2, 1, "schwarz", 1e-30, 5000),
            "cap16_jacobi": (2, 16, 2, 1, "jacobi", 1e-12, 5),
        }[name]
        dim, n, m, w, kind, tol, mi = spec
        grid = O.build_grid(dim, n)
        op = O.build_operator(grid)
        pre = O.SchwarzPrecond(op, O.build_decomposition(grid, m, w, kind))
        u, rep = O.pcg(O.FFTMatvec(op), pre, g[name + "_f"], tol=tol, max_iters=mi)
        n_it, conv, stag = g[name + "_meta"]
        # same algorithm, same numpy/scipy: bitwise identical
        assert rep.n_it == n_it and rep.converged == bool(conv) and rep.stagnated == bool(stag)
        assert np.array_equal(np.array(rep.residual_history), g[name + "_hist"])
        assert np.array_equal(u, g[name + "_u"])

    def test_c1_pcg(self, golden):
        g = golden("ref_c1")
        grid = O.build_grid(2, 32)
        op = O.build_operator(grid, "cell")
        f = np.random.default_rng(0).standard_normal(op.n)
        for kind in ("schwarz", "jacobi"):
            pre = O.SchwarzPrecond(op, O.build_decomposition(grid, 4, 1, kind))
            u, rep = O.pcg(O.FFTMatvec(op), pre, f, tol=1e-10)
            assert rep.n_it == g[f"{kind}_meta"][0]
            assert np.array_equal(np.array(rep.residual_history), g[f"{kind}_hist"])
            assert np.array_equal(u, g[f"{kind}_u"])
        assert g["schwarz_meta"][0] == 24 and g["jacobi_meta"][0] == 78

    def test_c2_lanczos(self, golden):
        g = golden("ref_c2")
        grid = O.build_grid(2, 64)
        op = O.build_operator(grid, "cell")
        mv = O.FFTMatvec(op)
        for kind in ("schwarz", "jacobi"):
            pre = O.SchwarzPrecond(op, O.build_decomposition(grid, 8, 1, kind))
            for which in ("min", "max"):
                lam = O.lanczos_extremal(mv, pre, op.n, which=which, max_iters=300)
                assert lam == pytest.approx(float(g[f"lam_{kind}_{which}"][0]), rel=1e-13)

    def test_small_lanczos_vs_dense(self, golden):
        g = golden("ref_lanczos_small")
        for name, (dim, n, m, kind, which) in {"j16max": (2, 16, 2, "jacobi", "max"),
                                                "s16min": (2, 16, 4, "schwarz", "min"),
                                                "s8_3dmin": (3, 8, 2, "schwarz", "min")}.items():
            grid = O.build_grid(dim, n)
            op = O.build_operator(grid)
            pre = O.SchwarzPrecond(op, O.build_decomposition(grid, m, 1, kind))
            lam = O.lanczos_extremal(O.FFTMatvec(op), pre, op.n, which=which)
            lam_ref, _, dmin, dmax = g[name]
            assert lam == pytest.approx(lam_ref, rel=1e-13)
            w = O.dense_spectrum(op, pre)
            assert w[0] == pytest.approx(dmin, rel=1e-10) and w[-1] == pytest.approx(dmax, rel=1e-10)


class TestReferenceGoldenSuites:
    """goldens.json suites on the hot path (jacobi / schwarz / cbd rows)."""

    @pytest.mark.parametrize("suite,case", [
        (name, c) for name in ("spectrum-2d", "spectrum-3d", "schwarz-scaling-2d")
        for c in _suites()[name]["cases"]],
        ids=lambda x: x if isinstance(x, str) else f"{x['dim']}d_n{x['n']}_m{x['m']}_{x['kind']}")
    def test_spectrum_suites(self, suite, case):
        if case["n"] ** case["dim"] > 1024 and not os.environ.get("IEDD_SLOW"):
            pytest.skip("dense N=4096 eigensolve: set IEDD_SLOW=1")
        tol = _suites()[suite]["tol"]
        grid = O.build_grid(case["dim"], case["n"])
        op = O.build_operator(grid)
        dec = O.build_decomposition(grid, case["m"], case["overlap"], case["kind"])
        w = O.dense_spectrum(op, O.SchwarzPrecond(op, dec))
        assert abs(w[-1] - case["lambda_max"]) <= tol
        assert abs(w[0] - case["lambda_min"]) <= tol

    def test_iteration_suites(self):
        suites = _suites()
        for name in ("iterations-2d", "iterations-3d"):
            s = suites[name]
            for case in s["cases"]:
                if case["kind"] == "cbd":
                    continue  # TestCBD: goldens.json's 3D CBD n_it is stale (the reference gives 22/21)
                grid = O.build_grid(case["dim"], case["n"])
                op = O.build_operator(grid)
                mv = O.FFTMatvec(op)
                pre = O.SchwarzPrecond(op, O.build_decomposition(grid, case["m"], case["overlap"],
                                                                 case["kind"]))
                f, _ = O.make_rhs(mv, op.n, mode=s["rhs"], seed=s["seed"])
                _, rep = O.pcg(mv, pre, f, tol=s["tol"])
                assert rep.converged and abs(rep.n_it - case["n_it"]) <= s["tol_iters"]

    def test_pairing_suite(self):
        # goldens.json "pairing": two-halves Jacobi split on the cell lattice
        for case in _suites()["pairing"]["cases"]:
            grid = O.build_grid(case["dim"], case["n"])
            op = O.build_operator(grid, "cell")
            mi = grid.multi_indices()
            halves = [np.nonzero(mi[:, 0] < case["n"] // 2)[0], np.nonzero(mi[:, 0] >= case["n"] // 2)[0]]
            dec = O.Decomposition("jacobi", grid, 2, 0, halves)
            w = O.dense_spectrum(op, O.SchwarzPrecond(op, dec, dense_limit=op.n))
            assert np.max(np.abs(w + w[::-1] - 2.0)) <= 1e-8


@pytest.mark.skipif(not os.path.isdir("/root/reference/pkg/src"), reason="reference only in build container")
def test_oracle_vs_live_reference_geometry():
    import sys
    sys.path.insert(0, "/root/reference/pkg/src")
    from iedd import geometry
    for dim, n, m, w in [(2, 32, 4, 1), (2, 12, 3, 2), (3, 8, 2, 1), (1, 16, 4, 2)]:
        for kind in ("jacobi", "schwarz"):
            a = geometry.build_decomposition(geometry.build_grid(dim, n), m, w, kind).subdomains
            b = O.build_decomposition(O.build_grid(dim, n), m, w, kind).subdomains
            assert len(a) == len(b) and all(np.array_equal(x, y) for x, y in zip(a, b))


def _cbd_meta():
    with open(os.path.join(GOLDEN, "ref_cbd.json")) as fh:
        return json.load(fh)


class TestCBD:
    """Colour-block-diagonal rows (geometry.py:164-176, 227-235) against the
    reference run itself (tools/gen_goldens.py --only cbd -> ref_cbd.*)."""

    def test_solve_rows(self):
        g = dict(np.load(os.path.join(GOLDEN, "ref_cbd.npz")))
        for case in _cbd_meta():
            if "n_it_ref" not in case or case["n"] ** case["dim"] > 1024:
                continue
            grid = O.build_grid(case["dim"], case["n"])
            op = O.build_operator(grid)
            mv = O.FFTMatvec(op)
            pre = O.SchwarzPrecond(op, O.build_decomposition(grid, case["m"], case["overlap"], "cbd"))
            r = np.random.default_rng(7).standard_normal(op.n)
            z = g["z_" + case["key"]]
            assert np.linalg.norm(pre.apply(r) - z) <= 1e-12 * np.linalg.norm(z)
            f, _ = O.make_rhs(mv, op.n, mode="noise", seed=0)
            u, rep = O.pcg(mv, pre, f, tol=1e-12)
            assert rep.converged and rep.n_it == case["n_it_ref"], case
            assert np.linalg.norm(u - g["u_" + case["key"]]) <= 1e-10 * np.linalg.norm(u)

    def test_stale_golden_rows(self):
        # the reference's own goldens.json lists n_it 27 for both 3D CBD rows;
        # the reference computes 22 and 21 (outside its +-2), so parity is
        # anchored on the reference run, not that number
        rows = {c["key"]: c for c in _cbd_meta() if "n_it_ref" in c}
        assert rows["3d_n8_m4"]["n_it"] == 27 and rows["3d_n8_m4"]["n_it_ref"] == 22
        assert rows["3d_n16_m8"]["n_it_ref"] == 21

    def test_lanczos_rows_vs_suite(self):
        for case in _cbd_meta():
            if "lanczos_min" in case:
                assert abs(case["lanczos_min"] - case["lambda_min"]) <= 2e-3
                assert abs(case["lanczos_max"] - case["lambda_max"]) <= 2e-3
