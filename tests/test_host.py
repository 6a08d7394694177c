"""CPU-only tests: the C-ABI library loads and exports every symbol the
header declares (no compute calls), the host-side API mirrors the reference
(geometry, metadata, error messages), against the oracle and the golden
fixtures."""

import ctypes
import os
import re

import numpy as np
import pytest

from oracle import iedd_oracle as O

from .conftest import ROOT

HEADER = os.path.join(ROOT, "include", "iedd_b200.h")


def _declared():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|void|int64_t|const char\*)\s+\**(ie_\w+)\s*\(", text, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2108_12574_b200 import _lib
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2108_12574_b200 import build
        build.build()
    return _lib


class TestCABI:
    def test_header_declares_entry_points(self):
        names = _declared()
        for must in ("ie_matvec_create", "ie_matvec_f64", "ie_precond_create", "ie_precond_apply_f64",
                     "ie_pcg_f64", "ie_lanczos_f64", "ie_assemble_block_f64"):
            assert must in names

    def test_library_exports_every_declared_symbol(self, lib):
        so = ctypes.CDLL(lib.LIB_PATH)
        for name in _declared():
            assert hasattr(so, name), name

    def test_binding_signatures_cover_header(self, lib):
        assert set(_declared()) <= set(lib._SIGS)

    def test_no_compute_without_device_error_path(self, lib):
        # argument validation is host-only: a NULL geometry is rejected without touching the GPU
        L = lib.lib()
        h = ctypes.c_void_p()
        assert L.ie_matvec_create_method(None, 0, ctypes.byref(h)) == lib.IE_ERR_ARG
        assert "bad geometry" in lib.last_error()
        assert L.ie_launch_count() >= 0

    def test_sm100a_cubin(self, lib):
        import subprocess
        out = subprocess.run(["cuobjdump", "--list-elf", lib.LIB_PATH], capture_output=True, text=True).stdout
        assert "sm_100a" in out


class TestGeometryMirror:
    @pytest.mark.parametrize("dim,n,m,w", [(2, 32, 4, 1), (2, 12, 3, 2), (3, 8, 2, 1), (1, 16, 4, 2),
                                           (2, 256, 32, 2), (3, 32, 4, 1)])
    @pytest.mark.parametrize("kind", ["jacobi", "schwarz"])
    def test_vs_oracle(self, dim, n, m, w, kind):
        import paper_2108_12574_b200 as ie
        a = ie.build_decomposition(ie.build_grid(dim, n), m, w, kind).subdomains
        b = O.build_decomposition(O.build_grid(dim, n), m, w, kind).subdomains
        assert len(a) == len(b) and all(np.array_equal(x, y) for x, y in zip(a, b))

    def test_errors(self):
        import paper_2108_12574_b200 as ie
        with pytest.raises(ValueError, match="divide"):
            ie.build_partitioning(ie.build_grid(2, 16), 3)
        with pytest.raises(ValueError, match="kind"):
            ie.build_decomposition(ie.build_grid(2, 8), 2, 1, "multigrid")
        with pytest.raises(ValueError):
            ie.build_grid(4, 8)
        with pytest.raises(ValueError):
            ie.build_grid(2, 1)

    def test_grid_points_and_index_roundtrip(self):
        import paper_2108_12574_b200 as ie
        g = ie.build_grid(2, 2)
        assert {tuple(p) for p in g.points} == {(0.25, 0.25), (0.25, 0.75), (0.75, 0.25), (0.75, 0.75)}
        g3 = ie.build_grid(3, 6)
        for idx in (0, 5, 37, 215):
            assert g3.index_of(g3.multi_of(idx)) == idx

    def test_cbd_index_sets(self):
        import paper_2108_12574_b200 as ie
        d = ie.build_decomposition(ie.build_grid(2, 16), 4, 1, "cbd")
        assert d.n_subdomains == 4
        assert np.array_equal(np.unique(np.concatenate(d.subdomains)), np.arange(256))
        from oracle import iedd_oracle as O
        for dim, n, m, w in ((2, 16, 4, 1), (2, 12, 3, 2), (3, 8, 4, 1), (2, 64, 16, 1)):
            a = ie.build_decomposition(ie.build_grid(dim, n), m, w, "cbd").subdomains
            b = O.build_decomposition(O.build_grid(dim, n), m, w, "cbd").subdomains
            assert len(a) == len(b) == 2 ** dim
            assert all(np.array_equal(x, y) for x, y in zip(a, b))

    def test_two_halves(self):
        import paper_2108_12574_b200 as ie
        d = ie.two_halves_decomposition(ie.build_grid(2, 8))
        assert [s.size for s in d.subdomains] == [32, 32]


class TestOperatorMetadata:
    def test_diagonal_vs_reference_fixtures(self, golden):
        import paper_2108_12574_b200 as ie
        g = golden("ref_small")
        for key, val in g.items():
            if key.startswith("diag_"):
                _, dim, h = key.split("_")
                assert ie.diagonal_entry(int(dim), float(h)) == pytest.approx(float(val), rel=1e-14)

    def test_lattices(self):
        import paper_2108_12574_b200 as ie
        assert ie.build_operator(ie.build_grid(2, 8)).lattice == "span"
        assert ie.build_operator(ie.build_grid(3, 4)).lattice == "cell"
        assert ie.build_operator(ie.build_grid(2, 8)).lattice_spacing == pytest.approx(1 / 7)
        op = ie.build_operator(ie.build_grid(2, 8), lattice="cell")
        assert op.lattice_spacing == pytest.approx(1 / 8) and op.weight == 1 / 64
        with pytest.raises(ValueError):
            ie.build_operator(ie.build_grid(2, 8), lattice="torus")

    def test_value_object(self):
        import paper_2108_12574_b200 as ie
        op = ie.build_operator(ie.build_grid(2, 4))
        with pytest.raises(AttributeError):
            op.diag_value = 1.0

    def test_kernel_value(self):
        import paper_2108_12574_b200 as ie
        assert ie.kernel_value(np.array([1.0, 0.0])) == 0.0
        assert ie.kernel_value(np.array([0.0, 0.25, 0.0])) == pytest.approx(1 / np.pi, rel=1e-15)
        with pytest.raises(ValueError, match="singular"):
            ie.kernel_value(np.zeros(2))

    def test_make_rhs_modes_host(self):
        import paper_2108_12574_b200 as ie
        f, u = ie.make_rhs(lambda v: 2 * v, 8, mode="random", seed=1)
        assert np.array_equal(f, 2 * np.random.default_rng(1).standard_normal(8))
        f, u = ie.make_rhs(None, 8, mode="noise", seed=1)
        assert u is None and np.array_equal(f, np.random.default_rng(1).standard_normal(8))
        with pytest.raises(ValueError):
            ie.make_rhs(None, 8, mode="chebyshev")

    def test_backend_errors_before_device(self):
        import paper_2108_12574_b200 as ie
        grid = ie.build_grid(2, 16)
        op = ie.build_operator(grid)
        d = ie.build_decomposition(grid, 2, 1, "schwarz")
        with pytest.raises(ValueError, match="backend"):
            ie.from_decomposition(op, d, backend="qr")
        with pytest.raises(ValueError, match="rskel"):
            ie.from_decomposition(op, d, dense_limit=10)


class TestGoldenCli:
    """The golden subcommand's argument handling (cli.py:302-327, 363-390);
    the suites themselves run on the GPU (test_gpu_parity.TestGoldenRunner)."""

    def test_config_errors(self, capsys):
        from paper_2108_12574_b200.__main__ import main
        assert main(["golden"]) == 1
        assert "no golden suite named" in capsys.readouterr().err
        assert main(["golden", "nope"]) == 1
        err = capsys.readouterr().err
        assert "unknown golden suite 'nope'" in err and "interface-3d" in err
        assert main(["bogus"]) == 1

    def test_suites_present(self):
        from paper_2108_12574_b200 import golden
        g = golden.load_goldens()
        assert {"spectrum-2d", "spectrum-3d", "schwarz-scaling-2d", "interface-2d", "interface-3d",
                "iterations-2d", "iterations-3d", "pairing"} <= set(g)
        assert set(s["check"] for s in g.values()) == set(golden.RUNNERS)
