"""Sharded PCG host logic on CPU: world-size 1/2/3 over gloo with the oracle
backend must give bitwise-identical reports and solutions, and the plan must
cover the unknowns with chunk-aligned bands."""

import json
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2108_12574_b200 import geometry as G
from paper_2108_12574_b200.distributed import (CHUNK, Comm, band_bounds, blocks_intersecting, lanczos_sharded,
                                               make_plan, solve_sharded)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


CASE = dict(dim=2, n=128, m=16, w=2, kind="schwarz", lattice="cell", seed=4)


def _worker(rank, world, port, out_dir, case):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from tests.dist_cpu_backend import OracleBackend
        grid = G.build_grid(case["dim"], case["n"])
        dec = G.build_decomposition(grid, case["m"], case["w"], case["kind"])
        plan = make_plan(grid, dec, world, rank)
        be = OracleBackend(case["dim"], case["n"], case["m"], case["w"], case["kind"], case["lattice"], plan,
                           dist_fft=case.get("dist_fft", False))
        if case.get("dist_fft"):
            assert be.band is not None
        f = np.random.default_rng(case["seed"]).standard_normal(grid.n_points)
        u, rep = solve_sharded(be, Comm(plan), plan, be.tensor(f[plan.begin: plan.end]), tol=1e-10,
                               max_iters=case.get("max_iters"))
        np.savez(os.path.join(out_dir, f"r{rank}.npz"), u=u.numpy(), hist=np.array(rep.residual_history),
                 meta=np.array([rep.n_it, rep.converged, rep.stagnated]))
    finally:
        dist.destroy_process_group()


def _lz_worker(rank, world, port, out_dir, case):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from tests.dist_cpu_backend import OracleBackend
        grid = G.build_grid(case["dim"], case["n"])
        dec = G.build_decomposition(grid, case["m"], case["w"], case["kind"])
        plan = make_plan(grid, dec, world, rank)
        be = OracleBackend(case["dim"], case["n"], case["m"], case["w"], case["kind"], case["lattice"], plan,
                           dist_fft=True)
        out = []
        for which in ("min", "max"):
            lam, steps = lanczos_sharded(be, Comm(plan), plan, which=which, max_iters=case["max_iters"],
                                         return_steps=True)
            out += [lam, steps]
        np.save(os.path.join(out_dir, f"r{rank}.npy"), np.array(out))
    finally:
        dist.destroy_process_group()


def _run_lz(world, case):
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_lz_worker, args=(world, _free_port(), d, case), nprocs=world, join=True)
        return [np.load(os.path.join(d, f"r{r}.npy")) for r in range(world)]


def _run(world, case):
    with tempfile.TemporaryDirectory() as d:
        mp.spawn(_worker, args=(world, _free_port(), d, case), nprocs=world, join=True)
        return [dict(np.load(os.path.join(d, f"r{r}.npz"))) for r in range(world)]


class TestPlan:
    @pytest.mark.parametrize("dim,n,m,world", [(2, 1024, 128, 8), (2, 256, 32, 4), (2, 128, 16, 3),
                                               (3, 32, 4, 2), (2, 32, 4, 2)])
    def test_bands(self, dim, n, m, world):
        grid = G.build_grid(dim, n)
        b = band_bounds(grid, m, world)
        assert b[0] == 0 and b[-1] == grid.n_points and all(x <= y for x, y in zip(b, b[1:]))
        assert all(x % CHUNK == 0 for x in b[:-1])
        if (dim, n, world) == (2, 1024, 8):
            assert b == tuple(131072 * g for g in range(9))   # 16 subdomain rows per rank

    def test_blocks_cover_band(self):
        grid = G.build_grid(2, 128)
        dec = G.build_decomposition(grid, 16, 2, "schwarz")
        for world in (2, 3):
            for r in range(world):
                plan = make_plan(grid, dec, world, r)
                covered = np.zeros(grid.n_points, bool)
                for k in plan.blocks:
                    covered[dec.subdomains[k]] = True
                assert covered[plan.begin: plan.end].all()
                # every block touching the band is included (z is complete on the band)
                assert np.array_equal(plan.blocks, blocks_intersecting(dec.subdomains, plan.begin, plan.end))


class TestShardedSolve:
    def test_world_sizes_bitwise_equal_and_oracle_parity(self):
        from oracle import iedd_oracle as O
        res = {w: _run(w, CASE) for w in (1, 2, 3)}
        ref = res[1][0]
        for w in (2, 3):
            for r in range(w):
                assert np.array_equal(res[w][r]["hist"], ref["hist"])
                assert np.array_equal(res[w][r]["u"], ref["u"])
                assert np.array_equal(res[w][r]["meta"], ref["meta"])
        grid = O.build_grid(2, 128)
        op = O.build_operator(grid, "cell")
        pre = O.SchwarzPrecond(op, O.build_decomposition(grid, 16, 2, "schwarz"))
        f = np.random.default_rng(CASE["seed"]).standard_normal(op.n)
        u, rep = O.pcg(O.FFTMatvec(op), pre, f, tol=1e-10)
        assert abs(int(ref["meta"][0]) - rep.n_it) <= 1
        assert np.linalg.norm(ref["u"] - u) <= 1e-10 * np.linalg.norm(u)

    def test_distributed_fft_transposes(self):
        """BandFFT (row FFTs, all-to-all to column slabs, column pass, reverse
        all-to-all, inverse rows) over gloo at world sizes 1, 2, 4: bitwise
        identical runs, oracle parity."""
        from oracle import iedd_oracle as O
        case = dict(CASE, dist_fft=True)
        res = {w: _run(w, case) for w in (1, 2, 4)}
        ref = res[1][0]
        for w in (2, 4):
            for r in range(w):
                assert np.array_equal(res[w][r]["hist"], ref["hist"])
                assert np.array_equal(res[w][r]["u"], ref["u"])
        grid = O.build_grid(2, 128)
        op = O.build_operator(grid, "cell")
        pre = O.SchwarzPrecond(op, O.build_decomposition(grid, 16, 2, "schwarz"))
        f = np.random.default_rng(CASE["seed"]).standard_normal(op.n)
        u, rep = O.pcg(O.FFTMatvec(op), pre, f, tol=1e-10)
        # the 2-RHS packed band FFT rounds differently from pocketfft: n_it must lie in the reference's
        # own one-ulp envelope for this case (tests/golden/nit_envelope.json, tools/nit_envelope.py)
        with open(os.path.join(os.path.dirname(__file__), "golden", "nit_envelope.json")) as fh:
            env = json.load(fh)["gloo_n128_m16_w2_seed4"]
        assert env["reference"] == rep.n_it
        assert min(env["min"], rep.n_it - 1) <= int(ref["meta"][0]) <= max(env["max"], rep.n_it + 1)
        assert np.linalg.norm(ref["u"] - u) <= 1e-10 * np.linalg.norm(u)

    def test_band_fft_matvec_vs_oracle(self):
        """One BandFFT product at world size 1 against the oracle FFT matvec
        (both right-hand sides, p and u of very different magnitude)."""
        from oracle import iedd_oracle as O
        from tests.dist_cpu_backend import OracleBackend

        from paper_2108_12574_b200.distributed import ShardPlan

        class _Comm1:
            def alltoall(self, send, sc, rc):
                return send.clone()

            def allgather_partials(self, x):
                return x

        grid = G.build_grid(2, 64)
        dec = G.build_decomposition(grid, 8, 1, "schwarz")
        plan = ShardPlan(world=1, rank=0, N=grid.n_points, bounds=(0, grid.n_points),
                         blocks=np.arange(len(dec.subdomains)))
        be = OracleBackend(2, 64, 8, 1, "schwarz", "cell", plan, dist_fft=True)
        rng = np.random.default_rng(1)
        X = np.stack([rng.standard_normal(grid.n_points), 1e-9 * rng.standard_normal(grid.n_points)])
        from paper_2108_12574_b200.distributed import pow2_scale
        sc = (pow2_scale(float(np.abs(X[0]).max())), pow2_scale(float(np.abs(X[1]).max())))
        Y = be.band.matvec(_Comm1(), torch.from_numpy(X), sc).numpy()
        mv = O.FFTMatvec(O.build_operator(O.build_grid(2, 64), "cell"))
        for c in range(2):
            ref = mv.matvec(X[c])
            assert np.linalg.norm(Y[c] - ref) <= 1e-13 * np.linalg.norm(ref)

    def test_max_iters_exit(self):
        case = dict(CASE, max_iters=7)
        res = _run(2, case)
        assert int(res[0]["meta"][0]) == 7 and not res[0]["meta"][1]
        assert np.array_equal(res[0]["hist"], res[1]["hist"]) and len(res[0]["hist"]) == 8


class TestShardedLanczos:
    def test_world_sizes_bitwise_equal_and_oracle_parity(self):
        """Lanczos (spectrum.py:133-190) on the band decomposition over gloo:
        lambda_min / lambda_max and step counts identical for G = 1, 2, 4 and
        within 1e-8 of the oracle's Lanczos."""
        from oracle import iedd_oracle as O
        case = dict(dim=2, n=64, m=8, w=1, kind="schwarz", lattice="cell", max_iters=300)
        res = {w: _run_lz(w, case) for w in (1, 2, 4)}
        ref = res[1][0]
        for w in (2, 4):
            for r in range(w):
                assert np.array_equal(res[w][r], ref)
        grid = O.build_grid(2, 64)
        op = O.build_operator(grid, "cell")
        pre = O.SchwarzPrecond(op, O.build_decomposition(grid, 8, 1, "schwarz"))
        for k, which in enumerate(("min", "max")):
            lam = O.lanczos_extremal(O.FFTMatvec(op), pre, op.n, which=which, max_iters=300)
            assert abs(ref[2 * k] - lam) <= 1e-8 * abs(lam)
