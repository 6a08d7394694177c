"""Benchmark: Schwarz-PCG iterations/s on BASELINE.json config 5 (2D n=1024,
N=1,048,576, cell lattice, D=128x128 subdomains, 2-line overlap, f ~ N(0,1)
seed 3), plus the K1 direct-sum kernel's pair-evals/s against the measured
FP64 issue roofline.

A "step" is one PCG iteration of that 50-iteration run: one fused 2-RHS
A-pass over [p_k, u_{k-1}] (N^2 kernel pair evaluations), the dot products,
the vector updates and one Schwarz apply.  Timing follows the repo contract:
W untimed warm-up iterations, then exactly K iterations timed with CUDA
events on the launching stream (barrier + synchronize on both sides, max over
ranks).  Inputs (the 8 MB iterate vectors) are re-read from HBM each pass;
the per-step working set (factor pool + 10 vectors) exceeds the 126 MB L2
only without translation sharing, so the config records l2 "not flushed".

  python bench.py [--gpus N --steps K --warmup W]          # our arm
  python bench.py --impl reference [--steps K --warmup W]  # CPU oracle arm

Multi-GPU (torchrun, N > 1): rows and subdomains are sharded by
paper_2108_12574_b200.distributed (2D FFT over row bands with two NCCL
all-to-all transposes, r-halo exchange for the apply, all-gathered fixed-chunk
dot partials), plus the K1 direct sum on each rank's rows; see DESIGN.md.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Schwarz-PCG iter/s + kernel-matvec pair-evals/s (FP64) vs roofline, 1/2/4/8 GPU"
CFG = dict(dim=2, n=1024, m=128, w=2, seed=3)
WORKLOAD = "config5: 2D Laplace single-layer, n=1024 (N=1048576), cell lattice, Schwarz D=128x128 w=2, f~N(0,1) seed 3"
# FP64 instructions per pair in the 2-RHS inner loop: a kernel evaluation (8 FP64 instructions: DADD
# int->double, DFMA reduction, 5 Horner DFMA, DFMA) shared by the thread's 16 consecutive rows (ADJ
# window) + 2 DFMA (one per RHS) = 2.5 (SASS of k_matvec<2,2,8,true>: 92 DFMA + 4 DADD per 32 pairs = 3)
K1_FP64_PER_PAIR_2RHS = 2.5


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh)
    except OSError:
        return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                smax = float(parts[1])
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def config_keys(ws: int) -> dict:
    """The `config` object of the JSON line -- identical in both arms (ours
    and --impl reference) at the same N, so the driver can match them."""
    return {"workload": WORKLOAD, "N": CFG["n"] ** CFG["dim"], "subdomains": CFG["m"] ** CFG["dim"],
            "tol": 1e-10, "matvec": "circulant-embedding FFT (the reference's ToeplitzMatvec algorithm)",
            "l2": "not flushed: the per-iteration working set (10 N-vectors, 84 MB + FFT work buffer) "
                  "streams through HBM",
            "parallelism": "single GPU" if ws == 1 else f"row/subdomain bands x{ws}"}


def _time_iters(ie, mv, pre, f, iters, st):
    """Device time (ms) of exactly `iters` PCG iterations through ie.solve."""
    import torch
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    u, rep = ie.solve(mv, pre, f, tol=1e-10, max_iters=iters)
    e1.record(st)
    torch.cuda.synchronize()
    assert rep.n_it == iters, rep.n_it
    return e0.elapsed_time(e1), rep


def _time_calls(fn, reps, st):
    import torch
    fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def run_ours(args):
    import torch

    import paper_2108_12574_b200 as ie
    from paper_2108_12574_b200 import _lib

    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    if ws > 1 or os.environ.get("IEDD_FORCE_SHARDED"):
        import torch.distributed as dist
        if not dist.is_initialized():
            os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
            os.environ.setdefault("MASTER_PORT", "29511")
            os.environ.setdefault("RANK", str(rank))
            os.environ.setdefault("WORLD_SIZE", str(ws))
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        from paper_2108_12574_b200 import distributed as D
        return D.bench_sharded(args, METRIC, CFG, WORKLOAD, config_keys=config_keys(ws),
                               cpu_baseline=None if args.no_cpu else lambda: cpu_baseline(max(1, min(10, args.steps))))

    st = torch.cuda.current_stream()
    grid = ie.build_grid(CFG["dim"], CFG["n"])
    op = ie.build_operator(grid, lattice="cell")
    mv = ie.ToeplitzMatvec(op, method=args.matvec)        # production path (FFT unless --matvec direct)
    k1 = ie.KernelMatvec(op, method="direct")             # north-star K1 direct sum
    dec = ie.build_decomposition(grid, CFG["m"], CFG["w"], "schwarz")
    t0 = time.perf_counter()
    pre = ie.from_decomposition(op, dec, share_translated=not args.no_share)
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t0
    N = op.n
    # host input in pinned memory (the e2e contract: H2D from pinned host buffers)
    f_pinned = torch.empty(N, dtype=torch.float64, pin_memory=True)
    f_host = f_pinned.numpy()
    f_host[:] = np.random.default_rng(CFG["seed"]).standard_normal(N)
    f = torch.from_numpy(f_host).cuda()
    L = _lib.lib()
    peak_dfma = ctypes.c_double(0.0)
    _lib.check(L.ie_fp64_peak(ctypes.byref(peak_dfma), _lib.stream_ptr()), "fp64 peak")
    fp64_peak_tflops = 2.0 * peak_dfma.value / 1e12
    peaks = _peaks()

    # ---- primary: exactly K iterations after W warm-up iterations
    _time_iters(ie, mv, pre, f, max(args.warmup, 1), st)
    clocks = ClockSampler(local)
    clocks.start()
    n0 = _lib.launch_count()
    ms, rep = _time_iters(ie, mv, pre, f, args.steps, st)
    launches = _lib.launch_count() - n0

    # ---- per-kernel device times on the same stream
    X = torch.from_numpy(np.random.default_rng(9).standard_normal((2, N))).cuda()
    Y = torch.empty_like(X)
    mv_ms = _time_calls(lambda: mv.matvec_device(X, Y, nrhs=2), 20, st)
    r = torch.from_numpy(np.random.default_rng(10).standard_normal(N)).cuda()
    z = torch.empty_like(r)
    apply_ms = _time_calls(lambda: pre.apply_device(r, z), 50, st)
    # K1 direct sum (north-star kernel): 2-RHS pass, pair-evals/s vs FP64 issue roofline
    k1_ms = _time_calls(lambda: k1.matvec_device(X, Y, nrhs=2), 2, st)
    clk = clocks.stop()
    pairs = float(N) * float(N)
    pair_rate = pairs / (k1_ms * 1e-3)
    k1_tflops = pair_rate * K1_FP64_PER_PAIR_2RHS * 2 / 1e12
    k1_iters = max(1, min(3, args.steps))
    k1_step_ms, _ = _time_iters(ie, k1, pre, f, k1_iters, st)
    # end to end through the public API with host numpy buffers (median of 5), measured
    # after the nvidia-smi sampler has stopped (its driver queries stall CUDA calls)
    e2e_t = []
    for _ in range(5):
        t0 = time.perf_counter()
        u_h, rep_h = ie.solve(mv, pre, f_host, tol=1e-10, max_iters=args.steps)
        e2e_t.append(time.perf_counter() - t0)
    t_e2e = statistics.median(e2e_t)

    # ---- K3 apply with every block factorised (factors streamed from HBM): the HBM roofline
    apply_bytes = _apply_bytes(dec, N, False)
    noshare = {}
    if not args.skip_noshare:
        t0 = time.perf_counter()
        pre_ns = ie.from_decomposition(op, dec, share_translated=False)
        torch.cuda.synchronize()
        t_ns = time.perf_counter() - t0
        ns_ms = _time_calls(lambda: pre_ns.apply_device(r, z), 20, st)
        noshare = {"apply_ms": ns_ms, "achieved": apply_bytes / (ns_ms * 1e-3) / 1e9, "build_s": t_ns,
                   "factor_bytes": pre_ns.stats()["device_bytes"]}
        if peaks.get("hbm_gbs"):
            noshare["frac"] = noshare["achieved"] / peaks["hbm_gbs"]
        del pre_ns

    step_ms = ms / args.steps
    # ---- per-kernel device times inside the PCG iteration: a profiled solve
    # (ie_pcg_profile_f64: iterations launched one by one with CUDA events
    # between the kernel groups on the solver's stream), steady 2-RHS iterations
    ph = _profile_phases(ie, _lib, mv, pre, f, max(8, min(args.steps, 24)))
    kern = {"matvec_pass_ms": ph[0], "post_pass_ms": ph[1], "iter_a_ms": ph[2], "apply_ms": ph[3],
            "iter_b_ms": ph[4], "k4_vector_ms": ph[1] + ph[2] + ph[4],
            "standalone_matvec_pass_ms": mv_ms, "standalone_apply_ms": apply_ms}
    dmma = ctypes.c_double(0.0)
    _lib.check(L.ie_dmma_peak(ctypes.byref(dmma), _lib.stream_ptr()), "dmma peak")
    dmma_peak_tflops = dmma.value / 1e12
    traffic = _traffic()
    # K1b 2-RHS pass: n row FFTs forward, 2n column FFTs forward + inverse (fused), n row FFTs inverse,
    # each 5 M log2 M flops (M = 2n): the conventional complex-FFT count
    M = 2 * CFG["n"]
    lines = CFG["n"] + 2 * (2 * CFG["n"]) + CFG["n"]
    fft_flops = lines * 5.0 * M * np.log2(M)
    s2 = sum(float(sd.size) ** 2 for sd in dec.subdomains)
    s_sum = sum(sd.size for sd in dec.subdomains)
    hbm = peaks.get("hbm_gbs")
    rooflines = {
        "fft_pass": {"bound": "fp64", "kernel": "k_fft8 x3 (row fwd, fused column fwd*sym*inv, row inv)",
                     "achieved": fft_flops / (ph[0] * 1e-3) / 1e12, "unit": "TFLOP/s", "peak": fp64_peak_tflops,
                     "traffic": traffic.get("fft_pass"),
                     "note": "flops = 5 M log2 M per line FFT x 6n lines (M = 2n); peak = live 8-chain DFMA "
                             "microbenchmark (ie_fp64_peak); traffic = ncu dram bytes of the three launches"},
        "apply": {"bound": "fp64-tensor", "kernel": "k_apply_dmma2 (class GEMM on DMMA, gathers r) + k_scatter_fixed (+ the iteration's decider)",
                  "achieved": 2.0 * s2 / (ph[3] * 1e-3) / 1e12, "unit": "TFLOP/s", "peak": dmma_peak_tflops,
                  "traffic": traffic.get("apply"),
                  "note": f"flops = 2 sum_k s_k^2 (Sigma s = {s_sum}); peak = live DMMA m8n8k4 microbenchmark "
                          "(ie_dmma_peak)"},
        "k4_vectors": {"bound": "hbm", "kernel": "k_iter_a (r update, control) + k_update_u; the post pass and the p update ride in the FFT row passes",
                       "achieved": 80.0 * N / (kern["k4_vector_ms"] * 1e-3) / 1e9, "unit": "GB/s", "peak": hbm,
                       "traffic": traffic.get("k4_vectors"),
                       "note": "bytes = 80 N per iteration (SURVEY 8(d): read p, u, r, q, z, f, Au; write u, r, "
                               "p); the kernels move 104 N (q and p are read twice)"},
    }
    for r_ in rooflines.values():
        r_["frac"] = r_["achieved"] / r_["peak"] if r_.get("peak") else None
    shares = {"fft_pass": ph[0], "apply": ph[3], "k4_vectors": kern["k4_vector_ms"]}
    dom = max(shares, key=shares.get)
    roof = dict(rooflines[dom], dominant=dom, share_of_step=shares[dom] / step_ms)
    out = {
        "metric": METRIC,
        "value": args.steps / (ms * 1e-3),
        "unit": "iter/s",
        "n_gpus": 1,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": step_ms,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f64",
        "data": "synthetic (BASELINE.json config 5, seeded)",
        "config": config_keys(1),
        "details": {"matvec": f"{mv.method} ({'2 RHS per complex pass' if mv.method == 'fft' else 'K1 direct sum'})",
                    "share_translated": not args.no_share, "precond_build_s": t_build},
        "kernels_ms": kern,
        "roofline": roof,
        "rooflines": rooflines,
        "kernel_matvec": {
            "kernel": "k_matvec<2,2,16,ADJ> (K1 direct sum, log kernel evaluated on the fly, one evaluation "
                      "shared by 16 consecutive rows, 2 RHS)",
            "pair_evals_per_s": pair_rate, "pass_ms": k1_ms,
            "schwarz_pcg_iter_per_s": k1_iters / (k1_step_ms * 1e-3),
            # algorithmic roofline: every pair needs at least one DFMA per right-hand side (the log
            # evaluation is shared by 16 rows, so it is not charged): 2 DFMA = 4 flops per pair
            "roofline": {"bound": "fp64", "achieved": pair_rate * 4 / 1e12, "peak": fp64_peak_tflops,
                         "unit": "TFLOP/s", "frac": pair_rate * 4 / 1e12 / fp64_peak_tflops, "traffic": None,
                         "note": "flops = 4 per pair (the 2 DFMA a 2-RHS pair needs at least); peak = live 8-chain "
                                 "DFMA microbenchmark on all SMs; FP64 pipe issue (2.5 instructions per pair incl. "
                                 "the shared log evaluation) in issue_frac",
                         "issue_frac": k1_tflops / fp64_peak_tflops}},
        "apply_hbm_roofline_unshared": dict(noshare, bound="hbm", unit="GB/s", algorithmic_bytes=apply_bytes,
                                            peak=peaks.get("hbm_gbs"), kernel="k_apply_packed<5,2>"),
        "e2e": {"value": args.steps / t_e2e, "unit": "iter/s", "h2d_bytes_per_step": 8 * N / args.steps,
                "d2h_bytes_per_step": (8 * N + 8 * (args.steps + 1)) / args.steps,
                "note": "pcg.solve(numpy f in pinned memory) -> fresh numpy u, wall clock: "
                        "one H2D of f and one D2H of u (+ history) per solve of K steps"},
        "gpu_launches": launches,
        "clocks": clk,
    }
    if not args.no_configs:
        try:
            out["configs"] = _other_configs(ie)
        except Exception as e:  # the side block must never cost the bench line
            out["configs"] = {"error": f"{type(e).__name__}: {e}"}
    if not args.no_cpu:
        out["cpu_baseline"] = cpu_baseline(max(1, min(10, args.steps)))  # ~8 s of CPU work
    print(json.dumps(out))
    return out


def _other_configs(ie):
    """BASELINE.json's other configs (parity-test cases, not bench lines) through
    the drop-in API in the same run: converged PCG solves of c1 / c3 / c4 and
    the Lanczos lambda_min of c2 / c4 (best of 3 wall times after a warm-up
    call, the factorisation timed once), next to the iteration counts and
    t_pcg the unmodified reference recorded when the goldens were frozen
    (tools/gen_goldens.py, in the build container: other host, so context only)."""
    import torch
    gold = os.path.join(os.path.dirname(os.path.abspath(__file__)), "tests", "golden")

    def timed(fn, reps=3):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            r = fn()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        return min(ts), r

    res = {}
    for name, (dim, n, m, w, seed, kinds) in {"c1": (2, 32, 4, 1, 0, ("schwarz", "jacobi")),
                                              "c3": (2, 256, 32, 2, 1, ("schwarz",)),
                                              "c4": (3, 32, 4, 1, 2, ("schwarz",))}.items():
        grid = ie.build_grid(dim, n)
        op = ie.build_operator(grid, lattice="cell")
        mv = ie.ToeplitzMatvec(op)
        f = np.random.default_rng(seed).standard_normal(op.n)
        try:
            g = dict(np.load(os.path.join(gold, f"ref_{name}.npz")))
        except OSError:
            g = {}
        for kind in kinds:
            dec = ie.build_decomposition(grid, m, w, kind)
            ie.from_decomposition(op, dec)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            pre = ie.from_decomposition(op, dec)
            torch.cuda.synchronize()
            t_f = time.perf_counter() - t0
            t, (_, rep) = timed(lambda: ie.solve(mv, pre, f, tol=1e-10))
            row = {"n_it": rep.n_it, "converged": bool(rep.converged), "t_pcg_s": t, "t_build_s": t_f}
            if f"{kind}_meta" in g:
                row["reference_n_it"] = int(g[f"{kind}_meta"][0])
                row["reference_t_pcg_s"] = float(g[f"{kind}_times"][1])
            res[f"{name} {kind} pcg"] = row
    for name, (dim, n, m, w, kind, mi) in {"c2 schwarz": (2, 64, 8, 1, "schwarz", 300),
                                           "c2 jacobi": (2, 64, 8, 1, "jacobi", 300),
                                           "c4 schwarz": (3, 32, 4, 1, "schwarz", 200)}.items():
        grid = ie.build_grid(dim, n)
        op = ie.build_operator(grid, lattice="cell")
        mv = ie.ToeplitzMatvec(op)
        pre = ie.from_decomposition(op, ie.build_decomposition(grid, m, w, kind))
        t, (lam, steps) = timed(lambda: ie.extremal_eigenvalue_lanczos(mv, pre, op.n, which="min", max_iters=mi,
                                                                      return_steps=True))
        res[f"{name} lanczos lambda_min"] = {"lambda": lam, "steps": steps, "t_s": t}
    return res


def _profile_phases(ie, _lib, mv, pre, f, iters):
    """Mean device ms per steady-state iteration of [matvec, k_post_pass,
    k_iter_a, apply, k_iter_b] (ie_pcg_profile_f64)."""
    import torch
    u = torch.empty_like(f)
    hist = np.zeros(iters + 1)
    n_it = ctypes.c_int64(0)
    flags = np.zeros(2, dtype=np.int32)
    times = np.zeros(2)
    ph = np.zeros(5)
    _lib.check(_lib.lib().ie_pcg_profile_f64(mv.handle, pre.handle, _lib.ptr(f), _lib.ptr(u), 1e-10, iters,
                                             _lib.np_ptr(hist), ctypes.byref(n_it), _lib.np_ptr(flags),
                                             _lib.np_ptr(times), _lib.np_ptr(ph), _lib.stream_ptr()), "profile")
    return [float(x) for x in ph]


def _traffic():
    """Per-launch DRAM bytes (read + write) of the kernel groups from the
    committed ncu --set full capture (profiles/traffic.json), if present."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            return json.load(fh).get("bytes", {})
    except OSError:
        return {}


def _apply_bytes(dec, N, shared):
    """K3 algorithmic bytes: packed factors (once per block) + r in, z out."""
    fac = sum(s.size * (s.size + 1) // 2 * 8 for s in dec.subdomains)
    return fac + 16 * N


def _oracle_setup():
    """The reference's algorithm (oracle port) on all host cores: pocketfft
    through scipy.fft with one worker per core, the independent block solves
    on a fork pool of one process per core (oracle.PooledApply: the same
    solve_triangular calls, summed in ascending block id as the reference)."""
    from oracle import iedd_oracle as O
    cores = len(os.sched_getaffinity(0))
    grid = O.build_grid(CFG["dim"], CFG["n"])
    op = O.build_operator(grid, "cell")
    t0 = time.perf_counter()
    pre = O.SchwarzPrecond(op, O.build_decomposition(grid, CFG["m"], CFG["w"], "schwarz"))
    t_build = time.perf_counter() - t0
    mv = O.FFTMatvec(op, workers=cores)
    apply = O.PooledApply(pre, cores) if cores > 1 else pre
    f = np.random.default_rng(CFG["seed"]).standard_normal(op.n)
    return O, mv, apply, f, t_build, cores


def cpu_baseline(iters: int):
    """The CPU reference arm (oracle port of the reference's algorithm, FFT
    matvec, per-block triangular solves) timed on this host's cores: `iters`
    PCG iterations."""
    O, mv, pre, f, t_build, cores = _oracle_setup()
    O.pcg(mv, pre, f, tol=1e-10, max_iters=1)  # warm the pool and the FFT plans
    t0 = time.perf_counter()
    _, rep = O.pcg(mv, pre, f, tol=1e-10, max_iters=iters)
    dt = time.perf_counter() - t0
    if hasattr(pre, "close"):
        pre.close()
    return {"value": rep.n_it / dt, "unit": "iter/s", "cores": cores, "kind": "port",
            "sample": f"{rep.n_it} PCG iterations of config 5 (oracle: scipy.fft matvec on {cores} workers + "
                      f"per-block scipy solve_triangular on {cores} processes), build {t_build:.1f}s excluded",
            "host_cores_available": cores}


def run_reference(args):
    ws, rank, _ = _dist()
    if rank != 0:
        return None
    O, mv, pre, f, t_build, cores = _oracle_setup()
    if args.warmup:
        O.pcg(mv, pre, f, tol=1e-10, max_iters=args.warmup)
    t0 = time.perf_counter()
    _, rep = O.pcg(mv, pre, f, tol=1e-10, max_iters=args.steps)
    dt = time.perf_counter() - t0
    if hasattr(pre, "close"):
        pre.close()
    v = rep.n_it / dt
    out = {"metric": METRIC, "value": v, "unit": "iter/s", "n_gpus": ws, "steps": args.steps,
           "warmup": args.warmup, "ms_per_step": 1e3 * dt / rep.n_it, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (BASELINE.json config 5)",
           "impl": "reference",
           "config": config_keys(ws),
           "details": {"precond_build_s": t_build, "where": "host CPU (reference algorithm port, rank 0)"},
           "cpu_baseline": {"value": v, "unit": "iter/s", "cores": cores, "kind": "port",
                            "sample": f"{rep.n_it} PCG iterations of config 5 after {args.warmup} warm-up "
                                      f"(scipy.fft on {cores} workers, block solves on {cores} processes)"},
           "e2e": {"value": v, "unit": "iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-share", action="store_true", help="factorise every block (no translation sharing)")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--matvec", default="auto", choices=["auto", "fft", "direct"])
    ap.add_argument("--skip-noshare", action="store_true", help="skip the unshared-factor apply measurement")
    ap.add_argument("--no-configs", action="store_true", help="skip the c1-c4 solves / Lanczos runs (the configs block)")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)
    try:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            dist.destroy_process_group()
    except Exception:  # pragma: no cover
        pass


if __name__ == "__main__":
    main()
