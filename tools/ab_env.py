"""Same-box A/B of an environment switch on the config-5 PCG iteration time:
alternating processes, median of the per-process best of 5 timed solves.

  python tools/ab_env.py IEDD_B200_NO_L2PERSIST [reps]
  python tools/ab_env.py IEDD_B200_LIB=/path/to/other/libiedd_b200.so [reps]
"""
import json
import os
import statistics
import subprocess
import sys

CHILD = r'''
import os, sys, json, numpy as np, torch
sys.path.insert(0, os.environ["IEDD_ROOT"])
import paper_2108_12574_b200 as ie
grid = ie.build_grid(2, 1024); op = ie.build_operator(grid, lattice="cell")
mv = ie.ToeplitzMatvec(op)
pre = ie.from_decomposition(op, ie.build_decomposition(grid, 128, 2, "schwarz"))
f = torch.from_numpy(np.random.default_rng(3).standard_normal(op.n)).cuda()
ie.solve(mv, pre, f, tol=1e-10, max_iters=10)
st = torch.cuda.current_stream(); best = 1e9
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record(st)
    ie.solve(mv, pre, f, tol=1e-10, max_iters=50)
    e1.record(st); torch.cuda.synchronize(); best = min(best, e0.elapsed_time(e1))
print(json.dumps({"ms_per_iter": best / 50}))
'''


def main():
    var, _, val = sys.argv[1].partition("=")
    val = val or "1"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {"off": [], "on": []}
    for _ in range(reps):
        for key in ("off", "on"):
            env = dict(os.environ, IEDD_ROOT=root)
            env.pop(var, None)
            if key == "on":
                env[var] = val
            out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
            line = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
            if not line:
                print(out.stderr[-2000:])
                continue
            res[key].append(json.loads(line[-1])["ms_per_iter"])
    print(json.dumps({"var": var, "unset_ms": res["off"], "set_ms": res["on"],
                      "median_unset_ms": statistics.median(res["off"]) if res["off"] else None,
                      "median_set_ms": statistics.median(res["on"]) if res["on"] else None}))


if __name__ == "__main__":
    main()
