import os, sys, subprocess
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
code = r'''
import numpy as np, paper_2108_12574_b200 as ie, sys
n=int(sys.argv[1]); m=int(sys.argv[2])
grid=ie.build_grid(2,n); op=ie.build_operator(grid,lattice="cell")
mv=ie.KernelMatvec(op,method="fft")
pre=ie.from_decomposition(op, ie.build_decomposition(grid,m,1,"schwarz"))
f=np.random.default_rng(0).standard_normal(op.n)
try:
    u,rep=ie.solve(mv,pre,f,tol=1e-10,max_iters=int(sys.argv[3]))
    print(rep.n_it, ["%.6e"%x for x in rep.residual_history[:6]])
except Exception as e: print("ERR", e)
'''
for env in ({}, {"IEDD_B200_NO_FUSE_UPD": "1"}, {"IEDD_B200_NO_FUSE_POST": "1"}, {"IEDD_B200_NO_FUSE": "1"}):
    for args in (("32", "4", "6"), ("64", "8", "6"), ("256", "32", "6")):
        e = dict(os.environ); e.update(env)
        r = subprocess.run([sys.executable, "-c", code, *args], env=e, capture_output=True, text=True)
        print(env, args, r.stdout.strip(), r.stderr.strip()[-300:])
