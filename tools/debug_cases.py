"""Run one apply_streaming case per subprocess (sticky CUDA errors) and report."""
import subprocess, sys, json
cases = [(5,4,6,9),(7,8,8,9),(8,8,8,16),(1,1,12,9),(40,40,40,16),(1,5,7,4)]
code = r'''
import sys, numpy as np
sys.path.insert(0, ".")
from types import SimpleNamespace
from paper_2508_04484_b200 import dlra
from paper_2508_04484_b200.angular import PNOperators
from oracle import dlra_np
nx,ny,nz,m = [int(v) for v in sys.argv[1:5]]
nmax = int(round(m ** 0.5)) - 1
ops = PNOperators.build(nmax)
g = SimpleNamespace(nx=nx,ny=ny,nz=nz,dx=0.1,dy=0.2,dz=0.3)
n = nx*ny*nz
rng = np.random.default_rng(0)
inv_s = 1/rng.uniform(5,10,n); u = rng.standard_normal((n, (nmax+1)**2))
ctx = dlra.StreamingContext(inv_s, SimpleNamespace(grid=g), ops)
got = ctx.full_rhs(u)
ref = dlra_np.apply_streaming(u, inv_s, dlra_np.Grid(nx,ny,nz,0.1,0.2,0.3), dlra_np.Ops(ops.eig_v, ops.lam_plus, ops.lam_minus))
print(np.abs(got-ref).max()/np.abs(ref).max())
'''
for c in cases:
    r = subprocess.run([sys.executable, "-c", code] + [str(v) for v in c], capture_output=True, text=True,
                       env={**__import__("os").environ, "CUDA_LAUNCH_BLOCKING": "1"})
    print(c, r.returncode, (r.stdout.strip() or r.stderr.strip().splitlines()[-1])[:200])
