"""Config 1 (BASELINE configs[0]) step timing: wall time per energy step of the
device loop and the per-phase CUDA-event split (python tools/config1_profile.py [STEPS])."""
import sys, time, json
sys.path.insert(0, '.')
STEPS = int(sys.argv[1]) if len(sys.argv) > 1 else 200
import numpy as np
from paper_2508_04484_b200 import _lib
from paper_2508_04484_b200.driver import DeviceSolver
from paper_2508_04484_b200.problem import ProblemBundle
b = ProblemBundle.load('tests/golden/bundle_config1.npz')
s = DeviceSolver(b); s.init_state()
edges = b.pseudo_time_edges()
for k in range(5):
    s.set_coefficients(edges[k], edges[k+1]); s.step(edges[k]-edges[k+1])
h = s.h
h.call("pnd_synchronize")
h.call("pnd_timing", 1)
t0 = time.perf_counter(); c0 = time.process_time(); tc = 0.0
for k in range(5, 5 + STEPS):
    a = time.perf_counter(); s.set_coefficients(edges[k], edges[k+1]); tc += time.perf_counter() - a
    s.step(edges[k]-edges[k+1])
h.call("pnd_synchronize")
t = time.perf_counter() - t0
cpu = time.process_time() - c0
nph = len(_lib.PHASES); ms = np.zeros(nph); cnt = np.zeros(nph, dtype=np.int32)
h.call("pnd_timing_get", nph, _lib.ptr(ms), _lib.ptr(cnt))
print("per step ms", 1000*t/STEPS, "host coeff ms", 1000*tc/STEPS, "host cpu ms", 1000*cpu/STEPS)
hm = np.zeros(2, dtype=np.int64); h.call("pnd_spec_stats", _lib.ptr(hm)); print("speculative steps accepted/recomputed", hm.tolist())
for n, v in zip(_lib.PHASES, ms): print(n, round(v/STEPS, 4))
