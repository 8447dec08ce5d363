"""Adaptive-rank probe on the bench workload (256^3 water, P19 FP): run the
first energy steps from a rank-2 zero state with the tail threshold set
relative to the running largest singular value, and print the rank history
(how far the rank-adaptive config 2 of SURVEY.md §8(d) goes)."""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import bench  # noqa: E402
from paper_2508_04484_b200 import _lib as bench_lib  # noqa: E402

nside = int(sys.argv[1]) if len(sys.argv) > 1 else 128
# "abs:1e-8" = SURVEY.md §8(d) config 2's absolute threshold (theta = 1e-8 x beam
# weight, weight 1); a plain number is relative to the running largest sigma
arg = sys.argv[2] if len(sys.argv) > 2 else "1e-8"
absolute = arg.startswith("abs:")
rel = float(arg[4:] if absolute else arg)
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 400
wl = bench.Workload(nside=nside, rank=2)
s = wl.solver
b = wl.bundle
s.init_state(rank=2)
wl.k = 0
edges = wl.edges
smax = 0.0
hist, stop = [], None
t0 = time.perf_counter()
for k in range(min(steps, len(edges) - 1)):
    e_hi, e_lo = edges[k], edges[k + 1]
    b.truncation_tolerance = rel if absolute else max(rel * smax, 1e-300)
    b.rank_min, b.rank_max = 2, int(sys.argv[4]) if len(sys.argv) > 4 else 64
    s.set_coefficients(e_hi, e_lo)
    try:
        out = s.step(e_hi - e_lo, want_defect=False)
    except Exception as exc:  # noqa: BLE001 -- the reference's rank_max error ends the probe
        stop = f"step {k}: {exc}"
        break
    r = int(out[2])
    hist.append(r)
    sm = np.empty((r, r))
    s.h.call("pnd_state_get", None, bench_lib.ptr(sm), None)
    sig = np.linalg.svd(sm, compute_uv=False)
    smax = max(smax, float(sig[0]) if sig.size else 0.0)
    if k % 25 == 0 or int(out[2]) >= 30:
        print(k, f"E={e_lo:.2f}", "rank", int(out[2]), f"smax={smax:.3e}", flush=True)
wall = time.perf_counter() - t0
print(json.dumps({"grid": [nside] * 3, "theta": arg, "steps": len(hist), "wall_s": wall,
                  "ms_per_step": 1000.0 * wall / max(len(hist), 1),
                  "rank_at": {str(i): hist[i] for i in range(0, len(hist), 10)},
                  "final_rank": hist[-1] if hist else None, "stopped": stop}))
