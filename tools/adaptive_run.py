#!/usr/bin/env python
"""Rank-adaptive whole run of SURVEY.md §8(d) config 2's physics (water, P19
Fokker-Planck, 70 MeV pencil beam, CFL 0.2) on the device: from the
reference's zero state (rank_min 2), truncation threshold theta = 1e-8 x beam
weight (absolute, the reference's tail rule dlra.py:90-115), rank_max 200,
every energy step from E_max to the cutoff -- or until the tail rule asks for
more than rank_max, where the reference itself raises its rank_max error
(dlra.py:101-108) and so does this loop.

  python tools/adaptive_run.py NSIDE [CM=6.4] [THETA=1e-8] [RANK_MAX=200] [out.json]

The phantom is a CM-cm cube (h = CM / NSIDE); the rank history, wall time
and the dose's depth curve go to out.json.
"""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import bench  # noqa: E402

nside = int(sys.argv[1]) if len(sys.argv) > 1 else 128
cm = float(sys.argv[2]) if len(sys.argv) > 2 else 6.4
theta = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-8
rmax = int(sys.argv[4]) if len(sys.argv) > 4 else 200
out_path = sys.argv[5] if len(sys.argv) > 5 else None
wl = bench.Workload(nside=nside, rank=2, h=cm / nside)
b = wl.bundle
b.truncation_tolerance, b.rank_min, b.rank_max = theta, 2, rmax
s = wl.solver
s.init_state(rank=2)
edges = wl.edges
ranks, walls, stop = [], [], None
max_def = 0.0
t0 = time.perf_counter()
for k in range(len(edges) - 1):
    e_hi, e_lo = edges[k], edges[k + 1]
    s.set_coefficients(e_hi, e_lo)
    try:
        out = s.step(e_hi - e_lo, want_defect=True)
    except Exception as exc:  # noqa: BLE001 -- the reference's rank_max error ends the run
        stop = f"step {k} (E = {e_hi:.3f} MeV): {exc}"
        break
    ranks.append(int(out[2]))
    max_def = max(max_def, float(out[3]))
    walls.append(time.perf_counter() - t0)
    if k % 50 == 0:
        print(f"step {k} E={e_lo:.2f} rank {ranks[-1]} t={walls[-1]:.1f}s", flush=True)
s.h.call("pnd_synchronize")
wall = time.perf_counter() - t0
dose = s.dose()
nx, ny, nz = b.shape
summary = {"grid": [nside] * 3, "h_cm": cm / nside, "theta": theta, "rank_max": rmax,
           "reference_steps": len(edges) - 1, "steps_done": len(ranks), "completed": stop is None,
           "stopped": stop, "wall_s": wall, "ms_per_step": 1000 * wall / max(len(ranks), 1),
           "max_rank": max(ranks) if ranks else None,
           "mean_rank": float(np.mean(ranks)) if ranks else None,
           "max_orthonormality_defect": max_def,
           "dose_finite": bool(np.isfinite(dose).all()),
           "rank_history": ranks,
           "depth_dose": dose.reshape(nz, ny, nx).sum(axis=(1, 2)).tolist()}
print(json.dumps({k: v for k, v in summary.items() if k not in ("rank_history", "depth_dose")}))
if out_path:
    with open(out_path, "w") as fh:
        json.dump(summary, fh)
