"""Whole-range stability run of the bench physics (synthetic pencil beam, P19
Fokker-Planck, fixed rank) at a reduced grid: every energy step from E_max down
to the cutoff, reporting the step count, wall time, the dose's extremes and the
largest truncation tail / orthonormality defect seen.

  python tools/full_run.py NSIDE RANK [slabs] [out.json]
slabs: SURVEY.md §8(d) config 3's phantom (water / bone / lung z-slabs,
Boltzmann P7, 100 MeV); out.json gets the summary and the depth-dose curve."""
import json
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import bench  # noqa: E402

nside = int(sys.argv[1]) if len(sys.argv) > 1 else 128
rank = int(sys.argv[2]) if len(sys.argv) > 2 else 20
phantom = sys.argv[3] if len(sys.argv) > 3 else "water"
kw = dict(model="boltzmann", n_max=7, energy=100.0, phantom="slabs") if phantom == "slabs" else {}
wl = bench.Workload(nside=nside, rank=rank, **kw)
s = wl.solver
s.init_state(rank=rank)
wl.k = 0
edges = wl.edges
t0 = time.perf_counter()
worst_def = 0.0
for k in range(len(edges) - 1):
    out = wl.step()
    worst_def = max(worst_def, float(out[3]))
    if k % 1000 == 999:
        print(f"step {k + 1}: {time.perf_counter() - t0:.1f} s", flush=True)
s.h.call("pnd_synchronize")
dt = time.perf_counter() - t0
dose = s.dose()
print(f"{len(edges) - 1} steps in {dt:.1f} s ({1000 * dt / (len(edges) - 1):.1f} ms/step); "
      f"dose finite={np.isfinite(dose).all()} max={dose.max():.4e} min={dose.min():.4e}; "
      f"max orthonormality defect {worst_def:.2e}")
if len(sys.argv) > 4:
    nx, ny, nz = wl.bundle.shape
    with open(sys.argv[4], "w") as fh:
        json.dump({"grid": [nx, ny, nz], "rank": rank, "phantom": phantom,
                   "steps": len(edges) - 1, "wall_s": dt, "ms_per_step": 1000 * dt / (len(edges) - 1),
                   "dose_finite": bool(np.isfinite(dose).all()), "dose_max": float(dose.max()),
                   "max_orthonormality_defect": worst_def,
                   "depth_dose": dose.reshape(nz, ny, nx).sum(axis=(1, 2)).tolist()}, fh)
