"""Whole-range stability run of the bench physics (synthetic pencil beam, P19
Fokker-Planck, fixed rank) at a reduced grid: every energy step from E_max down
to the cutoff, reporting the step count, wall time, the dose's extremes and the
largest truncation tail / orthonormality defect seen."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import bench  # noqa: E402

nside = int(sys.argv[1]) if len(sys.argv) > 1 else 128
rank = int(sys.argv[2]) if len(sys.argv) > 2 else 20
wl = bench.Workload(nside=nside, rank=rank)
s = wl.solver
s.init_state(rank=rank)
wl.k = 0
edges = wl.edges
t0 = time.perf_counter()
worst_def = 0.0
for k in range(len(edges) - 1):
    out = wl.step()
    worst_def = max(worst_def, float(out[3]))
s.h.call("pnd_synchronize")
dt = time.perf_counter() - t0
dose = s.dose()
print(f"{len(edges) - 1} steps in {dt:.1f} s ({1000 * dt / (len(edges) - 1):.1f} ms/step); "
      f"dose finite={np.isfinite(dose).all()} max={dose.max():.4e} min={dose.min():.4e}; "
      f"max orthonormality defect {worst_def:.2e}")
