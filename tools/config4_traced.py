#!/usr/bin/env python
"""SURVEY.md §8(d) config 4 with TRACED uncollided fluxes: 256^3 water (h =
0.025 cm), P19 Fokker-Planck, four 90 MeV pencil beams at gantry 0/45/90/135
deg in the y-z plane aimed at the grid centre, in one low-rank solve.

Each beam is traced on the device (paper_2508_04484_b200.raytracer.
trace_beam_ops: traversal, signature de-duplication, CN march per distinct
signature, deposit) with the reference's own water energy operator
(tests/golden/water_ops90.npz) and kept on its ray footprint (sparse table:
the dense 256^3 x 128-group table is 17 GB per beam), then the joint solve
runs K energy steps at fixed rank from step floor(n_steps / 3) (CUDA events).
Per-beam dose time = (trace + the whole energy loop at the measured step
time + the uncollided tally) / beams.

    python tools/config4_traced.py [NSIDE=256] [RANK=20] [N_SIDE=21] [STEPS=4]
"""
import json
import math
import sys
import time
from pathlib import Path
from types import SimpleNamespace

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import bench  # noqa: E402

GANTRY = (0.0, 45.0, 90.0, 135.0)


def main():
    nside = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    rank = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    n_side = int(sys.argv[3]) if len(sys.argv) > 3 else 21
    steps = int(sys.argv[4]) if len(sys.argv) > 4 else 4
    from paper_2508_04484_b200 import _lib
    from paper_2508_04484_b200 import raytracer as rt
    from paper_2508_04484_b200.angular import beam_projection
    from paper_2508_04484_b200.driver import DeviceSolver
    from paper_2508_04484_b200.problem import UncollidedSlices

    W = np.load(ROOT / "tests" / "golden" / "water_ops90.npz")
    sp = W["space"]
    space = rt.EnergySpace(float(sp[0]), float(sp[1]), int(sp[2]), int(sp[3]))
    b, _, _ = bench.make_workload(nside=nside, n_max=19, rank=rank, energy=90.0)
    h = b.spacing[0]
    L = nside * h
    grid = SimpleNamespace(nx=nside, ny=nside, nz=nside, dx=h, dy=h, dz=h,
                           origin=(0.0, 0.0, 0.0))
    keys = np.zeros(b.n_cells, dtype=np.int32)
    gm, smin = {0: W["g_fp19"]}, {0: float(W["smin_fp19"])}  # P19 Fokker-Planck water
    fluxes, t_ms, traces = [], [], []
    rt.trace_beam_ops(SimpleNamespace(direction=(0.0, 0.0, 1.0), energy_mev=90.0,
                                      position_cm=(L / 2, L / 2, -0.5), weight=1.0,
                                      sigma_xy_cm=0.3, sigma_e_mev=0.9),
                      grid, space, keys, gm, smin, 3, 3.0, 0.01, sparse=True)  # warm-up
    for deg in GANTRY:
        th = math.radians(deg)
        d = (0.0, math.sin(th), math.cos(th))
        pos = tuple(L / 2 - (L / 2 + 0.5) * c for c in (0.0, d[1], d[2]))
        pos = (L / 2, pos[1], pos[2])
        beam = SimpleNamespace(direction=d, energy_mev=90.0, position_cm=pos, weight=1.0,
                               sigma_xy_cm=0.3, sigma_e_mev=0.9)
        t0 = time.perf_counter()
        f = rt.trace_beam_ops(beam, grid, space, keys, gm, smin, n_side, 3.0, 0.01, sparse=True)
        traces.append(time.perf_counter() - t0)
        fluxes.append(UncollidedSlices(f.values, f.residual_energy, space.e_min, space.e_max,
                                       f.cells, b.n_cells))
        t_ms.append(beam_projection(19, d))
    b.fluxes, b.t_ms = fluxes, np.stack(t_ms)
    t0 = time.perf_counter()
    solver = DeviceSolver(b)
    setup_s = time.perf_counter() - t0
    solver.h.call("pnd_state_random", rank, 12345)
    edges = b.pseudo_time_edges()
    k0 = (len(edges) - 1) // 3

    def step(k):
        solver.set_coefficients(edges[k], edges[k + 1])
        return solver.step(edges[k] - edges[k + 1], want_defect=True)

    for k in range(k0, k0 + 2):
        step(k)
    solver.h.call("pnd_synchronize")
    solver.h.call("pnd_event_record", 0)
    for k in range(k0 + 2, k0 + 2 + steps):
        out = step(k)
    solver.h.call("pnd_event_record", 1)
    solver.h.call("pnd_synchronize")
    ms = np.zeros(1)
    solver.h.call("pnd_event_elapsed", 0, 1, _lib.ptr(ms))
    t_step = ms[0] / 1000.0 / steps
    t0 = time.perf_counter()
    unc = b.uncollided_dose()
    tally_s = time.perf_counter() - t0
    dose = solver.dose()
    solver.close()
    n_steps = len(edges) - 1
    loop_s = t_step * n_steps
    nnz = [len(f.cells) for f in fluxes]
    print(json.dumps({
        "config": "SURVEY §8(d) config 4, traced", "grid": [nside] * 3, "rank": rank,
        "moments": b.n_moments, "beams": len(GANTRY), "rays_per_beam": n_side * n_side,
        "trace_s_per_beam": traces, "footprint_cells_per_beam": nnz,
        "footprint_fraction": [x / b.n_cells for x in nnz],
        "sparse_table_gb": sum(x * space.n_groups * 8 for x in nnz) / 1e9,
        "dense_table_gb": len(GANTRY) * b.n_cells * space.n_groups * 8 / 1e9,
        "setup_s": setup_s, "ms_per_step": 1000 * t_step, "steps_timed": steps,
        "reference_step_count": n_steps, "loop_s_extrapolated": loop_s,
        "uncollided_tally_s": tally_s,
        "per_beam_dose_time_s": (sum(traces) + setup_s + loop_s + tally_s) / len(GANTRY),
        "rank_out": int(out[2]), "dose_finite": bool(np.isfinite(dose).all()),
        "uncollided_max": float(unc.max())}))


if __name__ == "__main__":
    main()
