#!/usr/bin/env python
"""Steps/s on the other BASELINE.json workloads.

  python tools/config_sweep.py            # all points, one JSON line each
  python tools/config_sweep.py --point 512:20:slabs

Each point runs in its own process (a fresh handle, so the device memory of
one point never limits the next):
- config 3: 512^3 heterogeneous z-slab phantom (water / bone +1200 HU /
  lung -700 HU at 0-3-4-7 cm), Boltzmann scattering, P7 (m = 64), 100 MeV
  +z beam, fixed rank 20, on ONE B200 (the factor and work buffers of r = 20
  at 134 M cells are ~142 GB);
- config 4: the 256^3 water P19 Fokker-Planck workload with four 90 MeV
  beams (gantry 0/45/90/135 deg in the y-z plane) in one solve, fixed rank 20;
- config 5: the rank sweep r = 10, 20, 40, 64, 80, 120, 160, 200 on the
  bench's 256^3 water P19 Fokker-Planck workload (above 64 the column-blocked
  layout of csrc/xwide.cu).
Timing as bench.py: W warm-up steps, then K steps between CUDA events on the
handle's stream; steps start at floor(n_steps / 3). Reported next to SURVEY.md
§8(d)'s cost model: fp64_frac = 192 n r^2 flops / t / (measured FP64 DGEMM
peak), hbm_frac = (392 n r + 170 n) bytes / t / (measured HBM copy bandwidth).
"""

import argparse
import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

POINTS = ["256:10:water", "256:20:water", "256:40:water", "256:64:water", "256:80:water",
          "256:120:water", "256:160:water", "256:200:water", "512:20:slabs", "256:20:beams4"]
GANTRY = (0.0, 45.0, 90.0, 135.0)


def attach_gantry_beams(wl, groups=32):
    """Config 4: four 90 MeV pencil beams at gantry 0/45/90/135 deg in the y-z plane,
    aimed at the grid centre, in one solve. Each beam's uncollided group table
    (n x G, dense -- the beams are not z-separable) is the +z pencil's depth
    spectrum laid along the beam axis with a Gaussian lateral profile."""
    import math

    import bench
    from paper_2508_04484_b200 import _lib
    from paper_2508_04484_b200.angular import beam_projection
    from paper_2508_04484_b200.problem import UncollidedSlices

    b = wl.bundle
    nx, ny, nz = b.shape
    h = b.spacing[0]
    b1, _, beam = bench.make_workload(nside=nz, n_max=b.pn_order, energy=90.0, groups=groups)
    _, depth = bench.separable_flux(b1, beam)
    f0 = b1.fluxes[0]
    k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    x = ((i.ravel() + 0.5) * h - 0.5 * nx * h)
    y = ((j.ravel() + 0.5) * h - 0.5 * ny * h)
    z = ((k.ravel() + 0.5) * h - 0.5 * nz * h)
    del i, j, k
    sx = beam["sigma_xy"]
    tms, fluxes = [], []
    for bi, deg in enumerate(GANTRY):
        th = math.radians(deg)
        d = (0.0, math.sin(th), math.cos(th))
        t = y * d[1] + z * d[2]                       # along the axis, 0 at the centre
        rho2 = x * x + (y - t * d[1]) ** 2 + (z - t * d[2]) ** 2
        kd = np.clip(((t + 0.5 * nz * h) / h).astype(np.int64), 0, nz - 1)
        lat = np.exp(-0.5 * rho2 / sx ** 2) / (2 * math.pi * sx ** 2)
        vals = np.ascontiguousarray(depth[kd] * lat[:, None])
        tm = _lib.f64(beam_projection(b.pn_order, d))
        wl.solver.h.call("pnd_set_flux_table", bi, len(GANTRY), groups, _lib.ptr(vals),
                         _lib.ptr(tm))
        del vals, lat, rho2, kd, t
        tms.append(tm)
        fluxes.append(UncollidedSlices(np.zeros((1, groups)), np.zeros(1), f0.e_min, f0.e_max))
    b.fluxes = fluxes
    b.t_ms = np.stack(tms)
    wl.solver.upload_coefficient_tables()


def run_point(spec, steps, warmup):
    import torch

    import bench
    from paper_2508_04484_b200 import _lib

    nside, rank, phantom = spec.split(":")
    nside, rank = int(nside), int(rank)
    kw = dict(model="boltzmann", n_max=7, energy=100.0, phantom="slabs") \
        if phantom == "slabs" else dict(energy=90.0) if phantom == "beams4" else {}
    t0 = time.perf_counter()
    wl = bench.Workload(nside=nside, rank=rank, **kw)
    if phantom == "beams4":
        attach_gantry_beams(wl)
    setup_s = time.perf_counter() - t0
    h = wl.solver.h
    for _ in range(warmup):
        wl.step()
    h.call("pnd_synchronize")
    free, total = torch.cuda.mem_get_info()
    h.call("pnd_event_record", 0)
    for _ in range(steps):
        wl.step()
    h.call("pnd_event_record", 1)
    h.call("pnd_synchronize")
    ms = np.zeros(1)
    h.call("pnd_event_elapsed", 0, 1, _lib.ptr(ms))
    t = ms[0] / 1000.0 / steps
    b = wl.bundle
    n = b.n_cells
    fp64 = bench.measure_fp64_peak()
    peaks = ROOT / "MEASURED_PEAKS.json"
    bw = json.loads(peaks.read_text())["hbm_gbs"] * 1e9 if peaks.exists() else 7.7e12
    dose = wl.solver.dose() if hasattr(wl.solver, "dose") else None
    out = {
        "point": spec, "grid": [nside] * 3, "rank": rank, "moments": b.n_moments,
        "model": b.model, "classes": int(b.n_classes), "phantom": phantom,
        "beams": len(b.fluxes),
        "ms_per_step": 1000.0 * t, "steps_per_s": 1.0 / t, "steps": steps, "warmup": warmup,
        "reference_step_count": len(wl.edges) - 1,
        "whole_run_s_extrapolated": t * (len(wl.edges) - 1),
        "fp64_frac": 192.0 * n * rank * rank / t / (fp64 * 1e12),
        "hbm_frac": (392.0 * n * rank + 170.0 * n) / t / bw,
        "fp64_dgemm_tflops": fp64, "device_mem_used_gb": (total - free) / 1e9,
        "setup_s": setup_s,
    }
    if dose is not None:
        d = np.asarray(dose)
        out["dose_finite"] = bool(np.isfinite(d).all())
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--point")
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    if args.point:
        run_point(args.point, args.steps, args.warmup)
        return
    for p in POINTS:
        res = subprocess.run([sys.executable, __file__, "--point", p, "--steps", str(args.steps),
                              "--warmup", str(args.warmup)], capture_output=True, text=True)
        line = res.stdout.strip().splitlines()[-1] if res.returncode == 0 and res.stdout.strip() \
            else json.dumps({"point": p, "error": res.stderr[-600:]})
        print(line, flush=True)


if __name__ == "__main__":
    main()
