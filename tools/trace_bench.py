#!/usr/bin/env python
"""Uncollided tracer timing on BASELINE.md's 40^3 cases.

40^3 water at 1 mm, 121 rays per beam (n_side 11), 70 MeV: one 0 deg beam, one
30 deg beam, and four beams at 0/30/60/90 deg. The inputs (the reference's
energy operator for water, its s*(e_min), the beams) and the reference's own
trace_all_beams wall time on the build host's CPU come from
tests/golden/trace40.npz (tools/make_golden.py make_trace40). Per case the
device tracer (paper_2508_04484_b200.raytracer.trace_beam_ops: device
traversal, signature de-duplication, device CN march per distinct signature,
device deposit) is timed end to end on the host clock, after one warm-up, and
its flux is checked against the reference's (sampled cells, column sums,
residual energy). One JSON line per case.

    python tools/trace_bench.py [--repeat 3]
"""

import argparse
import json
import sys
import time
from pathlib import Path
from types import SimpleNamespace

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

CASES = ("deg0", "deg30", "beams4")


def load():
    T = np.load(ROOT / "tests" / "golden" / "trace40.npz")
    return {k: T[k] for k in T.files}


def trace_case(T, tag, rt):
    sp = T["space"]
    space = rt.EnergySpace(float(sp[0]), float(sp[1]), int(sp[2]), int(sp[3]))
    grid = SimpleNamespace(nx=40, ny=40, nz=40, dx=0.1, dy=0.1, dz=0.1, origin=(0.0, 0.0, 0.0))
    gm, smin = {0: T["g"]}, {0: float(T["smin"])}
    fluxes = []
    for i in range(int(T[tag + "_n_beams"])):
        p = f"{tag}_b{i}_"
        b = T[p + "beam"]
        beam = SimpleNamespace(direction=tuple(b[:3]), energy_mev=b[3],
                               position_cm=tuple(b[4:7]), weight=b[7], sigma_xy_cm=b[8],
                               sigma_e_mev=b[9])
        rays = T[p + "rays"]
        fluxes.append(rt.trace_beam_ops(beam, grid, space, T["keys"], gm, smin, int(rays[0]),
                                        float(rays[1]), float(rays[2])))
    return fluxes


def check(T, tag, fluxes):
    worst = 0.0
    for i, f in enumerate(fluxes):
        p = f"{tag}_b{i}_"
        for got, want in ((f.values[T["sample"]], T[p + "values_sample"]),
                          (f.values.sum(axis=0), T[p + "values_colsum"]),
                          (f.residual_energy, T[p + "residual"])):
            scale = max(np.abs(want).max(), 1e-300)
            worst = max(worst, float(np.abs(got - want).max() / scale))
        if f.n_rays != int(T[p + "n_rays"]):
            worst = float("inf")
    return worst


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--repeat", type=int, default=3)
    args = ap.parse_args()
    from paper_2508_04484_b200 import raytracer as rt

    T = load()
    for tag in CASES:
        trace_case(T, tag, rt)  # warm-up (kernels, allocations)
        times = []
        for _ in range(args.repeat):
            t0 = time.perf_counter()
            fluxes = trace_case(T, tag, rt)
            times.append(time.perf_counter() - t0)
        dev = check(T, tag, fluxes)
        cpu = float(T[tag + "_cpu_s"])
        print(json.dumps({
            "case": tag, "grid": [40, 40, 40], "rays_per_beam": 121,
            "beams": int(T[tag + "_n_beams"]), "gpu_s": min(times), "gpu_s_all": times,
            "reference_cpu_s": cpu, "speedup": cpu / min(times),
            "reference_marches": int(T[tag + "_marches"]), "reference_lus": int(T[tag + "_lus"]),
            "max_rel_dev_vs_reference": dev,
            "reference_host": "build container, 1 OpenBLAS thread (tools/make_golden.py)"}),
            flush=True)


if __name__ == "__main__":
    main()
