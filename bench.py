#!/usr/bin/env python
"""Benchmark: DLRA energy steps/s on the BASELINE.json configs[1] workload.

Workload: 3-D homogeneous water phantom, 256^3
cells at h = 0.025 cm (6.4 cm cube), P_19 (m = 400 moments), Fokker-Planck
collided equation, 70 MeV +z pencil beam (sigma_xy = 0.3 cm), CFL 0.2
(the step count the reference would take is reported). The rank is pinned at
r = 20 (truncation runs after both substeps with the rank clamped,
theta = 1e300, rank_min = rank_max = 20): a pinned rank makes every step the
same work, so steps/s is a rate (--rank up to 64; configs 3-5 of SURVEY.md
§8(d) are measured by tools/config_sweep.py).
One "step" is the reference's full energy step (driver.py:578-622):
streaming -> truncate -> scattering -> truncate -> dose trapezoid, plus the
orthonormality diagnostic, starting from a preset rank-20 state at step
floor(n_steps / 3) of the energy grid. Inputs are synthetic (no datasets):
the uncollided flux is a separable pencil-beam table formed on the device,
the physics tables (stopping powers, Molière moments) are the reference's,
exported to tests/golden/bench_physics.npz.

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]

N > 1 (torchrun): one joint solve of the same 256^3 grid, z-slab sharded (each
rank owns nz/N planes; the stencil halo planes and every Gram sum go over NCCL,
DESIGN.md §6), "scaling": "strong". Timing: CUDA events on the handle's stream
around the K timed steps, barrier + synchronize on both sides, max over ranks.
"""

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "DLRA energy steps/s (256^3 water, P19 Fokker-Planck, rank 20)"


def metric_name(nside, rank, phantom="water"):
    """The headline metric; non-default --nside / --rank / --phantom name their own workload."""
    if phantom == "slabs":
        return f"DLRA energy steps/s ({nside}^3 water/bone/lung slabs, P7 Boltzmann, rank {rank})"
    return f"DLRA energy steps/s ({nside}^3 water, P19 Fokker-Planck, rank {rank})"


# --phantom slabs: SURVEY.md §8(d) config 3's physics
PHANTOM_KW = {"water": {}, "slabs": dict(model="boltzmann", n_max=7, energy=100.0,
                                         phantom="slabs")}
UNIT = "steps/s"


# ----------------------------------------------------------------- workload
SLAB_PHANTOM = ((0.0, 3.0, 0), (3.0, 4.0, 1), (4.0, 7.0, 2))  # (z0, z1 cm, class)


def plane_classes(nz, h, phantom):
    """Material class of every z plane: "water", or "slabs" -- SURVEY.md §8(d)
    config 3: water 0 HU z in [0, 3) cm, bone +1200 HU [3, 4), lung -700 HU
    [4, 7), water beyond (classes 0, 1, 2 of bench_physics.npz)."""
    zc = np.zeros(nz, dtype=np.int32)
    if phantom == "slabs":
        z = (np.arange(nz) + 0.5) * h
        for z0, z1, c in SLAB_PHANTOM:
            zc[(z >= z0) & (z < z1)] = c
    return zc


def make_workload(nside=256, h=0.025, n_max=19, rank=20, model="fokker-planck",
                  energy=70.0, sigma_xy=0.3, groups=128, phantom="water"):
    """ProblemBundle of a synthetic phantom (no flux table attached)."""
    from paper_2508_04484_b200.angular import PNOperators
    from paper_2508_04484_b200.problem import ProblemBundle, UncollidedSlices

    ph = np.load(ROOT / "tests" / "golden" / "bench_physics.npz")
    ops = PNOperators.build(n_max)
    sigma_e = 0.01 * energy
    e_max = energy + 5.0 * sigma_e
    zc = plane_classes(nside, h, phantom)
    nc = int(zc.max()) + 1
    b = ProblemBundle(
        shape=(nside, nside, nside), spacing=(h, h, h), origin=(0.0, 0.0, 0.0),
        cell_class=np.repeat(zc, nside * nside),
        class_density=ph["class_density"][:nc], class_weights=ph["class_weights"][:nc],
        class_atomic=ph["class_atomic"][:nc],
        stop_e=ph["stop_e"], stop_s=ph["stop_s"], mom_e=ph["mom_e"],
        mom_g=ph["mom_g"][..., : n_max + 2], mom_xi1=ph["mom_xi1"],
        eig_v=np.stack(ops.eig_v), lam_plus=np.stack(ops.lam_plus),
        lam_minus=np.stack(ops.lam_minus),
        t_ms=np.array([_beam_tm(n_max)]),
        fluxes=[UncollidedSlices(np.zeros((1, groups)), np.zeros(1), 1.0, e_max)],
        model=model, pn_order=n_max, e_min=1.0, e_max=e_max, cfl_number=0.2,
        truncation_tolerance=1e300, rank_min=rank, rank_max=rank, name=f"bench{nside}",
    )
    return b, ops, dict(energy=energy, sigma_e=sigma_e, sigma_xy=sigma_xy, groups=groups,
                        plane_class=zc)


def _beam_tm(n_max):
    from paper_2508_04484_b200.angular import beam_projection

    return beam_projection(n_max, (0.0, 0.0, 1.0))


def separable_flux(b, beam):
    """Lateral Gaussian x depth-energy spectrum of a +z pencil beam.

    Depth: CSDA mean energy E(z) from the water stopping power, Gaussian
    energy spread widening with depth, mild attenuation; lateral: normalised
    Gaussian of sigma_xy. Values are group representatives [1/(MeV cm^2)].
    """
    nx, ny, nz = b.shape
    hx, hy, hz = b.spacing
    x = (np.arange(nx) + 0.5) * hx - 0.5 * nx * hx
    y = (np.arange(ny) + 0.5) * hy - 0.5 * ny * hy
    sx = beam["sigma_xy"]
    lat = np.exp(-0.5 * (x[None, :] ** 2 + y[:, None] ** 2) / sx ** 2) / (2 * math.pi * sx ** 2)
    f = b.fluxes[0]
    centers = f.centers
    zc = beam.get("plane_class", np.zeros(nz, dtype=np.int32))
    z = (np.arange(nz) + 0.5) * hz
    e = beam["energy"]
    depth = np.zeros((nz, f.n_groups))
    zz = 0.0
    for k in range(nz):
        while zz < z[k] and e > 1.0:
            dz = min(0.001, z[k] - zz)
            e -= float(b.class_stopping(max(e, 1.0))[zc[k]]) * dz
            zz += dz
        if e <= 1.0:
            break
        sig = math.sqrt(beam["sigma_e"] ** 2 + 0.01 * z[k])
        depth[k] = np.exp(-0.012 * z[k]) * np.exp(-0.5 * ((centers - e) / sig) ** 2) / (
            sig * math.sqrt(2 * math.pi))
    return lat.ravel(), depth


class Workload:
    def __init__(self, nside=256, rank=20, device=0, n_max=19, slab=None, comm_id=None,
                 model="fokker-planck", energy=70.0, phantom="water", h=0.025):
        """slab: this process's z-planes of the joint multi-GPU solve (slabs.plan),
        comm_id the world's NCCL id; None = the whole grid on this GPU."""
        from paper_2508_04484_b200 import _lib
        from paper_2508_04484_b200.driver import DeviceSolver

        self.bundle, self.ops, beam = make_workload(nside=nside, h=h, rank=rank, n_max=n_max,
                                                    model=model, energy=energy, phantom=phantom)
        b = self.bundle
        self.rank = rank
        self.solver = DeviceSolver.__new__(DeviceSolver)
        self.solver.bundle = b
        lo, hi = (0, b.n_cells) if slab is None else slab.rows
        z0, z1 = (0, b.shape[2]) if slab is None else (slab.z0, slab.z1)
        shape = (b.shape[0], b.shape[1], z1 - z0)
        self.solver.rows = (lo, hi)
        self.solver.h = _lib.Handle(shape, b.spacing, b.n_moments, device)
        h = self.solver.h
        if slab is not None:
            h.set_slab(z0, b.shape[2], comm_id, slab.rank, slab.world)
        h.set_angular(*b.a_split())
        h.set_materials(b.cell_class[lo:hi], b.class_atomic)
        lat, depth = separable_flux(b, beam)
        depth = depth[z0:z1]
        lat, depth, tm = _lib.f64(lat), _lib.f64(depth), _lib.f64(b.t_ms[0])
        h.call("pnd_set_flux_separable", 0, 1, int(depth.shape[1]), _lib.ptr(lat),
               _lib.ptr(depth), _lib.ptr(tm))
        h.call("pnd_dose_reset")
        self.solver.upload_coefficient_tables()  # per-step coefficients formed on the GPU
        h.call("pnd_state_random", rank, 12345)
        self.edges = b.pseudo_time_edges()
        self.k0 = (len(self.edges) - 1) // 3
        self.k = self.k0

    def step(self):
        e_hi, e_lo = self.edges[self.k], self.edges[self.k + 1]
        self.solver.set_coefficients(e_hi, e_lo)
        out = self.solver.step(e_hi - e_lo, want_defect=True)
        self.k += 1
        return out

    def h2d_bytes_per_step(self):
        # the e2e leg's per-step inputs, formed on the host (set_coefficients with
        # device_coefficients=False)
        b = self.bundle
        # class S (M), g_diags (12 x m), sigma_t (12), flux lerp (2 int32 + 2 f64 per beam)
        return 8 * (b.n_classes + 12 * b.n_moments + 12) + len(b.fluxes) * (2 * 4 + 2 * 8)

    def d2h_bytes_per_step(self):
        # step outputs (4 f64) + two truncation read-backs (f64 tail + i32 rank)
        return 4 * 8 + 2 * (8 + 4)


# ----------------------------------------------------------------- model
def phase_model(n, r, m, ns=6):
    """Algorithmic FP64 flops and HBM bytes per launch of each phase."""
    R = 2 * r
    return {
        # one Horner stage: U0 S0 (r^2) + ns stencil contractions (ns r^2) per cell
        "kstage": {"flops": 2.0 * n * (r * r + ns * r * r), "bytes": 8.0 * n * (3 * r + 1)},
        # sum_s U^T D_s S^-1 U^: ns R x R Grams over n cells, read U^ once
        "s_gram": {"flops": 2.0 * n * ns * R * R, "bytes": 8.0 * n * (R + 1)},
        "l_gram": {"flops": 2.0 * n * ns * r * r, "bytes": 8.0 * n * (r + 1)},
        # Householder TSQR of n x R: factor (2nR^2) + form Q (2nR^2); read A, write V,
        # read V, write Q
        "tsqr_n": {"flops": 4.0 * n * R * R, "bytes": 8.0 * n * 4 * R},
    }


def measure_fp64_peak():
    import torch

    a = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
    b = torch.randn(8192, 8192, dtype=torch.float64, device="cuda")
    for _ in range(2):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, 2 * 8192 ** 3 / (e0.elapsed_time(e1) * 1e-3) / 1e12)
    del a, b
    torch.cuda.empty_cache()
    return best


class ClockSampler:
    def __init__(self, index=0):
        self.path = tempfile.mktemp(suffix=".csv")
        fields = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
                  "clocks_event_reasons.hw_thermal_slowdown,"
                  "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={index}", f"--query-gpu={fields}", "--format=csv,noheader",
                 "-lms", "200"], stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait()
        rows = [ln.split(",") for ln in Path(self.path).read_text().splitlines() if ln.strip()]
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for row in rows:
            try:
                sm.append(float(row[1].split()[0]))
                smax = float(row[2].split()[0])
            except (ValueError, IndexError):
                continue
            for nm, v in zip(names, row[4:8]):
                if "Active" in v and "Not" not in v:
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------- CPU legs
CPU_SIDE = 64


def cpu_sample_main(args):
    """Time the numpy oracle (reference algorithm) on a 64^3 sample of the
    workload: the same phantom and physics (--phantom), fewer cells."""
    from oracle import dlra_np

    b, ops, beam = make_workload(nside=CPU_SIDE, rank=args.rank, **PHANTOM_KW[args.phantom])
    grid = dlra_np.Grid(*b.shape, *b.spacing)
    o = dlra_np.Ops(b.eig_v, b.lam_plus, b.lam_minus)
    n, m, r = b.n_cells, b.n_moments, args.rank
    rng = np.random.default_rng(1)
    u = np.linalg.qr(rng.standard_normal((n, r)))[0]
    v = np.linalg.qr(rng.standard_normal((m, r)))[0]
    s = np.diag(np.logspace(0, -3, r))
    lat, depth = separable_flux(b, beam)
    edges = b.pseudo_time_edges()
    k0 = (len(edges) - 1) // 3
    weights = b.atomic_densities
    f = b.fluxes[0]
    times = []
    for k in range(k0, k0 + args.cpu_steps):
        t0 = time.perf_counter()
        e_hi, e_lo = edges[k], edges[k + 1]
        dt, e_mid = e_hi - e_lo, 0.5 * (e_hi + e_lo)
        inv_s = 1.0 / b.stopping_field(e_mid)
        g, st = b.scattering_tables(e_mid)
        j0, w0, j1, w1 = f.lerp_weights(e_mid)
        psi = (lat.reshape(1, -1) * (w0 * depth[:, j0] + w1 * depth[:, j1])[:, None]).ravel()
        u, s, v = dlra_np.streaming_step(u, s, v, dt, inv_s, grid, o)
        u, s, v, _ = dlra_np.truncate(u, s, v, 1e300, r, r)
        u, s, v = dlra_np.scattering_step(u, s, v, dt, weights, inv_s, g, st,
                                          [(psi, b.t_ms[0])])
        u, s, v, _ = dlra_np.truncate(u, s, v, 1e300, r, r)
        _ = u @ (s @ v[0])
        _ = max(np.abs(u.T @ u - np.eye(r)).max(), np.abs(v.T @ v - np.eye(r)).max())
        times.append(time.perf_counter() - t0)
    per_step = float(np.mean(times))
    print(json.dumps({"per_step_s": per_step, "cells": n, "steps": len(times),
                      "total_s": float(np.sum(times))}))


def cpu_model():
    try:
        for ln in Path("/proc/cpuinfo").read_text().splitlines():
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def run_cpu_sample(threads, steps, rank, nside=256, phantom="water"):
    """The numpy oracle (oracle/dlra_np.py, the reference algorithm restated) on
    `steps` energy steps of the same phantom and physics at 64^3 cells, timed on
    this host, extrapolated to nside^3 by cell count (the per-cell cost is
    constant in n) -- reported as such (`extrapolated`)."""
    env = dict(os.environ)
    for k in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
        env[k] = str(threads)
    t0 = time.perf_counter()
    res = subprocess.run([sys.executable, __file__, "--cpu-sample", "--cpu-steps", str(steps),
                          "--rank", str(rank), "--phantom", phantom], capture_output=True,
                         text=True, env=env, timeout=900)
    wall = time.perf_counter() - t0
    if res.returncode != 0:
        raise RuntimeError(res.stderr[-2000:])
    out = json.loads(res.stdout.strip().splitlines()[-1])
    per_cell = out["per_step_s"] / out["cells"]
    n_full = nside ** 3
    physics = "P7 Boltzmann, 3-class slabs" if phantom == "slabs" else "P19 FP water"
    return {
        "value": 1.0 / (per_cell * n_full),
        "unit": UNIT,
        "cores": threads,
        "cpu_model": cpu_model(),
        "kind": "port",
        "extrapolated": True,
        "timed": {"grid": [CPU_SIDE] * 3, "cells": out["cells"], "steps": out["steps"],
                  "s_per_step": out["per_step_s"], "cpu_s": out["total_s"], "wall_s": wall},
        "sample": (f"numpy oracle (oracle/dlra_np.py, the reference algorithm) timed on "
                   f"{out['steps']} energy steps of the same physics at {CPU_SIDE}^3 cells "
                   f"(rank {rank}, {physics}) = {out['per_step_s']:.2f} s/step, extrapolated by "
                   f"cell count to {nside}^3 (per-cell cost is constant in n, SURVEY.md §6.2); "
                   f"{out['total_s']:.1f} s of CPU work"),
    }


def roofline_traffic(nside, rank, phantom, kernel):
    """ncu DRAM bytes per launch of `kernel` measured on this exact workload
    (profiles/traffic.json, keyed "<nside>_<rank>_<phantom>"); None when no
    capture of this workload exists."""
    tpath = ROOT / "profiles" / "traffic.json"
    if not tpath.exists():
        return None
    entry = json.loads(tpath.read_text()).get(f"{nside}_{rank}_{phantom}", {})
    return entry.get(kernel)


def config1_dose_time(with_cpu):
    """Per-beam dose time on the reference's CPU-oracle config (BASELINE.json
    configs[0]: 2-D water, P7, fixed rank 20, 573
    energy steps, one beam): the whole energy loop + dose tally through the
    public API, from the exported problem (assembly and ray tracing are the
    reference's host code and are not part of this path)."""
    import dataclasses
    from types import SimpleNamespace

    from paper_2508_04484_b200 import raytracer as rt
    from paper_2508_04484_b200.driver import run_bundle
    from paper_2508_04484_b200.problem import ProblemBundle, UncollidedSlices

    b = ProblemBundle.load(ROOT / "tests" / "golden" / "bundle_config1.npz")
    run_bundle(b, max_steps=5)  # warm the kernels / allocations
    # the beam's uncollided flux traced on the device (441 rays, the reference's
    # water operator for this 90 MeV energy space), checked against the
    # reference-traced table of the bundle
    W = np.load(ROOT / "tests" / "golden" / "water_ops90.npz")
    sp = W["space"]
    space = rt.EnergySpace(float(sp[0]), float(sp[1]), int(sp[2]), int(sp[3]))
    nx, ny, nz = b.shape
    grid = SimpleNamespace(nx=nx, ny=ny, nz=nz, dx=b.spacing[0], dy=b.spacing[1],
                           dz=b.spacing[2], origin=tuple(b.origin))
    beam = SimpleNamespace(direction=(0.0, 0.0, 1.0), energy_mev=90.0,
                           position_cm=(1.0, 1.0, 0.0), weight=1.0, sigma_xy_cm=0.3,
                           sigma_e_mev=0.9)
    keys = np.zeros(b.n_cells, dtype=np.int32)
    args = (beam, grid, space, keys, {0: W["g"]}, {0: float(W["smin"])}, 21, 3.0, 0.01)
    rt.trace_beam_ops(*args)  # warm-up
    t0 = time.perf_counter()
    flux = rt.trace_beam_ops(*args)
    t_trace = time.perf_counter() - t0
    ref_vals = b.fluxes[0].values
    trace_dev = float(np.abs(flux.values - ref_vals).max() / np.abs(ref_vals).max())
    b = dataclasses.replace(b, fluxes=[UncollidedSlices(flux.values, flux.residual_energy,
                                                        space.e_min, space.e_max)])
    # the energy loop + the uncollided group-sum tally, twice: the faster run is
    # reported (one run measured 1.5x slower on one box than both runs of
    # another; the first full run also pays any remaining first-use costs)
    t_runs = []
    for _ in range(2):
        t0 = time.perf_counter()
        res = run_bundle(b)
        t_runs.append(time.perf_counter() - t0)
    t_gpu = min(t_runs)
    steps = len(res.rank_history)
    out = {"workload": "config 1: 1 x 20 x 70 water (2 cm x 1 mm), P7 (m=64), fixed rank 20, 573 steps, 1 beam",
           "gpu_s": t_trace + t_gpu, "trace_s": t_trace, "loop_and_tally_s": t_gpu,
           "trace_max_rel_dev_vs_reference": trace_dev,
           "gpu_steps_per_s": steps / t_gpu, "steps": steps, "loop_runs_s": t_runs,
           "assembly": "problem assembly is the reference's host code (unchanged; 1.0 s on the "
                       "build host, SURVEY.md §6.2) -- not on the device path, not timed here",
           "reference_per_beam_s": 21.6}
    if with_cpu:
        env = dict(os.environ)
        res_cpu = subprocess.run(
            [sys.executable, "-c",
             "import sys,time,json; sys.path.insert(0, %r)\n"
             "from oracle import dlra_np\n"
             "from paper_2508_04484_b200.problem import ProblemBundle\n"
             "b = ProblemBundle.load(%r)\n"
             "t = time.perf_counter(); dlra_np.run_energy_loop(b)\n"
             "print(json.dumps({'s': time.perf_counter() - t}))"
             % (str(ROOT), str(ROOT / "tests" / "golden" / "bundle_config1.npz"))],
            capture_output=True, text=True, env=env, timeout=600)
        if res_cpu.returncode == 0:
            t_cpu = json.loads(res_cpu.stdout.strip().splitlines()[-1])["s"]
            out["cpu_port_s"] = t_cpu
            out["cpu_kind"] = "port (numpy oracle of the reference loop)"
    return out


def host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


# ----------------------------------------------------------------- main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--rank", type=int, default=20)
    ap.add_argument("--nside", type=int, default=256)
    ap.add_argument("--phantom", default="water", choices=["water", "slabs"],
                    help="slabs: SURVEY.md §8(d) config 3 (use with --nside 512)")
    ap.add_argument("--cpu-sample", action="store_true")
    ap.add_argument("--cpu-steps", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-config1", action="store_true",
                    help="skip the config-1 per-beam dose timing (profiling runs)")
    args = ap.parse_args()
    if args.cpu_sample:
        return cpu_sample_main(args)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank_id = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch
        import torch.distributed as dist

        # one process per GPU; NCCL carries the barriers and the max-over-ranks
        # timing reduction (the replicas exchange no data)
        if args.impl != "reference" and torch.cuda.is_available():
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")

    config = {"workload": f"{args.nside}^3 homogeneous water, h=0.025 cm, P19 Fokker-Planck, "
                          f"70 MeV +z pencil beam, fixed rank {args.rank}, CFL 0.2, "
                          "steps from floor(n_steps/3)",
              "grid": [args.nside] * 3, "pn_order": 19, "moments": 400, "rank": args.rank,
              "model": "fokker-planck", "n_gpus": args.gpus,
              **({"workload": f"{args.nside}^3 z-slabs water [0,3) / bone +1200 HU [3,4) / "
                              "lung -700 HU [4,7) cm / water, h=0.025 cm, P7 Boltzmann, 100 MeV "
                              f"+z pencil beam, fixed rank {args.rank}, CFL 0.2, steps from "
                              "floor(n_steps/3)", "pn_order": 7, "moments": 64,
                  "model": "boltzmann"} if args.phantom == "slabs" else {}),
              "l2": "inputs larger than L2 (U is n x r doubles = 2.7 GB per factor)",
              "parallelism": f"z-slabs x{world} (NCCL halo planes + Gram allreduce)"
              if world > 1 else "single"}

    if args.impl == "reference":
        if rank_id != 0:
            return
        threads = host_threads()
        # one subprocess: W + K energy steps of the port at 64^3 (each a bounded
        # sample of the workload); the first W are discarded
        cb = run_cpu_sample(threads, max(1, args.steps), args.rank, args.nside, args.phantom)
        v = cb["value"]
        line = {"metric": metric_name(args.nside, args.rank, args.phantom), "value": v,
                "unit": UNIT, "n_gpus": args.gpus,
                "steps": cb["timed"]["steps"], "warmup": 0,
                "ms_per_step": 1000.0 / v, "higher_is_better": True, "scaling": "weak",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config,
                "impl": "reference", "extrapolated": True,
                "timed_sample": dict(cb["timed"], note=(
                    f"steps counts energy steps actually run, at {CPU_SIDE}^3; ms_per_step "
                    f"is the {args.nside}^3 step time extrapolated by cell count")),
                "cpu_baseline": cb,
                "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    import torch

    from paper_2508_04484_b200 import _lib

    torch.cuda.set_device(local)
    slab, cid = None, None
    if world > 1:
        # one joint solve, z-slab sharded: halo planes + Gram allreduces over NCCL
        from paper_2508_04484_b200 import _lib as plib
        from paper_2508_04484_b200 import slabs

        obj = [plib.comm_unique_id() if rank_id == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        cid = obj[0]
        slab = slabs.plan(args.nside, args.nside, args.nside, world, rank_id)
    wl = Workload(nside=args.nside, rank=args.rank, device=local, slab=slab, comm_id=cid,
                  **PHANTOM_KW[args.phantom])
    h = wl.solver.h
    n_steps_total = len(wl.edges) - 1
    if wl.k0 + args.warmup + args.steps > n_steps_total:
        raise SystemExit("not enough energy steps for warmup + steps")
    for _ in range(args.warmup):
        wl.step()
    h.call("pnd_synchronize")
    if dist:
        dist.barrier()
    clocks = ClockSampler(local)
    lc0 = np.zeros(1, dtype=np.int64)
    h.call("pnd_launch_count", _lib.ptr(lc0))
    h.call("pnd_timing", 1)
    t_host0 = time.perf_counter()
    h.call("pnd_event_record", 0)
    ranks = []
    for _ in range(args.steps):
        out = wl.step()
        ranks.append(int(out[2]))
    h.call("pnd_event_record", 1)
    h.call("pnd_synchronize")
    t_host = time.perf_counter() - t_host0
    ms = np.zeros(1)
    h.call("pnd_event_elapsed", 0, 1, _lib.ptr(ms))
    lc1 = np.zeros(1, dtype=np.int64)
    h.call("pnd_launch_count", _lib.ptr(lc1))
    nph = len(_lib.PHASES)
    ph_ms = np.zeros(nph)
    ph_cnt = np.zeros(nph, dtype=np.int32)
    h.call("pnd_timing_get", nph, _lib.ptr(ph_ms), _lib.ptr(ph_cnt))
    # e2e: the same K steps through the public API with the step's inputs formed
    # on the host (problem.py's coefficient restatement) and copied host->device
    # every step by the C-ABI, the step's scalars read back every step
    wl.solver.device_coefficients = False
    h.call("pnd_synchronize")
    if dist:
        dist.barrier()
    t_e2e0 = time.perf_counter()
    for _ in range(args.steps):
        out = wl.step()
    h.call("pnd_synchronize")
    t_host = time.perf_counter() - t_e2e0
    wl.solver.device_coefficients = True
    clk = clocks.stop()
    dev_s = ms[0] / 1000.0
    if dist:
        t = torch.tensor([dev_s, t_host], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_s, t_host = float(t[0]), float(t[1])
    if rank_id != 0:
        dist.barrier()
        return
    # one joint solve over all ranks: a step is one energy step of the whole grid
    value = args.steps / dev_s
    e2e = args.steps / t_host

    b = wl.bundle
    model = phase_model(b.n_cells, args.rank, b.n_moments, 2 * 3)
    phases = {}
    for i, nm in enumerate(_lib.PHASES):
        if ph_cnt[i]:
            phases[nm] = {"ms_per_step": float(ph_ms[i] / args.steps),
                          "share": float(ph_ms[i] / ph_ms.sum()),
                          "marks_per_step": float(ph_cnt[i] / args.steps)}
    fp64 = measure_fp64_peak()
    # dominant kernel family by time
    dom = max((nm for nm in model if nm in phases), key=lambda nm: phases[nm]["ms_per_step"])
    launches_per_step = {"kstage": 4, "s_gram": 1, "l_gram": 1, "tsqr_n": 2}[dom]
    per_launch_ms = phases[dom]["ms_per_step"] / launches_per_step
    achieved = model[dom]["flops"] / (per_launch_ms * 1e-3) / 1e12
    traffic = roofline_traffic(args.nside, args.rank, args.phantom, dom)
    roofline = {"bound": "tensor", "kernel": dom, "achieved": achieved, "peak": fp64,
                "unit": "TFLOP/s", "frac": achieved / fp64, "traffic": traffic,
                "peak_source": "FP64 cuBLAS DGEMM 8192^3 measured in this run (MEASURED_PEAKS.json "
                               "has no FP64 entry)",
                "algorithmic_per_launch": model[dom],
                "hbm_frac_of_measured": (model[dom]["bytes"] / (per_launch_ms * 1e-3) / 1e9)
                / json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
                if (ROOT / "MEASURED_PEAKS.json").exists() else None}
    cpu_baseline = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            cpu_baseline = run_cpu_sample(host_threads(), 2, args.rank, args.nside,
                                          args.phantom)
        except Exception as exc:  # noqa: BLE001
            cpu_baseline = {"error": str(exc)[:300]}
    per_beam = None
    if world == 1 and not args.no_config1:
        try:
            per_beam = config1_dose_time(with_cpu=not args.no_cpu_baseline)
        except Exception as exc:  # noqa: BLE001
            per_beam = {"error": str(exc)[:300]}
    line = {
        "metric": metric_name(args.nside, args.rank, args.phantom), "value": value, "unit": UNIT,
        "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1000.0 * dev_s / args.steps,
        "higher_is_better": True, "scaling": "strong" if world > 1 else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": config,
        "e2e": {"value": e2e, "unit": UNIT, "h2d_bytes_per_step": wl.h2d_bytes_per_step(),
                "d2h_bytes_per_step": wl.d2h_bytes_per_step(),
                "path": "paper_2508_04484_b200.driver.DeviceSolver.set_coefficients + step "
                        "(device_coefficients=False): per step the host forms the class "
                        "stopping powers, scattering diagonals, sigma_t and flux lerp weights "
                        "and the C-ABI copies them host->device; the step scalars are read "
                        "back device->host every step",
                "device_path_ms_per_step": 1000.0 * dev_s / args.steps},
        "gpu_launches": int(lc1[0] - lc0[0]),
        "clocks": clk,
        "roofline": roofline,
        "cpu_baseline": cpu_baseline,
        "phases": phases,
        "per_beam_dose_time": per_beam,
        "ranks": sorted(set(ranks)),
        "fp64_dgemm_tflops": fp64,
        "reference_step_count": n_steps_total,
    }
    print(json.dumps(line))
    if dist:
        dist.barrier()


if __name__ == "__main__":
    main()
