"""Generate the golden fixtures under tests/golden/ from the reference.

Runs HERE only (the reference tree exists in this container, not on the GPU
box). It imports the unmodified reference package from
/root/reference/pkg/src, runs it on small seeded inputs and writes the
inputs and outputs as .npz fixtures. The fixtures travel with the repo; the
tests, smoke() and bench.py read only the fixtures, never the reference.

    PYTHONDONTWRITEBYTECODE=1 OPENBLAS_NUM_THREADS=1 python tools/make_golden.py

OPENBLAS_NUM_THREADS is pinned because the reference's collided output
depends on the BLAS thread count; the versions used are
recorded in every fixture under the key `provenance`.
"""

import json
import os
import sys
import time
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parents[1] / "tests" / "golden"

sys.path.insert(0, str(REF_SRC))
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import scipy  # noqa: E402

from pndose import angular, dlra, driver, raytracer, spatial  # noqa: E402
from pndose.angular import PNOperators  # noqa: E402
from pndose.fullrank import fullrank_scattering_step, fullrank_streaming_step  # noqa: E402

from paper_2508_04484_b200.problem import export_problem  # noqa: E402


def provenance():
    return json.dumps(
        {
            "numpy": np.__version__,
            "scipy": scipy.__version__,
            "openblas_threads": os.environ.get("OPENBLAS_NUM_THREADS"),
            "reference": str(REF_SRC),
            "generated": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
        }
    )


def save(name, **arrays):
    arrays["provenance"] = np.array(provenance())
    path = OUT / name
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({path.stat().st_size / 1024:.1f} KiB)")


def ops_arrays(ops, prefix=""):
    return {
        prefix + "eig_v": np.stack(ops.eig_v),
        prefix + "lam_plus": np.stack(ops.lam_plus),
        prefix + "lam_minus": np.stack(ops.lam_minus),
    }


# --------------------------------------------------------------- angular
def make_angular():
    out = {}
    for n_max in (1, 2, 3, 5, 7):
        ops = PNOperators.build(n_max)
        out[f"a_{n_max}"] = np.stack(ops.matrices)
        out[f"spectral_radius_{n_max}"] = np.array(ops.spectral_radius)
        for d in range(3):
            v = ops.eig_v[d]
            out[f"aplus_{n_max}_{d}"] = (v * ops.lam_plus[d]) @ v.T
            out[f"aminus_{n_max}_{d}"] = (v * ops.lam_minus[d]) @ v.T
        out[f"tm_{n_max}"] = angular.beam_projection(n_max, (0.0, 0.6, 0.8))
        out[f"fp_{n_max}"] = angular.scattering_matrix_fp(2.5e-3, n_max)
    save("angular.npz", **out)


# --------------------------------------------------------------- kernels
KERNEL_CASES = [
    # name, grid, n_max, r
    ("g3d", spatial.Grid3D(5, 4, 6, 0.2, 0.25, 0.2), 2, 3),
    ("g3d_b", spatial.Grid3D(7, 6, 5, 0.1, 0.15, 0.3), 3, 5),
    ("gz", spatial.Grid3D(1, 1, 12, 1.0, 1.0, 0.1), 2, 2),
    ("gyz", spatial.Grid3D(1, 6, 7, 2.0, 0.1, 0.1), 3, 4),
    ("gx3", spatial.Grid3D(3, 1, 1, 0.3, 1.0, 1.0), 1, 1),
]


def make_kernels():
    out = {}
    for name, grid, n_max, r in KERNEL_CASES:
        rng = np.random.default_rng(sum(name.encode()) * 31 + r)
        ops = PNOperators.build(n_max)
        stencils = spatial.build_stencils(grid)
        n, m = grid.n_cells, ops.basis.size
        inv_s = 1.0 / rng.uniform(8.0, 20.0, n)
        ctx = dlra.StreamingContext(inv_s, stencils, ops)
        u_full = rng.standard_normal((n, m))
        u0 = dlra.orthonormal_columns(rng.standard_normal((n, r)))
        v0 = dlra.orthonormal_columns(rng.standard_normal((m, r)))
        k = rng.standard_normal((n, r))
        l = rng.standard_normal((m, r))
        s = rng.standard_normal((r, r))
        kf = ctx._moment_factors(v0)
        lf = ctx.l_step_factors(u0)
        sf = ctx.s_step_factors(u0, v0)
        p = name + "_"
        out.update(
            {
                p + "grid": np.array([grid.nx, grid.ny, grid.nz, grid.dx, grid.dy, grid.dz]),
                p + "n_max": np.array(n_max),
                p + "inv_s": inv_s,
                p + "u_full": u_full,
                p + "apply_streaming": spatial.apply_streaming(u_full, inv_s, stencils, ops),
                p + "u0": u0,
                p + "v0": v0,
                p + "k": k,
                p + "l": l,
                p + "s": s,
                p + "k_rhs": ctx.k_rhs(k, kf),
                p + "l_rhs": ctx.l_rhs(l, lf),
                p + "s_rhs": ctx.s_rhs(s, u0, sf),
                # (Ds+- U0)^T U0 per active axis, stacked [axis][+/-]
                p + "q_grams": np.array([[f[2], f[3]] for f in lf]),
                p + "active": np.array(ctx.active_axes),
            }
        )
        out.update(ops_arrays(ops, p))
    save("kernels.npz", **out)


# --------------------------------------------------------------- steps
def make_steps():
    out = {}
    # streaming: full-rank-ish well-conditioned state on a small 3-D grid
    for name, grid, n_max, r, dt in (
        ("str3d", spatial.Grid3D(6, 5, 7, 0.2, 0.2, 0.25), 2, 3, 0.02),
        ("str2d", spatial.Grid3D(1, 8, 9, 2.0, 0.1, 0.1), 3, 4, 0.01),
        ("strz", spatial.Grid3D(1, 1, 64, 1.0, 1.0, 0.1), 3, 2, 0.05),
    ):
        rng = np.random.default_rng(len(name) * 1000 + r)
        ops = PNOperators.build(n_max)
        stencils = spatial.build_stencils(grid)
        n, m = grid.n_cells, ops.basis.size
        inv_s = 1.0 / rng.uniform(8.0, 20.0, n)
        ctx = dlra.StreamingContext(inv_s, stencils, ops)
        u0 = dlra.orthonormal_columns(rng.standard_normal((n, r)))
        v0 = dlra.orthonormal_columns(rng.standard_normal((m, r)))
        s0 = np.diag(np.logspace(0, -2, r)) + 0.01 * rng.standard_normal((r, r))
        st = dlra.LowRankState(u0, s0, v0)
        aug = dlra.streaming_step(st, dt, ctx)
        tr, tail = dlra.truncate(aug, dlra.TruncationPolicy(0.0, rank_min=1, rank_max=2 * r))
        trr, tailr = dlra.truncate(aug, dlra.TruncationPolicy(1e300, rank_min=r, rank_max=r))
        full = fullrank_streaming_step(st.matrix(), dt, ctx)
        p = name + "_"
        out.update(
            {
                p + "grid": np.array([grid.nx, grid.ny, grid.nz, grid.dx, grid.dy, grid.dz]),
                p + "n_max": np.array(n_max),
                p + "dt": np.array(dt),
                p + "inv_s": inv_s,
                p + "u0": u0,
                p + "s0": s0,
                p + "v0": v0,
                p + "aug_matrix": aug.matrix(),
                p + "aug_sigma": np.linalg.svd(aug.s, compute_uv=False),
                p + "trunc0_matrix": tr.matrix(),
                p + "trunc0_rank": np.array(tr.rank),
                p + "trunc0_tail": np.array(tail),
                p + "truncr_matrix": trr.matrix(),
                p + "truncr_tail": np.array(tailr),
                p + "full_matrix": full,
            }
        )
        out.update(ops_arrays(ops, p))

    # scattering: random contexts (homogeneous / heterogeneous, with sources)
    for name, n, n_max, r, homog, n_src in (
        ("scat_h", 60, 2, 3, True, 1),
        ("scat_x", 80, 3, 5, False, 2),
        ("scat_max", 200, 3, 16, True, 1),
    ):
        rng = np.random.default_rng(n * 7 + r)
        m = (n_max + 1) ** 2
        if homog:
            weights = np.tile(np.abs(rng.standard_normal(12)), (n, 1)) * 1e22
        else:
            weights = np.abs(rng.standard_normal((n, 12))) * 1e22
        g_diags = np.abs(rng.standard_normal((12, m))) * 1e-28
        sigma_t = g_diags[:, 0] + np.abs(rng.standard_normal(12)) * 1e-28
        inv_s = 1.0 / rng.uniform(8.0, 20.0, n)
        sources = [
            (np.abs(rng.standard_normal(n)), rng.standard_normal(m)) for _ in range(n_src)
        ]
        ctx = dlra.ScatteringContext(weights, inv_s, g_diags, sigma_t, sources)
        if r == m:
            uu, ss, vvt = np.linalg.svd(rng.standard_normal((n, m)), full_matrices=False)
            u0, s0, v0 = uu, np.diag(ss), vvt.T
        else:
            u0 = dlra.orthonormal_columns(rng.standard_normal((n, r)))
            v0 = dlra.orthonormal_columns(rng.standard_normal((m, r)))
            s0 = np.diag(np.logspace(0, -1, r)) + 0.05 * rng.standard_normal((r, r))
        st = dlra.LowRankState(u0, s0, v0)
        dt = 0.3
        aug = dlra.scattering_step(st, dt, ctx)
        tr, tail = dlra.truncate(aug, dlra.TruncationPolicy(0.0, rank_min=1, rank_max=2 * r))
        full = fullrank_scattering_step(st.matrix(), dt, ctx)
        p = name + "_"
        out.update(
            {
                p + "n_max": np.array(n_max),
                p + "dt": np.array(dt),
                p + "weights": weights,
                p + "inv_s": inv_s,
                p + "g_diags": g_diags,
                p + "sigma_t": sigma_t,
                p + "psi": np.array([s[0] for s in sources]),
                p + "tm": np.array([s[1] for s in sources]),
                p + "u0": u0,
                p + "s0": s0,
                p + "v0": v0,
                p + "aug_matrix": aug.matrix(),
                p + "aug_shape": np.array([aug.u.shape[1], aug.v.shape[1]]),
                p + "aug_sigma": np.linalg.svd(aug.s, compute_uv=False),
                p + "trunc0_matrix": tr.matrix(),
                p + "trunc0_rank": np.array(tr.rank),
                p + "full_matrix": full,
            }
        )

    # truncation rule cases (dlra.py:90-115)
    cases = []
    rng = np.random.default_rng(23)
    for i in range(12):
        q = 8
        sig = np.sort(np.abs(rng.standard_normal(q)) * np.exp(-np.arange(q)))[::-1]
        theta = 10.0 ** rng.uniform(-4, 0)
        rmin, rmax = 1 + i % 3, q
        s = np.diag(sig)
        st = dlra.LowRankState(np.eye(q), s, np.eye(q))
        tr, tail = dlra.truncate(st, dlra.TruncationPolicy(theta, rmin, rmax))
        cases.append([theta, rmin, rmax, tr.rank, tail] + list(sig))
    out["trunc_cases"] = np.array(cases)
    save("steps.npz", **out)


# --------------------------------------------------------------- traversal
def make_traverse():
    rays = []
    grids = {
        "a": spatial.Grid3D(4, 4, 10, 0.1, 0.1, 0.1),
        "b": spatial.Grid3D(5, 5, 5, 0.2, 0.2, 0.2),
        "c": spatial.Grid3D(20, 20, 70, 0.1, 0.1, 0.1),
        "d": spatial.Grid3D(7, 9, 11, 0.13, 0.07, 0.21, origin=(-0.3, 0.2, -0.1)),
        "e": spatial.Grid3D(1, 20, 70, 2.0, 0.1, 0.1),
    }
    rng = np.random.default_rng(99)
    out = {}
    for gname, g in grids.items():
        (x0, x1), (y0, y1), (z0, z1) = g.extent()
        origins, dirs = [], []
        # axis-aligned, diagonal and random rays, plus beam-like bundles
        for _ in range(60):
            o = np.array([rng.uniform(x0 - 0.2, x1 + 0.2), rng.uniform(y0 - 0.2, y1 + 0.2),
                          z0 - rng.uniform(0.01, 0.5)])
            d = rng.standard_normal(3)
            d[2] = abs(d[2]) + 0.1
            d /= np.linalg.norm(d)
            origins.append(o)
            dirs.append(d)
        for axis in range(3):
            for sgn in (1.0, -1.0):
                d = np.zeros(3)
                d[axis] = sgn
                for _ in range(6):
                    o = np.array([rng.uniform(x0, x1), rng.uniform(y0, y1), rng.uniform(z0, z1)])
                    o[axis] = (x0, y0, z0)[axis] - 0.3 if sgn > 0 else (x1, y1, z1)[axis] + 0.3
                    origins.append(o)
                    dirs.append(d.copy())
        d = np.array([1.0, 1.0, 1.0]) / np.sqrt(3.0)
        origins.append(np.array([x0, y0, z0]) - 0.1 * d)
        dirs.append(d)
        # a stratified pencil beam bundle (the reference's own start points)
        beam = raytracer.BeamSource((0.0, 0.6, 0.8), 50.0, (0.5 * (x0 + x1), y0, z0), sigma_xy_cm=0.2)
        e1, e2 = beam.transverse_frame()
        offsets, _ = raytracer.stratified_ray_offsets(beam.sigma_xy_cm, 7, 3.0)
        for off in offsets:
            origins.append(np.asarray(beam.position_cm) + off[0] * e1 + off[1] * e2)
            dirs.append(np.asarray(beam.direction))
        cells, t0, t1, offs = [], [], [], [0]
        for o, d in zip(origins, dirs):
            path = raytracer.traverse_grid(g, o, d)
            for c, a, b in path:
                cells.append(c)
                t0.append(a)
                t1.append(b)
            offs.append(len(cells))
        p = gname + "_"
        out.update(
            {
                p + "grid": np.array([g.nx, g.ny, g.nz, g.dx, g.dy, g.dz] + list(g.origin)),
                p + "origins": np.array(origins),
                p + "dirs": np.array(dirs),
                p + "cells": np.array(cells, dtype=np.int64),
                p + "t0": np.array(t0),
                p + "t1": np.array(t1),
                p + "offsets": np.array(offs, dtype=np.int64),
            }
        )
    out["grids"] = np.array(list(grids))
    save("traverse.npz", **out)


# --------------------------------------------------------------- end to end
def smoke_raw(**over):
    raw = {
        "name": "smoke",
        "grid": {"nx": 8, "ny": 8, "nz": 12,
                 "delta_x_cm": 0.25, "delta_y_cm": 0.25, "delta_z_cm": 0.25},
        "phantom": {"background_hu": 0.0},
        "beams": [{"direction": [0, 0, 1], "energy_mev": 20.0, "position_cm": [1.0, 1.0, 0.0]}],
        "pn_order": 3,
        "transport": {"cfl_number": 0.2},
        "energy": {"groups": 64},
        "rays": {"n_side": 5},
    }
    raw.update(over)
    return raw


def config1_raw():
    import yaml

    with open("/root/reference/pkg/configs/homogeneous_90MeV.yaml") as fh:
        raw = yaml.safe_load(fh)
    raw["grid"]["nx"] = 1
    raw["grid"]["delta_x_cm"] = 2.0
    raw["transport"].update({"truncation_tolerance": 1e300, "rank_min": 20, "rank_max": 20})
    raw.pop("output", None)
    return raw


def lockstep_raw():
    return {
        "grid": {"nx": 8, "ny": 8, "nz": 8,
                 "delta_x_cm": 0.25, "delta_y_cm": 0.25, "delta_z_cm": 0.25},
        "phantom": {"background_hu": 0.0},
        "beams": [{"direction": [0, 0, 1], "energy_mev": 20.0, "position_cm": [1.0, 1.0, 0.0]}],
        "pn_order": 3,
        "transport": {"cfl_number": 0.0003, "truncation_tolerance": 0.0,
                      "rank_min": 16, "rank_max": 16},
        "energy": {"e_min_mev": 19.0, "e_max_mev": 21.0, "groups": 64},
        "rays": {"n_side": 5},
    }


def hetero_raw():
    raw = smoke_raw(name="hetero")
    raw["grid"] = {"nx": 8, "ny": 8, "nz": 16,
                   "delta_x_cm": 0.25, "delta_y_cm": 0.25, "delta_z_cm": 0.25}
    raw["phantom"] = {
        "background_hu": 0.0,
        "boxes": [
            {"origin_cm": [0, 0, 1.0], "size_cm": [2, 2, 0.75], "hu": 1200.0},
            {"origin_cm": [1.0, 0, 2.0], "size_cm": [1, 2, 1.0], "hu": -700.0},
        ],
    }
    raw["beams"] = [
        {"direction": [0, 0, 1], "energy_mev": 25.0, "position_cm": [1.0, 1.0, 0.0]},
        {"direction": [0, 0.6, 0.8], "energy_mev": 22.0, "position_cm": [1.0, 0.3, 0.0],
         "weight": 0.5},
    ]
    raw["transport"] = {"cfl_number": 0.2, "truncation_tolerance": 1e300,
                        "rank_min": 6, "rank_max": 6}
    return raw


def hetero_beam_raw(i):
    """One beam of the heterogeneous two-beam case, with the joint run's
    energy grid pinned (e_max of both beams): a subset of the beam-batched
    partition {0}, {1} (SURVEY.md §8(e) "Beams")."""
    raw = hetero_raw()
    raw["name"] = f"hetero_b{i}"
    raw["beams"] = [raw["beams"][i]]
    e_max = max(b["energy_mev"] * (1.0 + 5.0 * 0.01) for b in hetero_raw()["beams"])
    raw["energy"] = dict(raw.get("energy", {}), e_max_mev=e_max)
    return raw


def fp_raw():
    raw = smoke_raw(name="fp", model="fokker-planck")
    raw["physics"] = {"fp_correction_scale": 0.5}
    raw["transport"] = {"cfl_number": 0.2, "truncation_tolerance": 1e300,
                        "rank_min": 4, "rank_max": 4}
    return raw


def rank1_raw():
    raw = smoke_raw(name="rank1")
    raw["transport"] = {"cfl_number": 0.2, "truncation_tolerance": 1e-6,
                        "rank_min": 1, "rank_max": 40}
    return raw


def fp19_raw():
    """The benchmarked physics (BASELINE configs[1]: water, P19 Fokker-Planck,
    m = 400, fixed rank 20) on a 10 x 10 x 12 grid the reference finishes in
    seconds per step."""
    return {
        "name": "fp19",
        "grid": {"nx": 10, "ny": 10, "nz": 12,
                 "delta_x_cm": 0.1, "delta_y_cm": 0.1, "delta_z_cm": 0.1},
        "phantom": {"background_hu": 0.0},
        "beams": [{"direction": [0, 0, 1], "energy_mev": 30.0, "position_cm": [0.5, 0.5, 0.0],
                   "sigma_xy_cm": 0.2}],
        "model": "fokker-planck",
        "pn_order": 19,
        "transport": {"cfl_number": 0.2, "truncation_tolerance": 1e300,
                      "rank_min": 20, "rank_max": 20},
        "energy": {"groups": 128},
        "rays": {"n_side": 11},
    }


def slabs7_raw():
    """BASELINE configs[2]'s physics (water / bone / lung z-slabs, Boltzmann
    P7, fixed rank 20) on a 10 x 10 x 24 grid: water z < 0.6 cm, bone
    [0.6, 0.9), lung [0.9, 1.5), water beyond."""
    return {
        "name": "slabs7",
        "grid": {"nx": 10, "ny": 10, "nz": 24,
                 "delta_x_cm": 0.1, "delta_y_cm": 0.1, "delta_z_cm": 0.1},
        "phantom": {
            "background_hu": 0.0,
            "boxes": [
                {"origin_cm": [0, 0, 0.6], "size_cm": [1, 1, 0.3], "hu": 1200.0},
                {"origin_cm": [0, 0, 0.9], "size_cm": [1, 1, 0.6], "hu": -700.0},
            ],
        },
        "beams": [{"direction": [0, 0, 1], "energy_mev": 40.0, "position_cm": [0.5, 0.5, 0.0],
                   "sigma_xy_cm": 0.2}],
        "model": "boltzmann",
        "pn_order": 7,
        "transport": {"cfl_number": 0.2, "truncation_tolerance": 1e300,
                      "rank_min": 20, "rank_max": 20},
        "energy": {"groups": 128},
        "rays": {"n_side": 11},
    }


def run_lockstep_record(tag, raw, record):
    """The reference's own energy loop (driver.py:577-622, the same calls in
    the same order as run_simulation) recording, at the steps in `record`,
    the input state, the frozen contexts and the factors after each substep
    and truncation: the T2 per-step fixtures (lock_<tag>.npz). Each substep
    also runs from the reference's own previous output, so a GPU test can
    check every substep of every recorded step in isolation."""
    config = driver.ProblemConfig.from_dict(raw)
    problem = driver.assemble_problem(config)
    fluxes = driver.trace_all_beams(problem)
    t_ms = [angular.beam_projection(config.pn_order, b.direction) for b in config.beams]
    edges = driver.pseudo_time_edges(problem)
    n, m = problem.n_cells, problem.n_moments
    policy = dlra.TruncationPolicy(config.truncation_tolerance, rank_min=config.rank_min,
                                   rank_max=config.rank_max)
    state = dlra.LowRankState.zero(n, m, min(config.rank_min, n, m), seed=config.seed)
    out = {"steps": np.array(sorted(record)), "edges": edges,
           "weights": np.asarray(problem.material.atomic_densities),
           "t_ms": np.stack(t_ms)}
    g = problem.grid  # the P_N operators are the bundle's (bundle_<tag>.npz)
    out["grid"] = np.array([g.nx, g.ny, g.nz, g.dx, g.dy, g.dz])
    for k in range(max(record) + 1):
        e_hi, e_lo = edges[k], edges[k + 1]
        dt = e_hi - e_lo
        sc, cc, _ = driver.step_contexts(problem, fluxes, t_ms, e_hi, e_lo)
        p = f"k{k}_"
        if k in record:
            out.update({p + "u": state.u, p + "s": state.s, p + "v": state.v,
                        p + "dt": np.array(dt), p + "inv_s": sc.inv_s,
                        p + "g_diags": cc.g_diags, p + "sigma_t": cc.sigma_t,
                        p + "psi": np.array([s[0] for s in cc.sources])})
        state = dlra.streaming_step(state, dt, sc)
        if k in record:
            out.update({p + "sa_u": state.u, p + "sa_s": state.s, p + "sa_v": state.v})
        if config.truncate_after in ("streaming", "both"):
            state, tail = dlra.truncate(state, policy)
            if k in record:
                out.update({p + "st_u": state.u, p + "st_s": state.s, p + "st_v": state.v,
                            p + "st_tail": np.array(tail)})
        state = dlra.scattering_step(state, dt, cc)
        if k in record:
            out.update({p + "ca_u": state.u, p + "ca_s": state.s, p + "ca_v": state.v})
        if config.truncate_after in ("scattering", "both"):
            state, tail = dlra.truncate(state, policy)
            if k in record:
                out.update({p + "ct_u": state.u, p + "ct_s": state.s, p + "ct_v": state.v,
                            p + "ct_tail": np.array(tail)})
    save(f"lock_{tag}.npz", **out)


def run_e2e(tag, raw, with_contexts=True):
    t0 = time.perf_counter()
    config = driver.ProblemConfig.from_dict(raw)
    problem = driver.assemble_problem(config)
    fluxes = driver.trace_all_beams(problem)
    t_ms = [angular.beam_projection(config.pn_order, b.direction) for b in config.beams]
    bundle = export_problem(problem, fluxes, t_ms)
    save(f"bundle_{tag}.npz", **bundle)

    res = driver.run_simulation(config, solver="dlra")
    unc = driver.uncollided_dose(problem, fluxes)
    edges = driver.pseudo_time_edges(problem)
    out = {
        "deposited": res.dose.deposited,
        "dose": res.dose.dose,
        "uncollided": unc,
        "rank_history": np.array([[k, e, r] for k, e, r in res.rank_history]),
        "edges": edges,
        "diagnostics": np.array(json.dumps(driver._jsonable(res.diagnostics))),
        "runtime_s": np.array(time.perf_counter() - t0),
    }
    if with_contexts:
        # per-step contexts at a few steps: pins the host coefficient path
        steps = sorted({0, 1, len(edges) // 3, len(edges) - 2})
        out["ctx_steps"] = np.array(steps)
        for k in steps:
            sc, cc, s_field = driver.step_contexts(problem, fluxes, t_ms, edges[k], edges[k + 1])
            out[f"ctx{k}_inv_s"] = sc.inv_s
            out[f"ctx{k}_g_diags"] = cc.g_diags
            out[f"ctx{k}_sigma_t"] = cc.sigma_t
            out[f"ctx{k}_psi"] = np.array([s[0] for s in cc.sources])
            out[f"ctx{k}_s_field"] = s_field
    save(f"e2e_{tag}.npz", **out)
    print(f"  {tag}: {res.diagnostics['n_steps']} steps in {time.perf_counter() - t0:.1f}s")


def make_e2e(which):
    cases = {
        "smoke": smoke_raw(),
        "config1": config1_raw(),
        "lockstep": lockstep_raw(),
        "hetero": hetero_raw(),
        "fp": fp_raw(),
        "rank1": rank1_raw(),
        "fp19": fp19_raw(),
        "hetero_b0": hetero_beam_raw(0),
        "hetero_b1": hetero_beam_raw(1),
        "slabs7": slabs7_raw(),
    }
    for tag, raw in cases.items():
        if which and tag not in which:
            continue
        run_e2e(tag, raw, with_contexts=(tag != "lockstep"))


def make_lock(which):
    """T2 per-step fixtures at the benchmarked physics (lock_<tag>.npz)."""
    cases = {"fp19": (fp19_raw(), {2, 25, 50}), "slabs7": (slabs7_raw(), {2, 150, 300})}
    for tag, (raw, record) in cases.items():
        if which and tag not in which:
            continue
        t0 = time.perf_counter()
        run_lockstep_record(tag, raw, record)
        print(f"  lock {tag}: {time.perf_counter() - t0:.1f}s")


def make_march():
    """One Crank-Nicolson march (raytracer.py:285-350) for the tracer tests."""
    space = raytracer.EnergyDGSpace(1.0, 31.5, 32, 2)

    def const(v):
        return lambda e: np.full_like(np.asarray(e, dtype=float), v)

    coeff = {0: (lambda e: 2.0 + 0.05 * np.asarray(e, dtype=float), const(0.04), const(0.3)),
             1: (const(4.0), None, None)}
    psi0 = raytracer.project_initial_spectrum(space, 30.0, 0.3)
    segs = [(0, 0.1, 0), (1, 0.07, 1), (2, 0.1, 0), (3, 0.013, 1)]
    recs, psi = raytracer.march_ray(space, segs, coeff, psi0)
    ops = {}
    for key in coeff:
        mass, g = raytracer.assemble_energy_operators(space, *coeff[key])
        ops[f"g_{key}"] = g
    save(
        "march.npz",
        mass=space.mass_diagonal(),
        psi0=psi0,
        psi_exit=psi,
        seg_len=np.array([s[1] for s in segs]),
        seg_key=np.array([s[2] for s in segs]),
        averages=np.array([r.group_averages for r in recs]),
        residual=np.array([r.residual_energy for r in recs]),
        s_min=np.array([float(coeff[k][0](np.array([1.0]))[0]) for k in (0, 1)]),
        **ops,
    )


def make_trace():
    """trace_all_beams (driver.py:398-449 -> raytracer.py:452-529) on the
    heterogeneous phantom with one axial and one oblique beam: the inputs the
    device tracer consumes (assembled energy operators per material key,
    s*(e_min), keys per cell, beam + ray parameters) and the reference's
    outputs (group flux per cell, residual energy per cell, live rays)."""
    config = driver.ProblemConfig.from_dict(hetero_raw())
    problem = driver.assemble_problem(config)
    captured = []
    orig = driver.trace_beam

    def spy(beam, grid, space, keys, coefficients, **kw):
        flux = orig(beam, grid, space, keys, coefficients, **kw)
        captured.append((beam, grid, space, np.asarray(keys), coefficients, kw, flux))
        return flux

    driver.trace_beam = spy
    try:
        driver.trace_all_beams(problem)
    finally:
        driver.trace_beam = orig
    out = {}
    for i, (beam, grid, space, keys, coeff, kw, flux) in enumerate(captured):
        p = f"b{i}_"
        uk = sorted(int(k) for k in np.unique(keys))
        for k in uk:
            mass, g = raytracer.assemble_energy_operators(space, *coeff[k])
            out[p + f"g_{k}"] = g
            out[p + f"smin_{k}"] = np.array(
                float(np.atleast_1d(coeff[k][0](np.array([space.e_min])))[0]))
        e1, e2 = beam.transverse_frame()
        offs, wts = raytracer.stratified_ray_offsets(beam.sigma_xy_cm, kw["n_side"],
                                                      kw["span_sigmas"])
        out.update({
            p + "keys": keys.astype(np.int32),
            p + "key_list": np.array(uk),
            p + "mass": space.mass_diagonal(),
            p + "space": np.array([space.e_min, space.e_max, space.n_groups, space.degree]),
            p + "grid": np.array([grid.nx, grid.ny, grid.nz, grid.dx, grid.dy, grid.dz,
                                  *grid.origin]),
            p + "beam": np.array([*beam.direction, beam.energy_mev, *beam.position_cm,
                                  beam.weight, beam.sigma_xy_cm, beam.sigma_e_mev]),
            p + "rays": np.array([kw["n_side"], kw["span_sigmas"], kw["max_step"]]),
            p + "frame": np.stack([e1, e2]),
            p + "offsets": offs,
            p + "weights": wts,
            p + "psi0": raytracer.project_initial_spectrum(space, beam.energy_mev,
                                                           beam.sigma_e_mev),
            p + "values": flux.values,
            p + "residual": flux.residual_energy,
            p + "n_rays": np.array(flux.n_rays),
        })
    out["n_beams"] = np.array(len(captured))
    save("trace.npz", **out)


TRACE40_CASES = {"deg0": (0.0,), "deg30": (30.0,), "beams4": (0.0, 30.0, 60.0, 90.0)}


def trace40_raw(angles):
    """BASELINE.md / SURVEY.md §6.2's tracer timing case: 40^3 water at 1 mm,
    121 rays per beam (n_side 11), 70 MeV beams in the y-z plane aimed at the
    grid centre from 2.5 cm outside it."""
    import math

    beams = []
    for deg in angles:
        th = math.radians(deg)
        d = (0.0, math.sin(th), math.cos(th))
        beams.append({"direction": list(d), "energy_mev": 70.0,
                      "position_cm": [2.0, 2.0 - 4.5 * d[1], 2.0 - 4.5 * d[2]]})
    return {
        "name": "trace40",
        "grid": {"nx": 40, "ny": 40, "nz": 40,
                 "delta_x_cm": 0.1, "delta_y_cm": 0.1, "delta_z_cm": 0.1},
        "phantom": {"background_hu": 0.0},
        "beams": beams,
        "pn_order": 3,
        "transport": {"cfl_number": 0.2},
        "energy": {"groups": 128},
        "rays": {"n_side": 11},
    }


def make_trace40():
    """Inputs and (sampled) outputs of the reference tracer on the 40^3 timing
    cases, with the reference's own trace_all_beams wall time on this host's
    CPU (the GPU box cannot run the reference): tools/trace_bench.py times the
    device tracer on the same inputs and checks it against these values."""
    out = {}
    rng = np.random.default_rng(40)
    sample = np.sort(rng.choice(40 ** 3, 4000, replace=False))
    out["sample"] = sample
    for tag, angles in TRACE40_CASES.items():
        config = driver.ProblemConfig.from_dict(trace40_raw(angles))
        problem = driver.assemble_problem(config)
        captured = []
        orig = driver.trace_beam
        calls = {"march": 0, "lu": 0}
        om, olu = raytracer.march_ray, raytracer.lu_factor

        def spy(beam, grid, space, keys, coefficients, **kw):
            flux = orig(beam, grid, space, keys, coefficients, **kw)
            captured.append((beam, space, np.asarray(keys), coefficients, kw, flux))
            return flux

        def mspy(*a, **k):
            calls["march"] += 1
            return om(*a, **k)

        def luspy(*a, **k):
            calls["lu"] += 1
            return olu(*a, **k)

        driver.trace_beam = spy
        raytracer.march_ray, raytracer.lu_factor = mspy, luspy
        try:
            t0 = time.perf_counter()
            driver.trace_all_beams(problem)
            wall = time.perf_counter() - t0
        finally:
            driver.trace_beam = orig
            raytracer.march_ray, raytracer.lu_factor = om, olu
        p = tag + "_"
        out[p + "cpu_s"] = np.array(wall)
        out[p + "marches"] = np.array(calls["march"])
        out[p + "lus"] = np.array(calls["lu"])
        out[p + "n_beams"] = np.array(len(captured))
        for i, (beam, space, keys, coeff, kw, flux) in enumerate(captured):
            q = f"{p}b{i}_"
            if "g" not in out:  # one material (water): one energy operator for every case
                mass, g = raytracer.assemble_energy_operators(space, *coeff[0])
                out["g"] = g
                out["mass"] = space.mass_diagonal()
                out["smin"] = np.array(
                    float(np.atleast_1d(coeff[0][0](np.array([space.e_min])))[0]))
                out["space"] = np.array([space.e_min, space.e_max, space.n_groups,
                                         space.degree])
                out["keys"] = keys.astype(np.int32)
            out.update({
                q + "beam": np.array([*beam.direction, beam.energy_mev, *beam.position_cm,
                                      beam.weight, beam.sigma_xy_cm, beam.sigma_e_mev]),
                q + "rays": np.array([kw["n_side"], kw["span_sigmas"], kw["max_step"]]),
                q + "values_sample": flux.values[sample],
                q + "values_norm": np.array(np.linalg.norm(flux.values)),
                q + "values_colsum": flux.values.sum(axis=0),
                q + "residual": flux.residual_energy,
                q + "n_rays": np.array(flux.n_rays),
            })
        print(f"  trace40 {tag}: reference {wall:.2f} s, {calls['march']} marches, "
              f"{calls['lu']} LUs")
    save("trace40.npz", **out)


def make_water_ops90():
    """The reference's CN energy operator for water on the energy space of a
    90 MeV beam (e_max = 94.5 MeV, 128 groups, P2 DG) and its s*(e_min), for
    the physics it depends on (sigma_t carries the transport correction of the
    P_N order and model): keys g / smin -- P7 Boltzmann (BASELINE configs[0],
    the config-1 beam traced in bench.py); g_fp19 / smin_fp19 -- P19
    Fokker-Planck (tools/config4_traced.py)."""
    got = {}
    for tag, model, pn in (("", "boltzmann", 7), ("_fp19", "fokker-planck", 19)):
        raw = trace40_raw((0.0,))
        raw["grid"] = {"nx": 6, "ny": 6, "nz": 6, "delta_x_cm": 0.1, "delta_y_cm": 0.1,
                       "delta_z_cm": 0.1}
        raw["beams"][0].update({"energy_mev": 90.0, "position_cm": [0.3, 0.3, -1.0],
                                "direction": [0.0, 0.0, 1.0]})
        raw["model"], raw["pn_order"] = model, pn
        config = driver.ProblemConfig.from_dict(raw)
        problem = driver.assemble_problem(config)
        orig = driver.trace_beam

        def spy(beam, grid, space, keys, coefficients, **kw):
            mass, g = raytracer.assemble_energy_operators(space, *coefficients[0])
            got.update({"g" + tag: g, "mass": mass,
                        "space": np.array([space.e_min, space.e_max, space.n_groups,
                                           space.degree]),
                        "smin" + tag: np.array(float(np.atleast_1d(
                            coefficients[0][0](np.array([space.e_min])))[0]))})
            return orig(beam, grid, space, keys, coefficients, **kw)

        driver.trace_beam = spy
        try:
            driver.trace_all_beams(problem)
        finally:
            driver.trace_beam = orig
    save("water_ops90.npz", **got)


def make_bench_physics():
    """Physics tables for the synthetic benchmark phantoms (water / bone / lung
    classes, stopping tables, moment tables up to degree 21 over 1..105 MeV)."""
    from pndose.driver import MomentTables
    from pndose.physics import MaterialField, default_schneider_table, default_stopping_library

    hu = np.array([0.0, 1200.0, -700.0])
    density, weights = default_schneider_table().convert(hu)
    mat = MaterialField(density=density, weights=weights)
    lib = default_stopping_library()
    symbols = list(lib.tables)
    mt = MomentTables(1.0, 105.0, 21, n_points=48, n_nodes=256, exponent=1.0)
    save(
        "bench_physics.npz",
        hu=hu,
        class_density=np.asarray(mat.density),
        class_weights=np.asarray(mat.weights),
        class_atomic=np.asarray(mat.atomic_densities),
        stop_e=np.stack([lib.tables[s].energies for s in symbols]),
        stop_s=np.stack([lib.tables[s].values for s in symbols]),
        mom_e=mt.energies,
        mom_g=mt.g,
        mom_xi1=mt.xi1,
    )


def make_volume():
    """A small volume in the reference's own ASCII VTK writer (driver.py:672-690)
    for the output-reader parity test."""
    from pndose.driver import write_volume
    from pndose.spatial import Grid3D

    grid = Grid3D(4, 3, 5, 0.1, 0.2, 0.3, origin=(1.0, 2.0, 3.0))
    rng = np.random.default_rng(0)
    dep = rng.random(grid.n_cells) * np.exp(rng.uniform(-30, 5, grid.n_cells))
    write_volume(OUT / "volume_ref.vtk", grid, {"deposited_energy": dep, "dose": 2.0 * dep})
    save("volume_ref.npz", deposited_energy=dep, dose=2.0 * dep)


if __name__ == "__main__":
    OUT.mkdir(parents=True, exist_ok=True)
    what = set(sys.argv[1:])
    if not what or "angular" in what:
        make_angular()
    if not what or "kernels" in what:
        make_kernels()
    if not what or "steps" in what:
        make_steps()
    if not what or "traverse" in what:
        make_traverse()
    if not what or "trace" in what:
        make_trace()
    if not what or "march" in what:
        make_march()
    if not what or "bench" in what:
        make_bench_physics()
    if not what or "trace40" in what:
        make_trace40()
    if not what or "ops90" in what:
        make_water_ops90()
    if not what or "volume" in what:
        make_volume()
    e2e = {w[4:] for w in what if w.startswith("e2e:")}
    if not what or "e2e" in what or e2e:
        make_e2e(e2e)
    lock = {w[5:] for w in what if w.startswith("lock:")}
    if not what or "lock" in what or lock:
        make_lock(lock)
