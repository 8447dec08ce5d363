"""GPU parity of the uncollided tracer (march + deposit) against the reference.

- march_ray (raytracer.py:285-350) on the reference's own march fixture:
  group averages per segment, below-cutoff residual and exit spectrum;
- trace_beam (raytracer.py:452-529) for an axial and an oblique beam through
  the heterogeneous phantom: the (cell x group) flux, the residual energy per
  cell and the live-ray count, from the reference's assembled operators.
The device factors each (material, dz) CN system by block elimination
instead of a dense LU, so agreement is to FP64 rounding (T1-class), not bits.
"""

from types import SimpleNamespace

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu


def relmax(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(b).max(), 1e-300))


def test_march_matches_reference():
    from paper_2508_04484_b200 import raytracer as rt

    M = golden("march.npz")
    space = rt.EnergySpace(1.0, 31.5, 32, 2)
    plan = rt._Marches(rt.MAX_STEP_CM)
    plan.add([(float(l), int(k)) for l, k in zip(M["seg_len"], M["seg_key"])])
    psi0 = rt.project_initial_spectrum(space, 30.0, 0.3)
    assert relmax(psi0, M["psi0"]) < 1e-14
    av, res, psi = plan.run(space, {0: M["g_0"], 1: M["g_1"]},
                            {0: float(M["s_min"][0]), 1: float(M["s_min"][1])}, psi0,
                            want_exit=True)
    assert relmax(av, M["averages"]) < 1e-11
    assert relmax(res, M["residual"]) < 1e-11
    assert relmax(psi[0], M["psi_exit"]) < 1e-11


@pytest.mark.parametrize("beam_index", [0, 1])
def test_trace_beam_matches_reference(beam_index):
    from paper_2508_04484_b200 import raytracer as rt

    T = golden("trace.npz")
    p = f"b{beam_index}_"
    sp = T[p + "space"]
    space = rt.EnergySpace(float(sp[0]), float(sp[1]), int(sp[2]), int(sp[3]))
    gr = T[p + "grid"]
    grid = SimpleNamespace(nx=int(gr[0]), ny=int(gr[1]), nz=int(gr[2]), dx=gr[3], dy=gr[4],
                           dz=gr[5], origin=tuple(gr[6:9]))
    b = T[p + "beam"]
    beam = SimpleNamespace(direction=tuple(b[:3]), energy_mev=b[3], position_cm=tuple(b[4:7]),
                           weight=b[7], sigma_xy_cm=b[8], sigma_e_mev=b[9])
    keys = [int(k) for k in T[p + "key_list"]]
    gm = {k: T[p + f"g_{k}"] for k in keys}
    smin = {k: float(T[p + f"smin_{k}"]) for k in keys}
    rays = T[p + "rays"]
    flux = rt.trace_beam_ops(beam, grid, space, T[p + "keys"], gm, smin, int(rays[0]),
                             float(rays[1]), float(rays[2]))
    assert flux.n_rays == int(T[p + "n_rays"])
    assert relmax(flux.values, T[p + "values"]) < 1e-10
    assert relmax(flux.residual_energy, T[p + "residual"]) < 1e-10
    # same cells touched
    np.testing.assert_array_equal(flux.values != 0.0, T[p + "values"] != 0.0)


@pytest.mark.parametrize("tag", ["deg0", "deg30", "beams4"])
def test_trace40_matches_reference(tag):
    """BASELINE.md's tracer timing cases (40^3 water, 121 rays/beam, 0 deg,
    30 deg, four beams 0/30/60/90 deg): the device tracer's flux against the
    reference's at 4,000 sampled cells, its group sums and residual energy."""
    import sys

    from conftest import ROOT

    sys.path.insert(0, str(ROOT / "tools"))
    import trace_bench

    from paper_2508_04484_b200 import raytracer as rt

    T = trace_bench.load()
    fluxes = trace_bench.trace_case(T, tag, rt)
    assert trace_bench.check(T, tag, fluxes) < 1e-10


def test_trace_footprint_table_matches_dense():
    """trace_beam_ops(sparse=True) keeps the table on the rays' footprint: its
    rows equal the dense table's there (same per-cell deposit order, bit for
    bit) and the dense table is zero elsewhere; a device run from the sparse
    tables gives the dense run's dose bit for bit."""
    import dataclasses

    from conftest import GOLDEN
    from paper_2508_04484_b200 import raytracer as rt
    from paper_2508_04484_b200.driver import run_bundle
    from paper_2508_04484_b200.problem import ProblemBundle, UncollidedSlices

    T = golden("trace.npz")
    p = "b1_"
    sp = T[p + "space"]
    space = rt.EnergySpace(float(sp[0]), float(sp[1]), int(sp[2]), int(sp[3]))
    gr = T[p + "grid"]
    grid = SimpleNamespace(nx=int(gr[0]), ny=int(gr[1]), nz=int(gr[2]), dx=gr[3], dy=gr[4],
                           dz=gr[5], origin=tuple(gr[6:9]))
    b = T[p + "beam"]
    beam = SimpleNamespace(direction=tuple(b[:3]), energy_mev=b[3], position_cm=tuple(b[4:7]),
                           weight=b[7], sigma_xy_cm=b[8], sigma_e_mev=b[9])
    keys = [int(k) for k in T[p + "key_list"]]
    gm = {k: T[p + f"g_{k}"] for k in keys}
    smin = {k: float(T[p + f"smin_{k}"]) for k in keys}
    rays = T[p + "rays"]
    args = (beam, grid, space, T[p + "keys"], gm, smin, int(rays[0]), float(rays[1]),
            float(rays[2]))
    dense = rt.trace_beam_ops(*args, sparse=False)
    sparse = rt.trace_beam_ops(*args, sparse=True)
    assert sparse.cells is not None and len(sparse.cells) < dense.values.shape[0]
    np.testing.assert_array_equal(sparse.values, dense.values[sparse.cells])
    np.testing.assert_array_equal(sparse.residual_energy, dense.residual_energy[sparse.cells])
    mask = np.ones(dense.values.shape[0], bool)
    mask[sparse.cells] = False
    assert not dense.values[mask].any()
    # device runs from dense vs footprint tables
    bb = ProblemBundle.load(GOLDEN / "bundle_hetero.npz")
    fl = []
    for f in bb.fluxes:
        cells = np.flatnonzero(np.any(f.values != 0.0, axis=1) | (f.residual != 0.0))
        fl.append(UncollidedSlices(f.values[cells], f.residual[cells], f.e_min, f.e_max,
                                   cells.astype(np.int32), bb.n_cells))
    r_dense = run_bundle(bb, max_steps=25)
    r_sparse = run_bundle(dataclasses.replace(bb, fluxes=fl), max_steps=25)
    assert r_sparse.dose.deposited.tobytes() == r_dense.dose.deposited.tobytes()


def test_config1_beam_traced_matches_reference_table():
    """BASELINE configs[0]'s beam (90 MeV +z, 441 rays, 1 x 20 x 70 at 2 cm x
    1 mm) traced on the device with the reference's water operator for that
    energy space (water_ops90.npz) reproduces the reference-traced table the
    config-1 bundle carries (trace_all_beams output, bundle_config1.npz)."""
    from conftest import GOLDEN
    from paper_2508_04484_b200 import raytracer as rt
    from paper_2508_04484_b200.problem import ProblemBundle

    b = ProblemBundle.load(GOLDEN / "bundle_config1.npz")
    W = golden("water_ops90.npz")
    sp = W["space"]
    space = rt.EnergySpace(float(sp[0]), float(sp[1]), int(sp[2]), int(sp[3]))
    nx, ny, nz = b.shape
    grid = SimpleNamespace(nx=nx, ny=ny, nz=nz, dx=b.spacing[0], dy=b.spacing[1],
                           dz=b.spacing[2], origin=tuple(b.origin))
    beam = SimpleNamespace(direction=(0.0, 0.0, 1.0), energy_mev=90.0,
                           position_cm=(1.0, 1.0, 0.0), weight=1.0, sigma_xy_cm=0.3,
                           sigma_e_mev=0.9)
    flux = rt.trace_beam_ops(beam, grid, space, np.zeros(b.n_cells, dtype=np.int32),
                             {0: W["g"]}, {0: float(W["smin"])}, 21, 3.0, 0.01)
    assert relmax(flux.values, b.fluxes[0].values) < 1e-10
    assert relmax(flux.residual_energy, b.fluxes[0].residual) < 1e-10
