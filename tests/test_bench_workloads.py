"""Host side of the bench workloads (bench.py, tools/config_sweep.py): the
synthetic phantoms reproduce SURVEY.md §8(d)'s configurations -- the energy
step counts the reference's CFL rule gives for them (driver.py:503-520) and
config 3's slab layout."""

import numpy as np


def test_config2_water_step_count():
    import bench

    b, _, _ = bench.make_workload(nside=256)
    assert b.n_moments == 400 and b.model == "fokker-planck"
    assert len(b.pseudo_time_edges()) - 1 == 1515


def test_config3_slab_phantom():
    import bench

    zc = bench.plane_classes(512, 0.025, "slabs")
    # water [0, 3) cm, bone [3, 4), lung [4, 7), water beyond, h = 0.025 cm
    assert np.bincount(zc).tolist() == [352, 40, 120]
    assert (zc[:120] == 0).all() and (zc[120:160] == 1).all() and (zc[160:280] == 2).all()
    assert (zc[280:] == 0).all()
    b, _, beam = bench.make_workload(nside=512, n_max=7, model="boltzmann", energy=100.0,
                                     phantom="slabs")
    assert b.n_moments == 64 and b.n_classes == 3
    # the CFL uses min S over all classes: low-density lung shrinks dE ~3x
    assert len(b.pseudo_time_edges()) - 1 == 9171
    _, depth = bench.separable_flux(b, beam)
    assert depth.shape == (512, 128) and np.isfinite(depth).all()


def test_config4_step_count():
    import bench

    b, _, _ = bench.make_workload(nside=256, energy=90.0)
    assert len(b.pseudo_time_edges()) - 1 == 2367
