"""Dose-volume writers (paper_2508_04484_b200/output.py).

- the reference's own ASCII file (tests/golden/volume_ref.vtk, written by
  pndose.driver.write_volume in tools/make_golden.py) reads back here to its
  %.12e values; the ASCII writer reproduces it byte for byte;
- the binary writer round-trips bit-exactly (test_driver.py:234-244 is the
  reference's round-trip test, at 1e-6 for ASCII);
- z-slab parallel writes (every rank its own cell range, positional writes)
  give the same bytes as one writer -- in-process and with two gloo ranks.
"""

import os
import socket

import numpy as np
import pytest

from conftest import GOLDEN


def grid():
    from paper_2508_04484_b200.output import VolumeGrid

    return VolumeGrid(4, 3, 5, 0.1, 0.2, 0.3, origin=(1.0, 2.0, 3.0))


def test_reads_reference_ascii_and_rewrites_it(tmp_path):
    from paper_2508_04484_b200.output import read_volume, write_volume

    g = np.load(GOLDEN / "volume_ref.npz")
    grid_r, arrays = read_volume(GOLDEN / "volume_ref.vtk")
    assert grid_r.shape == (4, 3, 5)
    np.testing.assert_allclose(grid_r.origin, (1.0, 2.0, 3.0), rtol=1e-12)
    for name in ("deposited_energy", "dose"):
        np.testing.assert_allclose(arrays[name], g[name], rtol=1e-12, atol=0)
    out = tmp_path / "ascii.vtk"
    write_volume(out, grid(), {"deposited_energy": g["deposited_energy"], "dose": g["dose"]},
                 binary=False)
    assert out.read_bytes() == (GOLDEN / "volume_ref.vtk").read_bytes()


def test_binary_round_trip_is_bit_exact(tmp_path):
    from paper_2508_04484_b200.output import compare_volumes, read_volume, write_volume

    rng = np.random.default_rng(3)
    dep = rng.standard_normal(60) * 1e-17
    path = tmp_path / "vol.vtk"
    write_volume(path, grid(), {"deposited_energy": dep, "dose": 2.0 * dep})
    g2, arrays = read_volume(path)
    assert g2 == grid()
    np.testing.assert_array_equal(arrays["deposited_energy"], dep)
    np.testing.assert_array_equal(arrays["dose"], 2.0 * dep)
    assert compare_volumes(path, path) == {"rel_l2": 0.0, "rel_linf": 0.0}
    # a reference ASCII volume and the binary one of the same values agree to %.12e
    ref = np.load(GOLDEN / "volume_ref.npz")
    write_volume(path, grid(), {"deposited_energy": ref["deposited_energy"]})
    rep = compare_volumes(GOLDEN / "volume_ref.vtk", path)
    assert rep["rel_linf"] < 1e-12


def test_slab_writes_match_one_writer(tmp_path):
    from paper_2508_04484_b200.output import write_volume, write_volume_slab

    rng = np.random.default_rng(5)
    arrays = {"deposited_energy": rng.random(60), "dose": rng.random(60)}
    one = tmp_path / "one.vtk"
    write_volume(one, grid(), arrays)
    par = tmp_path / "par.vtk"
    par.write_bytes(b"x" * 100000)  # stale longer content is cut to length
    nxy = 12
    for rank, (z0, z1) in reversed(list(enumerate([(0, 2), (2, 3), (3, 5)]))):
        local = {k: v[z0 * nxy:z1 * nxy] for k, v in arrays.items()}
        write_volume_slab(par, grid(), list(arrays), local, z0 * nxy, rank)
    assert par.read_bytes() == one.read_bytes()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _slab_worker(rank, world, port, path, ref_path):
    import torch.distributed as dist

    from paper_2508_04484_b200.output import write_volume_slab

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(7)
    full = {"deposited_energy": rng.random(60), "dose": rng.random(60)}
    planes = [(0, 3), (3, 5)][rank]
    lo, hi = planes[0] * 12, planes[1] * 12
    write_volume_slab(path, grid(), list(full), {k: v[lo:hi] for k, v in full.items()}, lo, rank)
    dist.barrier()
    dist.destroy_process_group()


def test_slab_writes_two_gloo_ranks(tmp_path):
    import torch.multiprocessing as mp

    from paper_2508_04484_b200.output import write_volume

    rng = np.random.default_rng(7)
    full = {"deposited_energy": rng.random(60), "dose": rng.random(60)}
    ref = tmp_path / "ref.vtk"
    write_volume(ref, grid(), full)
    path = tmp_path / "two.vtk"
    mp.start_processes(_slab_worker, args=(2, _free_port(), str(path), str(ref)), nprocs=2,
                       join=True, start_method="spawn")
    assert path.read_bytes() == ref.read_bytes()
