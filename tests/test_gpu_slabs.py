"""Slab decomposition on one GPU: two z-slabs, one host thread each, joined by
the library's "local" transport (device-to-device halo copies, host-summed
Grams; no kernel waits on another rank, so this is safe on a single GPU).
The decomposed solve must reproduce the undecomposed one: same rank history,
dose equal to rounding. NCCL carries the same calls between processes on a
multi-GPU box (comm.cu)."""

import threading
import uuid

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def _run_slabs(bundle, world, max_steps=None):
    from paper_2508_04484_b200 import slabs
    from paper_2508_04484_b200.driver import run_bundle

    cid = ("local:" + uuid.uuid4().hex).encode().ljust(128, b"\0")
    nx, ny, nz = bundle.shape
    results, errors = [None] * world, []

    def work(r):
        try:
            sl = slabs.plan(nx, ny, nz, world, r)
            results[r] = run_bundle(bundle, max_steps=max_steps, slab=sl, comm_id=cid)
        except Exception as exc:  # noqa: BLE001
            errors.append(exc)

    th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    assert not any(t.is_alive() for t in th), "slab ranks did not finish"
    assert not errors, errors
    return results


@pytest.mark.parametrize("tag,world", [("smoke", 2), ("hetero", 2), ("hetero", 3)])
def test_slab_solve_matches_single_device(tag, world):
    from paper_2508_04484_b200.driver import run_bundle
    from paper_2508_04484_b200.problem import ProblemBundle

    b = ProblemBundle.load(GOLDEN / f"bundle_{tag}.npz")
    full = run_bundle(b)
    parts = _run_slabs(b, world)
    dep = np.concatenate([p.dose.deposited for p in parts])
    for p in parts:
        assert [r for _, _, r in p.rank_history] == [r for _, _, r in full.rank_history]
        assert p.diagnostics["max_orthonormality_defect"] < 1e-10
    ref = full.dose.deposited
    assert np.linalg.norm(dep - ref) / np.linalg.norm(ref) < 1e-10


def test_nccl_world_of_one():
    """The NCCL transport's setup on one GPU: dlopen, unique id, a one-rank
    communicator; the solve is unchanged (exchanges are no-ops at world 1)."""
    from paper_2508_04484_b200 import _lib, slabs
    from paper_2508_04484_b200.driver import run_bundle
    from paper_2508_04484_b200.problem import ProblemBundle

    b = ProblemBundle.load(GOLDEN / "bundle_smoke.npz")
    cid = _lib.comm_unique_id()
    assert len(cid) == 128 and any(cid)
    full = run_bundle(b, max_steps=4)
    one = run_bundle(b, max_steps=4, slab=slabs.plan(*b.shape, 1, 0), comm_id=cid)
    np.testing.assert_array_equal(one.dose.deposited, full.dose.deposited)


def test_slab_solve_wide_rank():
    """Ranks above 32 (the 32-column block chains of wide.cu) under the slab
    decomposition: halo planes of every block copy, Gram allreduces of every
    pair, against the undecomposed solve."""
    import dataclasses

    from paper_2508_04484_b200.driver import run_bundle
    from paper_2508_04484_b200.problem import ProblemBundle

    b = ProblemBundle.load(GOLDEN / "bundle_config1.npz")
    b = dataclasses.replace(b, truncation_tolerance=1e300, rank_min=40, rank_max=40)
    full = run_bundle(b, max_steps=25)
    parts = _run_slabs(b, 2, max_steps=25)
    dep = np.concatenate([p.dose.deposited for p in parts])
    for p in parts:
        assert [r for _, _, r in p.rank_history] == [r for _, _, r in full.rank_history]
        assert p.rank_history[-1][2] == 40
    ref = full.dose.deposited
    assert np.linalg.norm(dep - ref) / np.linalg.norm(ref) < 1e-10


def test_slab_solve_blocked_rank_and_footprint_flux():
    """Ranks above 64 (the column-blocked layout of xwide.cu: per-block halo
    planes, rectangular S-Gram pairs, Gram allreduces) and ray-footprint
    uncollided tables restricted to each slab's rows, under a three-slab
    decomposition, against the undecomposed solve."""
    import dataclasses

    from paper_2508_04484_b200.driver import run_bundle
    from paper_2508_04484_b200.problem import ProblemBundle, UncollidedSlices

    b = ProblemBundle.load(GOLDEN / "bundle_fp19.npz")  # 10 x 10 x 12, m = 400
    fl = []
    for f in b.fluxes:
        cells = np.flatnonzero(np.any(f.values != 0.0, axis=1) | (f.residual != 0.0))
        fl.append(UncollidedSlices(f.values[cells], f.residual[cells], f.e_min, f.e_max,
                                   cells.astype(np.int32), b.n_cells))
    b = dataclasses.replace(b, fluxes=fl, truncation_tolerance=1e300, rank_min=70,
                            rank_max=70)
    full = run_bundle(b, max_steps=6)
    parts = _run_slabs(b, 3, max_steps=6)
    dep = np.concatenate([p.dose.deposited for p in parts])
    for p in parts:
        assert [r for _, _, r in p.rank_history] == [r for _, _, r in full.rank_history]
        assert p.rank_history[-1][2] == 70
    ref = full.dose.deposited
    assert np.linalg.norm(dep - ref) / np.linalg.norm(ref) < 1e-10


def test_kstage_plane_split_is_bit_identical():
    """The K stage split into interior planes and the four boundary planes
    (overlapping a slab's halo exchange with the interior, streaming_step)
    computes every chunk exactly as the single launch does."""
    import os

    from paper_2508_04484_b200.driver import run_bundle
    from paper_2508_04484_b200.problem import ProblemBundle

    b = ProblemBundle.load(GOLDEN / "bundle_smoke.npz")
    one = run_bundle(b)
    os.environ["PND_KSTAGE_SPLIT"] = "1"
    try:
        split = run_bundle(b)
    finally:
        os.environ.pop("PND_KSTAGE_SPLIT", None)
    np.testing.assert_array_equal(split.dose.deposited, one.dose.deposited)
    assert [r for _, _, r in split.rank_history] == [r for _, _, r in one.rank_history]
