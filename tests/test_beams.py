"""Beam-batched runs (SURVEY.md §8(e) "Beams"), host logic on CPU.

Subsets of beams are independent low-rank solves whose doses are summed; the
subsets go to groups of ranks (a multi-rank group z-slab shards its subset).
Here the per-subset solve is the numpy oracle (the device solve is
tests/test_gpu_beams.py) and the world is 2 gloo ranks: the summed dose must
equal the oracle's per-subset runs summed in one process, for one subset per
rank and for one subset sharded over both ranks.
"""

import os
import socket
from types import SimpleNamespace

import numpy as np
import pytest

from conftest import GOLDEN
from oracle import dlra_np
from paper_2508_04484_b200 import slabs
from paper_2508_04484_b200.problem import ProblemBundle

STEPS = 6


def test_partition_and_assignment():
    assert slabs.beam_partition(4) == [(0,), (1,), (2,), (3,)]
    assert slabs.beam_partition(5, 2) == [(0, 2, 4), (1, 3)]
    with pytest.raises(ValueError):
        slabs.beam_partition(2, 3)
    # 8 ranks, 4 subsets: groups of 2 consecutive ranks
    a = [slabs.assign_parts(8, r, 4) for r in range(8)]
    assert [x.parts for x in a] == [(0,), (0,), (1,), (1,), (2,), (2,), (3,), (3,)]
    assert a[5].members == (4, 5) and a[5].local_rank == 1
    # 3 ranks, 2 subsets: the third rank idles
    assert slabs.assign_parts(3, 2, 2).parts == ()
    # 2 ranks, 5 subsets: round-robin, each rank alone
    assert slabs.assign_parts(2, 1, 5).parts == (1, 3) and slabs.assign_parts(2, 1, 5).local_world == 1


def _oracle_solve(sub, slab, cid):
    out = dlra_np.run_energy_loop(sub, max_steps=STEPS)
    dep = out["deposited"] + sub.uncollided_dose()
    lo, hi = (0, sub.n_cells) if slab is None else slab.rows
    return SimpleNamespace(dose=SimpleNamespace(deposited=dep[lo:hi]),
                           rank_history=[(k, 0.0, r) for k, r in enumerate(out["rank_history"])])


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, parts, path):
    import torch.distributed as dist

    from paper_2508_04484_b200.driver import run_beam_batched

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        b = ProblemBundle.load(GOLDEN / "bundle_hetero.npz")
        res = run_beam_batched(b, parts=parts, dist=dist, solve=_oracle_solve)
        if rank == 0:
            np.save(path, res.dose.deposited)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("parts", [[(0,), (1,)], [(0, 1)]])
def test_two_rank_beam_batched_dose(tmp_path, parts):
    import torch.multiprocessing as mp

    path = str(tmp_path / "dose.npy")
    mp.spawn(_worker, args=(2, _free_port(), parts, path), nprocs=2, join=True)
    got = np.load(path)
    b = ProblemBundle.load(GOLDEN / "bundle_hetero.npz")
    want = sum(_oracle_solve(b.subset_beams(p), None, None).dose.deposited for p in parts)
    np.testing.assert_allclose(got, want, rtol=1e-13, atol=1e-300)
