"""N > 1 host logic on CPU: z-slab plan, halo exchange and Gram allreduce over
torch.distributed "gloo" with world_size 2 (the GPU box path uses "nccl").

Each rank owns a contiguous block of z-planes, receives 2 halo planes from
each neighbour, applies the oracle's stencils on the halo-extended slab and
allreduces its partial Grams; the assembled results must equal the
single-process oracle on the whole grid (bit-for-bit up to summation order).
"""

import os
import socket

import numpy as np
import pytest

from oracle import dlra_np
from paper_2508_04484_b200 import slabs


def test_plan_covers_grid_contiguously():
    for nz, world in [(8, 2), (9, 2), (12, 4), (17, 8), (256, 8)]:
        sl = [slabs.plan(5, 4, nz, world, r) for r in range(world)]
        assert sl[0].z0 == 0 and sl[-1].z1 == nz
        for a, b in zip(sl, sl[1:]):
            assert a.z1 == b.z0
        assert all(s.planes >= 2 for s in sl)
        assert max(s.planes for s in sl) - min(s.planes for s in sl) <= 1
        assert sl[0].halo_below == 0 and sl[-1].halo_above == 0
    with pytest.raises(ValueError):
        slabs.plan(4, 4, 3, 2, 0)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nx, ny, nz, r = case
        rng = np.random.default_rng(5)
        grid = dlra_np.Grid(nx, ny, nz, 0.2, 0.3, 0.25)
        n = grid.n
        inv_s = 1.0 / rng.uniform(5.0, 10.0, n)
        k = rng.standard_normal((n, r))
        u0 = np.linalg.qr(rng.standard_normal((n, r)))[0]
        v0 = np.linalg.qr(rng.standard_normal((9, r)))[0]
        ops = dlra_np.Ops([np.linalg.qr(rng.standard_normal((9, 9)))[0] for _ in range(3)],
                          [rng.uniform(0, 1, 9) for _ in range(3)],
                          [-rng.uniform(0, 1, 9) for _ in range(3)])
        kf = [ops.factor(v0, a, s) for a, s in grid.stencils()]

        sl = slabs.plan(nx, ny, nz, world, rank)
        lo, hi = sl.rows
        pgrid = dlra_np.Grid(*slabs.padded_grid_shape(sl), 0.2, 0.3, 0.25)
        # K-stage right-hand side on the halo-extended slab
        kp = slabs.exchange_halo(sl, k[lo:hi])
        sp = slabs.exchange_halo(sl, inv_s[lo:hi, None])[:, 0]
        got = slabs.crop(sl, dlra_np.k_rhs(kp, sp, pgrid, kf))
        want = dlra_np.k_rhs(k, inv_s, grid, kf)[lo:hi]
        assert np.abs(got - want).max() <= 1e-13 * np.abs(want).max()
        # stencil Grams: local partial sums + allreduce
        up = slabs.exchange_halo(sl, u0[lo:hi])
        part = []
        for a, s in pgrid.stencils():
            d = slabs.crop(sl, dlra_np.stencil(pgrid, a, s, sp[:, None] * up))
            part.append(u0[lo:hi].T @ d)
        g = slabs.allreduce_sum(np.array(part))
        want_g = np.array(dlra_np.stencil_grams(u0, u0, inv_s, grid))
        assert np.abs(g - want_g).max() <= 1e-13 * np.abs(want_g).max()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("case", [(5, 4, 8, 3), (4, 6, 9, 2), (3, 1, 7, 4)])
def test_two_rank_halo_stencil_and_gram_allreduce(case):
    import torch.multiprocessing as mp

    mp.spawn(_worker, args=(2, _free_port(), case), nprocs=2, join=True)
