"""Z-slab decomposition of the n-side for one process per GPU.

The flat cell index k*nx*ny + j*nx + i has z slowest (spatial.py:62-63), so a
rank that owns planes [z0, z1) owns one contiguous row block of every n-side
matrix. Everything in the energy step is row-local except
  - the upwind stencils, which reach 2 planes along z: before each stencil
    phase (the 4 K-stages, the L-Grams on U0, the S-Grams on U^) a rank needs
    2 halo planes from each neighbour -- exactly the 2 nx*ny zero rows the
    cell-major device layout already keeps around every matrix;
  - the reductions over cells (stencil Grams, the augmentation Grams, B_i,
    source projections, the orthonormality defect), which become an allreduce
    of small r x r / R x R blocks.
All m-side and R x R work is replicated from the allreduced inputs, so ranks
stay bit-identical without broadcasts.

This module is the host-side plan and exchange logic (torch.distributed:
"nccl" on the GPU box, "gloo" in the CPU tests). The per-slab arithmetic it
is tested with is the numpy oracle; the device path consumes the same plan.
"""

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Slab:
    rank: int
    world: int
    nx: int
    ny: int
    nz: int
    z0: int
    z1: int

    @property
    def nxy(self):
        return self.nx * self.ny

    @property
    def planes(self):
        return self.z1 - self.z0

    @property
    def rows(self):
        """Row range [lo, hi) of this slab in the global cell index."""
        return self.z0 * self.nxy, self.z1 * self.nxy

    @property
    def halo_below(self):
        """Planes received from rank - 1 (0 at the global bottom face)."""
        return min(2, self.z0)

    @property
    def halo_above(self):
        return min(2, self.nz - self.z1)


def plan(nx, ny, nz, world, rank):
    """Balanced contiguous z-slabs; every rank gets >= 2 planes when nz allows
    (a halo of 2 planes must come from one neighbour)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    if nz < 2 * world and world > 1:
        raise ValueError(f"nz={nz} too small for {world} slabs of >= 2 planes")
    base, extra = divmod(nz, world)
    z0 = rank * base + min(rank, extra)
    z1 = z0 + base + (1 if rank < extra else 0)
    return Slab(rank, world, nx, ny, nz, z0, z1)


def exchange_halo(slab, local, dist=None, group=None):
    """Local rows (planes * nxy, c) -> rows with the neighbours' boundary
    planes attached: (halo_below + planes + halo_above) * nxy rows.

    Uses point-to-point send/recv of the 2 edge planes in each direction
    (one message per neighbour and direction)."""
    import torch

    if dist is None:
        import torch.distributed as dist
    nxy = slab.nxy
    local = np.ascontiguousarray(local)
    c = local.shape[1]
    t_local = torch.from_numpy(local)
    ops = []
    below = above = None
    if slab.halo_below:
        hb = slab.halo_below
        below = torch.empty((hb * nxy, c), dtype=t_local.dtype)
        ops.append(dist.P2POp(dist.isend, t_local[: hb * nxy].contiguous(), slab.rank - 1,
                              group))
        ops.append(dist.P2POp(dist.irecv, below, slab.rank - 1, group))
    if slab.halo_above:
        ha = slab.halo_above
        above = torch.empty((ha * nxy, c), dtype=t_local.dtype)
        ops.append(dist.P2POp(dist.isend, t_local[-ha * nxy:].contiguous(), slab.rank + 1,
                              group))
        ops.append(dist.P2POp(dist.irecv, above, slab.rank + 1, group))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    parts = [p.numpy() for p in (below,) if p is not None] + [local] + \
        [p.numpy() for p in (above,) if p is not None]
    return np.concatenate(parts, axis=0)


def allreduce_sum(arr, dist=None, group=None):
    """FP64 sum over ranks of a small block (Grams, projections)."""
    import torch

    if dist is None:
        import torch.distributed as dist
    t = torch.from_numpy(np.ascontiguousarray(arr, dtype=np.float64)).clone()
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t.numpy()


def crop(slab, padded):
    """Drop the halo planes again: rows of the owned planes only."""
    nxy = slab.nxy
    lo = slab.halo_below * nxy
    return padded[lo: lo + slab.planes * nxy]


def padded_grid_shape(slab):
    """(nx, ny, nz') of the halo-extended slab; its z-faces coincide with the
    global faces exactly where no neighbour exists, so the reference's
    boundary closure (spatial.py:81-118) applies there and only there."""
    return slab.nx, slab.ny, slab.halo_below + slab.planes + slab.halo_above


# ---------------------------------------------------------------- beam batching
# SURVEY.md §8(e) "Beams": rays and beams are independent, so a multi-beam run
# may be split into independent low-rank solves per beam subset whose doses
# are summed (not numerically the joint solve: its reference is the CPU run
# on the same partition). Subsets go to groups of ranks; a group of several
# ranks z-slab shards its subset's solve over its own communicator.


def beam_partition(n_beams, parts=None):
    """Beams dealt round-robin into `parts` subsets (default: one per beam)."""
    parts = n_beams if parts is None else int(parts)
    if not 1 <= parts <= max(n_beams, 1):
        raise ValueError(f"cannot split {n_beams} beams into {parts} subsets")
    return [tuple(range(p, n_beams, parts)) for p in range(parts)]


@dataclass(frozen=True)
class BeamAssignment:
    """This rank's share of a beam-batched run."""

    parts: tuple          # indices of the beam subsets this rank works on (in order)
    members: tuple        # world ranks of this rank's group (one group per subset when
                          # world >= subsets, else every rank alone)
    local_rank: int       # position in members (its z-slab when len(members) > 1)

    @property
    def local_world(self):
        return len(self.members)


def assign_parts(world, rank, n_parts):
    """world >= n_parts: subset p -> ranks [p g, (p + 1) g), g = world // n_parts
    (a rank past n_parts g idles); world < n_parts: each rank alone, subsets
    dealt round-robin (rank q solves q, q + world, ... one after another)."""
    if world < 1 or not 0 <= rank < world or n_parts < 1:
        raise ValueError("bad rank/world/parts")
    if world >= n_parts:
        g = world // n_parts
        p = rank // g
        if p >= n_parts:
            return BeamAssignment((), (rank,), 0)
        return BeamAssignment((p,), tuple(range(p * g, (p + 1) * g)), rank - p * g)
    return BeamAssignment(tuple(range(rank, n_parts, world)), (rank,), 0)


def sum_doses(local_dose, dist=None):
    """Sum the per-rank dose contributions (each rank holds zeros outside the
    rows it solved) over the world: the beam-batched total dose."""
    return allreduce_sum(local_dose, dist=dist)
