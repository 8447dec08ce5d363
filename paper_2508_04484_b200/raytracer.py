"""Uncollided ray traversal on the device (mirror of pndose.raytracer's walk).

`traverse_grid(grid, origin, direction)` keeps the reference signature
(raytracer.py:353-403) and returns the same [(cell, s_enter, s_exit)] list,
bit-exact; `traverse_rays` walks a whole bundle in one thread-per-ray kernel
and returns flat arrays (cells, t0, t1, offsets) for the deposition step.
"""

import numpy as np

from . import _lib
from .dlra import handle_for


def _grid_params(grid):
    shape = (int(grid.nx), int(grid.ny), int(grid.nz))
    spacing = (float(grid.dx), float(grid.dy), float(grid.dz))
    origin = tuple(float(v) for v in getattr(grid, "origin", (0.0, 0.0, 0.0)))
    return shape, spacing, origin


def traverse_rays(shape, spacing, origin, starts, dirs):
    """All rays of a bundle: (cells int64, t0, t1, offsets int64 (n_rays + 1))."""
    starts = _lib.f64(np.atleast_2d(starts))
    dirs = _lib.f64(np.atleast_2d(dirs))
    n_rays = starts.shape[0]
    h = handle_for(shape, spacing, 1)
    org = _lib.f64(origin)
    counts = np.zeros(n_rays, dtype=np.int32)
    h.call("pnd_traverse", _lib.ptr(org), n_rays, _lib.ptr(starts), _lib.ptr(dirs),
           _lib.ptr(counts), None, None, None, None)
    offsets = np.zeros(n_rays + 1, dtype=np.int64)
    np.cumsum(counts, out=offsets[1:])
    total = int(offsets[-1])
    cells = np.empty(total, dtype=np.int64)
    t0 = np.empty(total)
    t1 = np.empty(total)
    if total:
        h.call("pnd_traverse", _lib.ptr(org), n_rays, _lib.ptr(starts), _lib.ptr(dirs),
               _lib.ptr(counts), _lib.ptr(offsets), _lib.ptr(cells), _lib.ptr(t0), _lib.ptr(t1))
    return cells, t0, t1, offsets


def traverse_grid(grid, origin, direction):
    """Amanatides-Woo traversal of one ray (raytracer.py:353-403)."""
    shape, spacing, org = _grid_params(grid)
    cells, t0, t1, _ = traverse_rays(shape, spacing, org, np.asarray(origin, float)[None],
                                     np.asarray(direction, float)[None])
    return [(int(c), float(a), float(b)) for c, a, b in zip(cells, t0, t1)]
