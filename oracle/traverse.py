"""CPU oracle for the uncollided ray traversal -- TEST INFRASTRUCTURE ONLY.

Pure-Python restatement of the Amanatides-Woo walk in
/root/reference/pkg/src/pndose/raytracer.py:353-403, written so every
float64 operation happens in the same order as the reference (no fused
multiply-add is possible in Python), which makes its output the bit-exact
target for the CUDA traversal kernel. Pinned against the reference's own
paths in tests/golden/traverse.npz.

Python's builtin max/min keep the FIRST argument on ties; the order of the
arguments below matches the reference so signed zeros come out identical.
"""

import math


def traverse(shape, spacing, origin, p0, d):
    """[(cell, t_enter, t_exit)] of one ray (raytracer.py:353-403)."""
    nx, ny, nz = shape
    bounds = [(origin[a], origin[a] + shape[a] * spacing[a]) for a in range(3)]
    t_lo, t_hi = 0.0, math.inf
    for a in range(3):
        lo, hi = bounds[a]
        if abs(d[a]) < 1e-14:
            if not (lo <= p0[a] <= hi):
                return []
            continue
        t1 = (lo - p0[a]) / d[a]
        t2 = (hi - p0[a]) / d[a]
        t_lo = max(t_lo, min(t1, t2))
        t_hi = min(t_hi, max(t1, t2))
    if t_hi <= t_lo:
        return []
    eps = 1e-10 * max(spacing)
    te = t_lo + eps
    p = [p0[a] + te * d[a] for a in range(3)]
    idx = [min(shape[a] - 1, max(0, int((p[a] - bounds[a][0]) / spacing[a]))) for a in range(3)]
    step = [0, 0, 0]
    t_max = [math.inf] * 3
    t_delta = [math.inf] * 3
    for a in range(3):
        if d[a] > 1e-14:
            step[a] = 1
            t_max[a] = (bounds[a][0] + (idx[a] + 1) * spacing[a] - p0[a]) / d[a]
            t_delta[a] = spacing[a] / d[a]
        elif d[a] < -1e-14:
            step[a] = -1
            t_max[a] = (bounds[a][0] + idx[a] * spacing[a] - p0[a]) / d[a]
            t_delta[a] = -spacing[a] / d[a]
    out = []
    t = t_lo
    while t < t_hi - 1e-14:
        axis = 0
        if t_max[1] < t_max[axis]:
            axis = 1
        if t_max[2] < t_max[axis]:
            axis = 2
        t_next = min(t_max[axis], t_hi)
        if t_next > t:
            out.append((idx[2] * nx * ny + idx[1] * nx + idx[0], t, t_next))
        t = t_next
        idx[axis] += step[axis]
        if not (0 <= idx[axis] < shape[axis]):
            break
        t_max[axis] += t_delta[axis]
    return out
