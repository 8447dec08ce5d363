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


# ======================================================================
# Uncollided flux: energy march along rays + track-length deposit
# (raytracer.py:157-529 of the reference, on the device through
# pnd_march / pnd_deposit; the host keeps the small per-beam setup:
# ray bundle, initial spectrum, energy operators per material, the
# signature de-duplication and the (material, dz) stepper table).
# ======================================================================
import math
from dataclasses import dataclass

from .errors import ConfigError

MAX_STEP_CM = 0.01                 # CN step bound (raytracer.py:35)
SIPG_ETA = 10.0 * (2 + 1) ** 2     # straggling penalty 10 (p+1)^2, p = 2 (raytracer.py:36)
_QUAD_NODES = 6                    # Gauss-Legendre nodes per group (raytracer.py:37)


@dataclass(frozen=True)
class EnergySpace:
    """Equal-width energy groups x modal Legendre basis (EnergyDGSpace,
    raytracer.py:72-155): only what the march needs."""

    e_min: float
    e_max: float
    n_groups: int = 128
    degree: int = 2

    @classmethod
    def of(cls, space):
        return cls(float(space.e_min), float(space.e_max), int(space.n_groups),
                   int(space.degree))

    @property
    def n_local(self):
        return self.degree + 1

    @property
    def n_dof(self):
        return self.n_groups * self.n_local

    @property
    def width(self):
        return (self.e_max - self.e_min) / self.n_groups

    @property
    def edges(self):
        return np.linspace(self.e_min, self.e_max, self.n_groups + 1)

    @property
    def centers(self):
        e = self.edges
        return 0.5 * (e[:-1] + e[1:])

    def mass_diagonal(self):
        local = self.width / 2.0 * 2.0 / (2.0 * np.arange(self.n_local) + 1.0)
        return np.tile(local, self.n_groups)

    def basis(self):
        """(GL nodes x, weights w, P (q x nl), dP/dxi (q x nl), P(+1), P(-1), P'(+1), P'(-1))."""
        leg = np.polynomial.legendre
        x, w = leg.leggauss(_QUAD_NODES)
        eye = np.eye(self.n_local)
        p = leg.legvander(x, self.degree)
        dp = np.stack([leg.legval(x, leg.legder(eye[j])) for j in range(self.n_local)], axis=1)
        at = lambda xi: leg.legvander([xi], self.degree)[0]  # noqa: E731
        dat = lambda xi: np.array([leg.legval(xi, leg.legder(eye[j]))  # noqa: E731
                                   for j in range(self.n_local)])
        return x, w, p, dp, at(1.0), at(-1.0), dat(1.0), dat(-1.0)


def assemble_energy_operators(space, s_star_fn, t_fn=None, sigma_t_fn=None):
    """(mass diagonal, G) of M psi' + G psi = 0 along depth
    (raytracer.py:169-274): DG advection toward lower energy with a
    Lax-Friedrichs flux (wave speed S*), outflow at e_min, vacuum inflow at
    e_max; optional SIPG straggling (kappa = T/2) and absorption. G is
    block tridiagonal over groups; assembled group by group."""
    sp = EnergySpace.of(space)
    nl, ng, h = sp.n_local, sp.n_groups, sp.width
    x, w, p, dp, p_hi, p_lo, dp_hi, dp_lo = sp.basis()
    jac = 0.5 * h
    e_q = sp.centers[:, None] + jac * x[None, :]            # (G, q)
    G = np.zeros((sp.n_dof, sp.n_dof))

    def blk(a, b):
        return (slice(a * nl, (a + 1) * nl), slice(b * nl, (b + 1) * nl))

    s_q = np.asarray(s_star_fn(e_q), dtype=float)
    s_e = np.asarray(s_star_fn(sp.edges), dtype=float)
    sig_q = None if sigma_t_fn is None else np.asarray(sigma_t_fn(e_q), dtype=float)
    kap_q = None if t_fn is None else 0.5 * np.asarray(t_fn(e_q), dtype=float)
    kap_e = None if t_fn is None else 0.5 * np.asarray(t_fn(sp.edges), dtype=float)
    for g in range(ng):
        # volume: + int dphi_i/dE S* phi_j  (dphi/dE = P' 2/h)
        G[blk(g, g)] += (dp.T * (w * s_q[g])) @ p * jac * (2.0 / h)
        if sig_q is not None:
            G[blk(g, g)] += (p.T * (w * sig_q[g])) @ p * jac
        if kap_q is not None:
            G[blk(g, g)] += (dp.T * (w * kap_q[g])) @ dp * jac * (2.0 / h) ** 2
    for g in range(ng - 1):
        # face between group g (trace at xi=+1) and g+1 (trace at xi=-1):
        # qhat = c_lo psi_lo + c_hi psi_hi with c_lo = 0, c_hi = -S*(edge)
        sf = s_e[g + 1]
        c_lo, c_hi = -0.5 * sf + 0.5 * sf, -0.5 * sf - 0.5 * sf
        G[blk(g, g)] += np.outer(p_hi, c_lo * p_hi)
        G[blk(g, g + 1)] += np.outer(p_hi, c_hi * p_lo)
        G[blk(g + 1, g)] -= np.outer(p_lo, c_lo * p_hi)
        G[blk(g + 1, g + 1)] -= np.outer(p_lo, c_hi * p_lo)
        if kap_e is not None:
            kf = kap_e[g + 1]
            pen = SIPG_ETA * kf / h
            val = (p_hi, p_lo)
            der = ((2.0 / h) * dp_hi, (2.0 / h) * dp_lo)
            sgn = (1.0, -1.0)
            for a in range(2):
                for b in range(2):
                    ja, jb = sgn[a] * val[a], sgn[b] * val[b]
                    G[blk(g + a, g + b)] += (-np.outer(ja, 0.5 * kf * der[b])
                                             - np.outer(0.5 * kf * der[a], jb)
                                             + pen * np.outer(ja, jb))
    # bottom face (e_min): outflow, upwind interior trace
    G[blk(0, 0)] -= np.outer(p_lo, -s_e[0] * p_lo)
    return sp.mass_diagonal(), G


def project_initial_spectrum(space, mean_mev, sigma_mev):
    """L2 projection of the Gaussian beam spectrum (raytracer.py:157-166)."""
    sp = EnergySpace.of(space)
    x, w, p, _, _, _, _, _ = sp.basis()
    jac = 0.5 * sp.width
    e = sp.centers[:, None] + jac * x[None, :]
    f = np.exp(-0.5 * ((e - mean_mev) / sigma_mev) ** 2) / (sigma_mev * math.sqrt(2.0 * math.pi))
    rhs = jac * (f * w) @ p                                  # (G, nl)
    m_loc = jac * 2.0 / (2.0 * np.arange(sp.n_local) + 1.0)
    return (rhs / m_loc).ravel()


def stratified_ray_offsets(sigma, n_side=21, span_sigmas=3.0):
    """Midpoint-stratified lateral offsets and normalised Gaussian weights
    (raytracer.py:406-418)."""
    half = span_sigmas * sigma
    step = 2.0 * half / n_side
    c = -half + (np.arange(n_side) + 0.5) * step
    a, b = np.meshgrid(c, c, indexing="ij")
    off = np.column_stack([a.ravel(), b.ravel()])
    wt = np.exp(-0.5 * (off ** 2).sum(axis=1) / sigma ** 2)
    return off, wt / wt.sum()


def transverse_frame(direction):
    """Two unit vectors orthogonal to the beam (BeamSource.transverse_frame,
    raytracer.py:60-69)."""
    d = np.asarray(direction, dtype=float)
    helper = np.array([0.0, 1.0, 0.0]) if abs(d[0]) > 0.9 else np.array([1.0, 0.0, 0.0])
    e1 = np.cross(d, helper)
    e1 /= np.linalg.norm(e1)
    return e1, np.cross(d, e1)


class _Marches:
    """Host plan of a batch of marches: segments, halves, (key, dz) steppers."""

    def __init__(self, max_step):
        self.max_step = float(max_step)
        self.seg_off = [0]
        self.seg_key, self.half_dz, self.half_n, self.half_st = [], [], [], []
        self.st_index, self.st_key, self.st_dz = {}, [], []

    def add(self, segments):
        """segments: [(length, key)] of one march; returns its index."""
        for length, key in segments:
            self.seg_key.append(int(key))
            for _ in range(2):                               # two halves (raytracer.py:316)
                half = 0.5 * length
                if half <= 0.0:
                    self.half_dz.append(0.0)
                    self.half_n.append(0)
                    self.half_st.append(0)
                    continue
                n_sub = max(1, math.ceil(half / self.max_step))
                dz = half / n_sub
                ck = (int(key), round(dz, 14))               # the reference's LU cache key
                if ck not in self.st_index:
                    self.st_index[ck] = len(self.st_key)
                    self.st_key.append(int(key))
                    self.st_dz.append(dz)
                self.half_dz.append(dz)
                self.half_n.append(n_sub)
                self.half_st.append(self.st_index[ck])
        self.seg_off.append(len(self.seg_key))
        return len(self.seg_off) - 2

    def run(self, space, gmats, s_min, psi0, want_exit=False):
        sp = EnergySpace.of(space)
        keys = sorted(gmats)
        pos = {k: i for i, k in enumerate(keys)}
        g_all = _lib.f64(np.stack([np.asarray(gmats[k], dtype=float) for k in keys]))
        smin = _lib.f64([float(s_min[k]) for k in keys])
        n_m = len(self.seg_off) - 1
        nseg = len(self.seg_key)
        ng, nl = sp.n_groups, sp.n_local
        av = np.zeros((nseg, ng))
        res = np.zeros(nseg)
        psi = np.zeros((n_m, sp.n_dof)) if want_exit else None
        if n_m == 0:
            return av, res, psi
        h = handle_for((1, 1, 1), (1.0, 1.0, 1.0), 1)
        p_lo = _lib.f64(np.polynomial.legendre.legvander([-1.0], sp.degree)[0])
        st_key = _lib.i32([pos[k] for k in self.st_key])
        h.call("pnd_march", nl, ng, len(keys), _lib.ptr(g_all), _lib.ptr(_lib.f64(sp.mass_diagonal())),
               _lib.ptr(p_lo), float(sp.e_min), _lib.ptr(smin), _lib.ptr(_lib.f64(psi0)),
               len(self.st_key), _lib.ptr(st_key), _lib.ptr(_lib.f64(self.st_dz)), n_m,
               _lib.ptr(_lib.i32(self.seg_off)), _lib.ptr(_lib.i32([pos[k] for k in self.seg_key])),
               _lib.ptr(_lib.f64(self.half_dz)), _lib.ptr(_lib.i32(self.half_n)),
               _lib.ptr(_lib.i32(self.half_st)), _lib.ptr(av), _lib.ptr(res),
               _lib.ptr(psi) if psi is not None else None)
        return av, res, psi


@dataclass
class RaySegmentRecord:
    """march_ray record (raytracer.py:276-282)."""

    cell: int
    length: float
    group_averages: np.ndarray
    residual_energy: float


def march_ray(space, segments, coefficients, psi0, max_step=MAX_STEP_CM):
    """Drop-in for raytracer.march_ray (raytracer.py:285-350): the
    Crank-Nicolson march of one ray on the device. segments: [(cell, length,
    material_key)]; coefficients: key -> (s_star_fn, t_fn, sigma_t_fn)."""
    keys = sorted({int(k) for _, _, k in segments})
    gm, smin = {}, {}
    for k in keys:
        gm[k] = assemble_energy_operators(space, *coefficients[k])[1]
        smin[k] = float(np.atleast_1d(coefficients[k][0](np.array([space.e_min])))[0])
    plan = _Marches(max_step)
    plan.add([(float(length), int(k)) for _, length, k in segments])
    av, res, psi = plan.run(space, gm, smin, psi0, want_exit=True)
    recs = [RaySegmentRecord(int(c), float(length), av[i], float(res[i]))
            for i, (c, length, _) in enumerate(segments)]
    return recs, psi[0]


@dataclass
class UncollidedFlux:
    """Ray-traced uncollided flux (raytracer.py:421-448): values (n_cells x
    n_groups), residual energy per cell, live rays."""

    beam: object
    space: object
    values: np.ndarray
    residual_energy: np.ndarray
    n_rays: int
    # ray-footprint form: the cells the rays touched (strictly increasing);
    # values / residual_energy then hold only those rows (zero elsewhere)
    cells: np.ndarray = None
    n_cells: int = 0

    @property
    def group_energies(self):
        return EnergySpace.of(self.space).centers

    @property
    def undershoot(self) -> float:
        """Most negative flux value (raytracer.py:432-435; 0 if none)."""
        return float(min(self.values.min(initial=0.0), 0.0))

    def at_energy(self, e_mev) -> np.ndarray:
        """Group-centre interpolation, zero outside (raytracer.py:437-449)."""
        if self.cells is not None:
            out = np.zeros(self.n_cells)
            out[self.cells] = UncollidedFlux(self.beam, self.space, self.values,
                                             self.residual_energy, self.n_rays).at_energy(e_mev)
            return out
        centers = self.group_energies
        if e_mev <= centers[0] or e_mev >= centers[-1]:
            j = 0 if e_mev <= centers[0] else self.values.shape[1] - 1
            inside = self.space.e_min <= e_mev <= self.space.e_max
            return self.values[:, j] if inside else np.zeros(self.values.shape[0])
        j = int(np.searchsorted(centers, e_mev)) - 1
        w = (e_mev - centers[j]) / (centers[j + 1] - centers[j])
        return (1.0 - w) * self.values[:, j] + w * self.values[:, j + 1]


# traced tables larger than this are kept on the rays' footprint (sparse)
SPARSE_BYTES = 1 << 31


def trace_beam_ops(beam, grid, space, key_of_cell, gmats, s_min, n_side=21, span_sigmas=3.0,
                   max_step=MAX_STEP_CM, sparse=None):
    """trace_beam from assembled operators: gmats / s_min keyed by material.

    sparse: keep the (cell x group) table on the cells the rays touched only
    (UncollidedFlux.cells); None = when the dense table would exceed 2 GB."""
    shape, spacing, origin = _grid_params(grid)
    d = np.asarray(beam.direction, dtype=float)
    e1, e2 = transverse_frame(d)
    offs, wts = stratified_ray_offsets(beam.sigma_xy_cm, n_side, span_sigmas)
    psi0 = project_initial_spectrum(space, beam.energy_mev, beam.sigma_e_mev)
    start = np.asarray(beam.position_cm, dtype=float)
    starts = start[None, :] + offs[:, :1] * e1[None, :] + offs[:, 1:2] * e2[None, :]
    cells, t0, t1, offsets = traverse_rays(shape, spacing, origin, starts,
                                           np.repeat(d[None, :], len(offs), axis=0))
    keys = np.asarray(key_of_cell)
    plan = _Marches(max_step)
    by_sig = {}
    ray_seg_off, r_cells, r_len, ray_march, ray_w = [0], [], [], [], []
    n_alive = 0
    # the bundle's segments as Python scalars once (the per-ray loop below then
    # touches no numpy scalars); lengths are the same float64 differences
    off_l = offsets.tolist()
    cell_l = cells.tolist()
    len_l = (t1 - t0).tolist()
    # round(numpy float64, 12) as the reference's signature rounds (np.round)
    rnd_l = np.round(t1 - t0, 12).tolist()
    key_l = keys[cells].tolist() if len(cells) else []
    for r in range(len(offs)):
        lo, hi = off_l[r], off_l[r + 1]
        if hi == lo:
            continue                                         # ray misses the domain
        n_alive += 1
        idx = [i for i in range(lo, hi) if len_l[i] > 1e-12]
        segs = [(cell_l[i], len_l[i]) for i in idx]
        if not segs:
            continue
        sig = tuple((key_l[i], rnd_l[i]) for i in idx)
        if sig not in by_sig:
            by_sig[sig] = plan.add([(len_l[i], key_l[i]) for i in idx])
        ray_march.append(by_sig[sig])
        r_cells.extend(c for c, _ in segs)
        r_len.extend(length for _, length in segs)
        ray_seg_off.append(len(r_cells))
        ray_w.append(float(beam.weight) * float(wts[r]))
    av, res, _ = plan.run(space, gmats, s_min, psi0)
    sp = EnergySpace.of(space)
    n = shape[0] * shape[1] * shape[2]
    if sparse is None:
        sparse = n * sp.n_groups * 8 > SPARSE_BYTES
    volume = spacing[0] * spacing[1] * spacing[2]
    dep_cells = np.asarray(r_cells, dtype=np.int64)
    cells_u = None
    if sparse:
        # deposit into the footprint's rows: the same per-cell accumulation order
        cells_u = np.unique(dep_cells)
        dep_cells = np.searchsorted(cells_u, dep_cells).astype(np.int64)
        rows = max(len(cells_u), 1)
        h = handle_for((rows, 1, 1), (1.0, 1.0, 1.0), 1)
    else:
        rows = n
        h = handle_for(shape, spacing, 1)
    values = np.zeros((rows, sp.n_groups))
    residual = np.zeros(rows)
    h.call("pnd_deposit", sp.n_groups, len(ray_march), _lib.ptr(_lib.i32(ray_seg_off)),
           _lib.ptr(dep_cells), _lib.ptr(_lib.f64(r_len)),
           _lib.ptr(_lib.i32(ray_march)), _lib.ptr(_lib.i32(plan.seg_off)),
           _lib.ptr(_lib.f64(ray_w)), float(volume), len(plan.seg_key), _lib.ptr(av),
           _lib.ptr(res), _lib.ptr(values), _lib.ptr(residual))
    if sparse:
        k = len(cells_u)
        return UncollidedFlux(beam=beam, space=space, values=values[:k],
                              residual_energy=residual[:k], n_rays=n_alive,
                              cells=cells_u.astype(np.int32), n_cells=n)
    return UncollidedFlux(beam=beam, space=space, values=values, residual_energy=residual,
                          n_rays=n_alive)


def trace_beam(beam, grid, space, material_key_of_cell, coefficients, n_side=21,
               span_sigmas=3.0, max_step=MAX_STEP_CM, spectra_dump=None, sparse=None):
    """Drop-in for raytracer.trace_beam (raytracer.py:452-529): stratified
    bundle, device traversal, one device march per distinct ray signature,
    device deposit in ray order. Tables above 2 GB are returned on the rays'
    footprint (UncollidedFlux.cells; trace_beam_ops)."""
    if spectra_dump is not None:
        raise ConfigError("spectra_dump is served by the reference tracer (solver dlra-cpu)")
    keys = sorted(int(k) for k in np.unique(np.asarray(material_key_of_cell)))
    gm, smin = {}, {}
    for k in keys:
        gm[k] = assemble_energy_operators(space, *coefficients[k])[1]
        smin[k] = float(np.atleast_1d(coefficients[k][0](np.array([space.e_min])))[0])
    return trace_beam_ops(beam, grid, space, material_key_of_cell, gm, smin, n_side,
                          span_sigmas, max_step, sparse)
