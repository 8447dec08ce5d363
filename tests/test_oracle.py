"""CPU suite: pin the numpy oracle and the host-side logic to the reference.

Every expected value here was written by the reference itself
(tools/make_golden.py imports /root/reference/pkg/src and saves
tests/golden/*.npz). These tests run without a GPU (`-m "not gpu"`):
  - oracle kernels (apply_streaming, k_rhs, stencil Grams, l_rhs, s_rhs)
    against the reference's kernels.npz, <= 1e-12 (test_dlra.py:87-113,
    test_spatial.py:198-208 use the same tolerance);
  - oracle streaming/scattering steps + truncation (T2) against steps.npz;
  - the truncation rule on the reference's rule cases (test_dlra.py:211-246);
  - oracle Amanatides-Woo traversal, bit-exact, against traverse.npz;
  - an end-to-end oracle run against the reference dose (T5/T6 floors);
  - the host-side coefficient assembly of problem.py (stopping field,
    scattering tables, uncollided slices) against the reference's per-step
    contexts, and the angular operators of angular.py against angular.npz.
"""

import json
from types import SimpleNamespace

import numpy as np
import pytest

from conftest import GOLDEN, golden
from oracle import dlra_np
from oracle.traverse import traverse

KCASES = ["g3d", "g3d_b", "gz", "gyz", "gx3"]


def relmax(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(b).max(), 1e-300))


def rel(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / nb) if nb > 0 else float(
        np.linalg.norm(a))


def grid_of(arr):
    return dlra_np.Grid(int(arr[0]), int(arr[1]), int(arr[2]), float(arr[3]), float(arr[4]),
                        float(arr[5]))


def ops_of(npz, p):
    return dlra_np.Ops(list(npz[p + "eig_v"]), list(npz[p + "lam_plus"]),
                       list(npz[p + "lam_minus"]))


# ------------------------------------------------------------- T1 kernels
@pytest.mark.parametrize("case", KCASES)
def test_oracle_kernels_match_reference(kernels_npz, case):
    K, p = kernels_npz, case + "_"
    grid, ops = grid_of(K[p + "grid"]), ops_of(K, p)
    inv_s = K[p + "inv_s"]
    assert relmax(dlra_np.apply_streaming(K[p + "u_full"], inv_s, grid, ops),
                  K[p + "apply_streaming"]) < 1e-12
    st = grid.stencils()
    kf = [ops.factor(K[p + "v0"], a, s) for a, s in st]
    assert relmax(dlra_np.k_rhs(K[p + "k"], inv_s, grid, kf), K[p + "k_rhs"]) < 1e-12
    # Q_s = (D_s S^-1 U0)^T U0, stacked [axis][+, -] by the reference
    g = dlra_np.stencil_grams(K[p + "u0"], K[p + "u0"], inv_s, grid)
    q = np.array([[g[2 * i].T, g[2 * i + 1].T] for i in range(len(st) // 2)])
    assert relmax(q, K[p + "q_grams"]) < 1e-12
    l = K[p + "l"]
    l_rhs = np.zeros_like(l)
    for (a, s), qs in zip(st, [x.T for x in g]):
        l_rhs -= ops.a_mat(a, s) @ (l @ qs)
    assert relmax(l_rhs, K[p + "l_rhs"]) < 1e-12
    # s_rhs = -sum_s U0^T (D_s S^-1 U0) S F_s(V0): the precontracted Gram form
    s = K[p + "s"]
    s_rhs = np.zeros_like(s)
    for gs, fs in zip(g, kf):
        s_rhs -= gs @ s @ fs
    assert relmax(s_rhs, K[p + "s_rhs"]) < 1e-12


def test_oracle_rejects_two_cell_axis():
    with pytest.raises(ValueError, match="3-point"):
        dlra_np.Grid(2, 5, 5, 0.1, 0.1, 0.1)


# ------------------------------------------------------------- T2 steps
@pytest.mark.parametrize("case", ["str3d", "str2d", "strz"])
def test_oracle_streaming_step(steps_npz, case):
    S, p = steps_npz, case + "_"
    grid, ops = grid_of(S[p + "grid"]), ops_of(S, p)
    u, s, v = dlra_np.streaming_step(S[p + "u0"], S[p + "s0"], S[p + "v0"], float(S[p + "dt"]),
                                     S[p + "inv_s"], grid, ops)
    assert rel(u @ s @ v.T, S[p + "aug_matrix"]) < 1e-11
    sig = np.linalg.svd(s, compute_uv=False)
    assert relmax(sig[: len(S[p + "aug_sigma"])], S[p + "aug_sigma"]) < 1e-9
    r = S[p + "s0"].shape[0]
    u0, s0, v0, _ = dlra_np.truncate(u, s, v, 0.0, 1, 2 * r)
    assert s0.shape[0] == int(S[p + "trunc0_rank"])
    assert rel(u0 @ s0 @ v0.T, S[p + "trunc0_matrix"]) < 1e-11
    ur, sr, vr, tail = dlra_np.truncate(u, s, v, 1e300, r, r)
    assert rel(ur @ sr @ vr.T, S[p + "truncr_matrix"]) < 1e-10
    assert tail == pytest.approx(float(S[p + "truncr_tail"]), rel=1e-9)


@pytest.mark.parametrize("case", ["scat_h", "scat_x", "scat_max"])
def test_oracle_scattering_step(steps_npz, case):
    S, p = steps_npz, case + "_"
    u, s, v = dlra_np.scattering_step(S[p + "u0"], S[p + "s0"], S[p + "v0"], float(S[p + "dt"]),
                                      S[p + "weights"], S[p + "inv_s"], S[p + "g_diags"],
                                      S[p + "sigma_t"], list(zip(S[p + "psi"], S[p + "tm"])))
    assert rel(u @ s @ v.T, S[p + "aug_matrix"]) < 1e-11
    assert tuple(s.shape) == tuple(int(x) for x in S[p + "aug_shape"])


def test_oracle_truncation_rule_cases(steps_npz):
    for row in steps_npz["trunc_cases"]:
        theta, rmin, rmax, rank, tail = row[:5]
        sig = row[5:]
        q = sig.size
        u1, s1, v1, t = dlra_np.truncate(np.eye(q), np.diag(sig), np.eye(q), theta, int(rmin),
                                         int(rmax))
        assert s1.shape[0] == int(rank)
        assert t == pytest.approx(tail, rel=1e-12, abs=1e-300)


# ------------------------------------------------------------- T0 traversal
def test_oracle_traversal_bit_exact(traverse_npz):
    T = traverse_npz
    for gname in T["grids"]:
        p = str(gname) + "_"
        gr = T[p + "grid"]
        shape, spacing, origin = tuple(int(v) for v in gr[:3]), tuple(gr[3:6]), tuple(gr[6:9])
        offs = T[p + "offsets"]
        for i, (o, d) in enumerate(zip(T[p + "origins"], T[p + "dirs"])):
            segs = traverse(shape, spacing, origin, o, d)
            lo, hi = offs[i], offs[i + 1]
            assert [c for c, _, _ in segs] == list(T[p + "cells"][lo:hi])
            t0 = np.array([a for _, a, _ in segs], dtype=np.float64)
            t1 = np.array([b for _, _, b in segs], dtype=np.float64)
            np.testing.assert_array_equal(t0.view(np.int64), T[p + "t0"][lo:hi].view(np.int64))
            np.testing.assert_array_equal(t1.view(np.int64), T[p + "t1"][lo:hi].view(np.int64))


# ------------------------------------------------------------- T2 at the benchmarked physics
@pytest.mark.parametrize("tag,k", [("fp19", 25), ("slabs7", 150)])
def test_oracle_lockstep_substeps(tag, k):
    """The oracle's substeps from the reference's own states at the bench's
    physics (P19 Fokker-Planck m = 400; three-class Boltzmann P7; rank 20)
    reproduce the reference's augmented factors (T2, lock_<tag>.npz)."""
    L = golden(f"lock_{tag}.npz")
    B = golden(f"bundle_{tag}.npz")
    grid = grid_of(L["grid"])
    ops = dlra_np.Ops(list(B["eig_v"]), list(B["lam_plus"]), list(B["lam_minus"]))
    p = f"k{k}_"
    dt, inv_s = float(L[p + "dt"]), L[p + "inv_s"]
    u, s, v = dlra_np.streaming_step(L[p + "u"], L[p + "s"], L[p + "v"], dt, inv_s, grid, ops)
    want = L[p + "sa_u"] @ L[p + "sa_s"] @ L[p + "sa_v"].T
    assert rel(u @ s @ v.T, want) < 1e-11
    sources = list(zip(L[p + "psi"], L["t_ms"]))
    u, s, v = dlra_np.scattering_step(L[p + "st_u"], L[p + "st_s"], L[p + "st_v"], dt,
                                      L["weights"], inv_s, L[p + "g_diags"], L[p + "sigma_t"],
                                      sources)
    want = L[p + "ca_u"] @ L[p + "ca_s"] @ L[p + "ca_v"].T
    assert rel(u @ s @ v.T, want) < 1e-11


# ------------------------------------------------------------- end to end
FLOORS = json.loads((GOLDEN / "floors.json").read_text())


@pytest.mark.parametrize("tag", ["smoke", "rank1"])
def test_oracle_end_to_end_dose(tag):
    from paper_2508_04484_b200.problem import ProblemBundle

    b = ProblemBundle.load(GOLDEN / f"bundle_{tag}.npz")
    g = golden(f"e2e_{tag}.npz")
    out = dlra_np.run_energy_loop(b)
    np.testing.assert_array_equal(np.array(out["rank_history"]),
                                  g["rank_history"][:, 2].astype(int))
    # the reference adds the uncollided dose after the loop (driver.py:613-625)
    unc = g["uncollided"] if b.uncollided_tally != "steps" else 0.0
    dep = out["deposited"] + unc
    assert rel(dep, g["deposited"]) <= max(10.0 * FLOORS[tag]["total"], 1e-12)
    assert rel(out["deposited"], g["deposited"] - unc) <= max(
        10.0 * FLOORS[tag]["collided"], 1e-10)


# ------------------------------------------------------------- host logic
@pytest.mark.parametrize("tag", ["smoke", "hetero", "fp", "config1"])
def test_problem_contexts_match_reference(tag):
    """problem.py's per-step coefficients (stopping field, 1/S, Moliere g
    diagonals, sigma_t, uncollided slice) vs the reference's step_contexts
    (driver.py:523-538) at the recorded steps."""
    from paper_2508_04484_b200.problem import ProblemBundle

    b = ProblemBundle.load(GOLDEN / f"bundle_{tag}.npz")
    g = golden(f"e2e_{tag}.npz")
    edges = b.pseudo_time_edges()
    np.testing.assert_allclose(edges, g["edges"], rtol=0, atol=1e-12)
    for k in g["ctx_steps"]:
        p = f"ctx{int(k)}_"
        e_mid = 0.5 * (edges[k] + edges[k + 1])
        s_field = b.stopping_field(e_mid)
        assert relmax(s_field, g[p + "s_field"]) < 1e-14
        assert relmax(1.0 / s_field, g[p + "inv_s"]) < 1e-14
        gd, st = b.scattering_tables(e_mid)
        assert relmax(gd, g[p + "g_diags"]) < 1e-13
        assert relmax(st, g[p + "sigma_t"]) < 1e-13
        psi = b.psi_at(e_mid)
        assert relmax(psi, g[p + "psi"]) < 1e-13


@pytest.mark.parametrize("n_max", [1, 2, 3, 5, 7])
def test_angular_operators_match_reference(n_max):
    from paper_2508_04484_b200.angular import PNOperators, beam_projection

    A = golden("angular.npz")
    ops = PNOperators.build(n_max)
    for axis in range(3):
        ap = (ops.eig_v[axis] * ops.lam_plus[axis]) @ ops.eig_v[axis].T
        am = (ops.eig_v[axis] * ops.lam_minus[axis]) @ ops.eig_v[axis].T
        assert relmax(ap, A[f"aplus_{n_max}_{axis}"]) < 1e-12
        assert relmax(am, A[f"aminus_{n_max}_{axis}"]) < 1e-12
    assert relmax(beam_projection(n_max, (0.0, 0.6, 0.8)), A[f"tm_{n_max}"]) < 1e-12


# ------------------------------------------------------------- tracer host logic
def test_energy_operators_and_ray_bundle_match_reference():
    """raytracer.py host restatements: energy operators (169-274), initial
    spectrum (157-166), ray offsets/weights (406-418), transverse frame (60-69)."""
    from paper_2508_04484_b200 import raytracer as rt

    M = golden("march.npz")
    space = rt.EnergySpace(1.0, 31.5, 32, 2)

    def const(v):
        return lambda e: np.full_like(np.asarray(e, dtype=float), v)

    coeff = {0: (lambda e: 2.0 + 0.05 * np.asarray(e, dtype=float), const(0.04), const(0.3)),
             1: (const(4.0), None, None)}
    for k in (0, 1):
        mass, g = rt.assemble_energy_operators(space, *coeff[k])
        assert relmax(g, M[f"g_{k}"]) < 1e-14
        np.testing.assert_array_equal(mass, M["mass"])
    assert relmax(rt.project_initial_spectrum(space, 30.0, 0.3), M["psi0"]) < 1e-14
    T = golden("trace.npz")
    for b in range(int(T["n_beams"])):
        p = f"b{b}_"
        beam, rays = T[p + "beam"], T[p + "rays"]
        off, wts = rt.stratified_ray_offsets(beam[8], int(rays[0]), float(rays[1]))
        np.testing.assert_array_equal(off, T[p + "offsets"])
        np.testing.assert_array_equal(wts, T[p + "weights"])
        np.testing.assert_array_equal(np.stack(rt.transverse_frame(beam[:3])), T[p + "frame"])


def test_footprint_flux_equals_dense():
    """The ray-footprint (sparse) form of an uncollided table (UncollidedSlices
    with cells): at_energy and the group-sum tally equal the dense table's
    bit for bit (the cells outside the footprint hold zeros)."""
    import dataclasses

    from paper_2508_04484_b200.problem import ProblemBundle, UncollidedSlices

    b = ProblemBundle.load(GOLDEN / "bundle_hetero.npz")
    sparse = []
    for f in b.fluxes:
        cells = np.flatnonzero(np.any(f.values != 0.0, axis=1) | (f.residual != 0.0))
        sparse.append(UncollidedSlices(f.values[cells], f.residual[cells], f.e_min, f.e_max,
                                       cells.astype(np.int32), b.n_cells))
        assert len(cells) < b.n_cells
    bs = dataclasses.replace(b, fluxes=sparse)
    for e in (1.0, 5.3, 12.77, 22.0, 25.9, 30.0):
        np.testing.assert_array_equal(bs.psi_at(e), b.psi_at(e))
    np.testing.assert_array_equal(bs.uncollided_dose(), b.uncollided_dose())
    np.testing.assert_array_equal(sparse[0].dense().values, b.fluxes[0].values)
