"""GPU parity of the CUDA path (through the C-ABI) against the reference.

Tiers follow SURVEY.md §8(c):
  T0 bit-exact voxel lists and t-intervals (traversal);
  T1 kernel level on identical inputs, <= 1e-12 relative (FP64 reordering);
  T2 single-step reconstruction U S V^T after streaming / scattering /
     truncation, <= 1e-11 relative;
  T3 maximal-rank lockstep DLRA vs full rank, <= 1e-8;
  T4/T5 end-to-end dose vs the reference: dev <= 10 x the gauge floor of
     tests/golden/floors.json (written by tools/measure_floors.py) with equal
     rank histories; T6 the rank-1 regime.
Every expected value comes from the reference (tests/golden/*.npz) or the
numpy oracle pinned to it (tests/test_oracle.py).
"""

import json
from types import SimpleNamespace

import numpy as np
import pytest

from conftest import GOLDEN, golden

pytestmark = pytest.mark.gpu


def rel(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / nb) if nb > 0 else float(
        np.linalg.norm(a))


def relmax(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(b).max(), 1e-300))


def grid_ns(arr):
    nx, ny, nz = (int(v) for v in arr[:3])
    return SimpleNamespace(nx=nx, ny=ny, nz=nz, dx=float(arr[3]), dy=float(arr[4]),
                           dz=float(arr[5]))


def ops_ns(npz, p):
    return SimpleNamespace(eig_v=list(npz[p + "eig_v"]), lam_plus=list(npz[p + "lam_plus"]),
                           lam_minus=list(npz[p + "lam_minus"]))


KCASES = ["g3d", "g3d_b", "gz", "gyz", "gx3"]


@pytest.fixture(scope="module")
def dl():
    from paper_2508_04484_b200 import dlra

    return dlra


# ------------------------------------------------------------------ T1
@pytest.mark.parametrize("case", KCASES)
def test_apply_streaming(dl, kernels_npz, case):
    p = case + "_"
    K = kernels_npz
    ctx = dl.StreamingContext(K[p + "inv_s"], SimpleNamespace(grid=grid_ns(K[p + "grid"])),
                              ops_ns(K, p))
    got = ctx.full_rhs(K[p + "u_full"])
    assert relmax(got, K[p + "apply_streaming"]) < 1e-12


@pytest.mark.parametrize("case", KCASES)
def test_k_rhs_and_l_grams(dl, kernels_npz, case):
    p = case + "_"
    K = kernels_npz
    ctx = dl.StreamingContext(K[p + "inv_s"], SimpleNamespace(grid=grid_ns(K[p + "grid"])),
                              ops_ns(K, p))
    got = ctx.k_rhs(K[p + "k"], ctx._moment_factors(K[p + "v0"]))
    assert relmax(got, K[p + "k_rhs"]) < 1e-12
    lf = ctx.l_step_factors(K[p + "u0"])
    q = np.array([[f[2], f[3]] for f in lf])
    assert relmax(q, K[p + "q_grams"]) < 1e-12
    got_l = ctx.l_rhs(K[p + "l"], lf)
    assert relmax(got_l, K[p + "l_rhs"]) < 1e-12
    sf = ctx.s_step_factors(K[p + "u0"], K[p + "v0"])
    assert relmax(ctx.s_rhs(K[p + "s"], K[p + "u0"], sf), K[p + "s_rhs"]) < 1e-11


def test_non_finite_streaming_input(dl, kernels_npz):
    from paper_2508_04484_b200.errors import NumericalError

    p = "gz_"
    K = kernels_npz
    ctx = dl.StreamingContext(K[p + "inv_s"], SimpleNamespace(grid=grid_ns(K[p + "grid"])),
                              ops_ns(K, p))
    u = K[p + "u_full"].copy()
    u[0, 0] = np.nan
    with pytest.raises(NumericalError, match="non-finite"):
        ctx.full_rhs(u)


def test_two_cell_axis_rejected(dl, kernels_npz):
    from paper_2508_04484_b200.errors import ConfigError

    K = kernels_npz
    p = "g3d_"
    grid = SimpleNamespace(nx=2, ny=3, nz=3, dx=0.1, dy=0.1, dz=0.1)
    ctx = dl.StreamingContext(np.ones(18), SimpleNamespace(grid=grid), ops_ns(K, p))
    with pytest.raises(ConfigError, match="3-point"):
        ctx.full_rhs(np.zeros((18, K[p + "eig_v"].shape[1])))


@pytest.mark.parametrize("shape", [(7, 3), (40, 6), (300, 12), (1000, 40), (5, 9), (129, 64),
                                   (4000, 2), (400, 128), (600, 100)])
def test_orthonormalize_tsqr(dl, shape):
    rng = np.random.default_rng(sum(shape))
    a = rng.standard_normal(shape)
    if shape[1] >= 4:
        a[:, 1] = 0.0                      # exactly zero column
        a[:, 3] = 2.0 * a[:, 2]            # rank deficiency
    q = dl.orthonormal_columns(a)
    k = min(shape)
    assert q.shape == (shape[0], k)
    assert np.abs(q.T @ q - np.eye(k)).max() < 1e-13
    # the span of a is contained in span(q)
    assert np.abs(q @ (q.T @ a) - a).max() < 1e-12 * max(1.0, np.abs(a).max())


def test_orthonormalize_tall_beyond_grid_y(dl):
    """n > 65535 x 32 rows (the 128^3 initial state): the layout transposes put
    rows on grid x (grid y is capped at 65535 blocks)."""
    rng = np.random.default_rng(11)
    a = rng.standard_normal((2_200_000, 2))
    q = dl.orthonormal_columns(a)
    assert np.abs(q.T @ q - np.eye(2)).max() < 1e-13
    assert np.abs(q @ (q.T @ a) - a).max() < 1e-10 * np.abs(a).max()


def test_orthonormalize_zero_block_is_canonical(dl):
    # [0 | U0] -> first columns are +e_0.. (reference step-0 behaviour, Appendix C.4)
    rng = np.random.default_rng(5)
    u0 = np.linalg.qr(rng.standard_normal((700, 5)))[0]
    q = dl.orthonormal_columns(np.hstack([np.zeros((700, 5)), u0]))
    np.testing.assert_array_equal(q[:, :5], np.eye(700)[:, :5])


@pytest.mark.parametrize("pq", [(6, 6), (10, 4), (4, 10), (40, 40), (32, 16),
                                # wide R x R (global work buffer): ranks up to 64
                                (100, 100), (128, 128), (128, 80), (90, 128)])
def test_svd_small(pq):
    from paper_2508_04484_b200 import _lib
    from paper_2508_04484_b200.dlra import _generic_handle

    p, q = pq
    rng = np.random.default_rng(p * 100 + q)
    s = rng.standard_normal((p, q)) * np.exp(-0.3 * np.arange(q))
    k = min(p, q)
    pm, sig, qt = np.empty((p, k)), np.empty(k), np.empty((k, q))
    _generic_handle().call("pnd_svd_small", _lib.ptr(s), p, q, _lib.ptr(pm), _lib.ptr(sig),
                           _lib.ptr(qt))
    ref = np.linalg.svd(s, compute_uv=False)
    assert relmax(sig, ref) < 1e-13
    assert np.abs(pm.T @ pm - np.eye(k)).max() < 1e-13
    assert np.abs(qt @ qt.T - np.eye(k)).max() < 1e-13
    assert relmax(pm @ np.diag(sig) @ qt, s) < 1e-13
    # zero matrix -> identity factors (np.linalg.svd(0) convention)
    z = np.zeros((p, q))
    _generic_handle().call("pnd_svd_small", _lib.ptr(z), p, q, _lib.ptr(pm), _lib.ptr(sig),
                           _lib.ptr(qt))
    np.testing.assert_array_equal(pm, np.eye(p, k))
    np.testing.assert_array_equal(qt, np.eye(k, q))


# ------------------------------------------------------------------ T2
@pytest.mark.parametrize("case", ["str3d", "str2d", "strz"])
def test_streaming_step_and_truncate(dl, steps_npz, case):
    S = steps_npz
    p = case + "_"
    ctx = dl.StreamingContext(S[p + "inv_s"], SimpleNamespace(grid=grid_ns(S[p + "grid"])),
                              ops_ns(S, p))
    st = dl.LowRankState(S[p + "u0"], S[p + "s0"], S[p + "v0"])
    aug = dl.streaming_step(st, float(S[p + "dt"]), ctx)
    assert aug.orthonormality_defect() < 1e-13
    assert rel(aug.matrix(), S[p + "aug_matrix"]) < 1e-11
    sig = np.linalg.svd(aug.s, compute_uv=False)
    assert relmax(sig[: len(S[p + "aug_sigma"])], S[p + "aug_sigma"]) < 1e-9
    r = st.s.shape[0]
    tr0, tail0 = dl.truncate(aug, dl.TruncationPolicy(0.0, 1, 2 * r))
    assert tr0.rank == int(S[p + "trunc0_rank"])
    assert rel(tr0.matrix(), S[p + "trunc0_matrix"]) < 1e-11
    trr, tailr = dl.truncate(aug, dl.TruncationPolicy(1e300, r, r))
    assert rel(trr.matrix(), S[p + "truncr_matrix"]) < 1e-10
    assert tailr == pytest.approx(float(S[p + "truncr_tail"]), rel=1e-9)


@pytest.mark.parametrize("case", ["scat_h", "scat_x", "scat_max"])
def test_scattering_step_and_truncate(dl, steps_npz, case):
    S = steps_npz
    p = case + "_"
    ctx = dl.ScatteringContext(S[p + "weights"], S[p + "inv_s"], S[p + "g_diags"],
                               S[p + "sigma_t"], list(zip(S[p + "psi"], S[p + "tm"])))
    st = dl.LowRankState(S[p + "u0"], S[p + "s0"], S[p + "v0"])
    aug = dl.scattering_step(st, float(S[p + "dt"]), ctx)
    # the reference normalises rounding noise of the rank-deficient augmentation
    # into extra Householder directions (singular values ~1e-23); the device
    # deflates them, so compare the numerical rank
    ref_sig = S[p + "aug_sigma"]
    numerical = int(np.count_nonzero(ref_sig > 1e-12 * ref_sig[0]))
    sig = np.linalg.svd(aug.s, compute_uv=False)
    assert numerical <= min(aug.s.shape) <= S[p + "aug_shape"].min()
    assert relmax(sig[:numerical], ref_sig[:numerical]) < 1e-9
    assert aug.orthonormality_defect() < 1e-12
    assert rel(aug.matrix(), S[p + "aug_matrix"]) < 1e-11
    r = st.s.shape[0]
    tr0, _ = dl.truncate(aug, dl.TruncationPolicy(0.0, 1, 2 * r))
    assert numerical <= tr0.rank <= int(S[p + "trunc0_rank"])
    assert rel(tr0.matrix(), S[p + "trunc0_matrix"]) < 1e-10


def test_truncation_rule_cases(dl, steps_npz):
    for row in steps_npz["trunc_cases"]:
        theta, rmin, rmax, rank, tail = row[:5]
        sig = row[5:]
        q = sig.size
        st = dl.LowRankState(np.eye(q), np.diag(sig), np.eye(q))
        out, t = dl.truncate(st, dl.TruncationPolicy(theta, int(rmin), int(rmax)))
        assert out.rank == int(rank)
        assert t == pytest.approx(tail, rel=1e-12, abs=1e-300)


def test_truncation_rank_max_error(dl):
    from paper_2508_04484_b200.errors import NumericalError

    rng = np.random.default_rng(29)
    u = np.linalg.qr(rng.standard_normal((20, 6)))[0]
    v = np.linalg.qr(rng.standard_normal((10, 6)))[0]
    st = dl.LowRankState(u, np.diag([4.0, 2.0, 1.0, 0.5, 0.1, 0.01]), v)
    out, _ = dl.truncate(st, dl.TruncationPolicy(100.0, rank_min=3, rank_max=5))
    assert out.rank == 3
    with pytest.raises(NumericalError, match="rank_max"):
        dl.truncate(st, dl.TruncationPolicy(1e-9, rank_min=1, rank_max=2))


def test_singular_implicit_solve_reports_column(dl):
    from paper_2508_04484_b200.errors import NumericalError

    n, m, r = 4, 3, 2
    state = dl.LowRankState(u=np.eye(n)[:, :r], s=np.eye(r), v=np.eye(m)[:, :r])
    ctx = dl.ScatteringContext(np.ones((n, 12)) / 12.0, np.ones(n), np.zeros((12, m)),
                               -np.ones(12), [])
    with pytest.raises(NumericalError, match="column 0"):
        dl.scattering_step(state, 1.0, ctx)


# ------------------------------------------------------------------ T0
def test_traverse_bit_exact(traverse_npz):
    from paper_2508_04484_b200.raytracer import traverse_rays

    T = traverse_npz
    for gname in T["grids"]:
        p = str(gname) + "_"
        gr = T[p + "grid"]
        cells, t0, t1, offs = traverse_rays(tuple(int(v) for v in gr[:3]), tuple(gr[3:6]),
                                            tuple(gr[6:9]), T[p + "origins"], T[p + "dirs"])
        np.testing.assert_array_equal(offs, T[p + "offsets"])
        np.testing.assert_array_equal(cells, T[p + "cells"])
        # bit-exact float64 intervals
        np.testing.assert_array_equal(t0.view(np.int64), T[p + "t0"].view(np.int64))
        np.testing.assert_array_equal(t1.view(np.int64), T[p + "t1"].view(np.int64))


# ------------------------------------------------------------------ T3
def test_lockstep_maximal_rank_vs_fullrank():
    """Acceptance criterion 2 (test_acceptance.py:101-152) on the device:
    DLRA at maximal rank r = m = 16 vs the full-rank oracle, <= 1e-8."""
    from oracle import dlra_np
    from paper_2508_04484_b200.driver import DeviceSolver
    from paper_2508_04484_b200.problem import ProblemBundle

    b = ProblemBundle.load(GOLDEN / "bundle_lockstep.npz")
    grid = dlra_np.Grid(*b.shape, *b.spacing)
    ops = dlra_np.Ops(b.eig_v, b.lam_plus, b.lam_minus)
    solver = dlra_np.Grid  # noqa: F841
    dev = DeviceSolver(b)
    dev.init_state(rank=16)
    edges = b.pseudo_time_edges()
    n, m = b.n_cells, b.n_moments
    u = np.zeros((n, m))
    weights = b.atomic_densities
    worst = 0.0
    for k in range(len(edges) - 1):
        dt = edges[k] - edges[k + 1]
        dev.set_coefficients(edges[k], edges[k + 1])
        dev.step(dt, want_defect=False)
        e_mid = 0.5 * (edges[k] + edges[k + 1])
        inv_s = 1.0 / b.stopping_field(e_mid)
        g, s = b.scattering_tables(e_mid)
        u = dlra_np.fullrank_streaming_step(u, dt, inv_s, grid, ops)
        u = dlra_np.fullrank_scattering_step(u, dt, weights, inv_s, g, s,
                                             list(zip(b.psi_at(e_mid), b.t_ms)))
        if k % 20 == 0 or k == len(edges) - 2:
            uu, ss, vv = dev.state()
            norm = np.linalg.norm(u)
            if norm > 0:
                worst = max(worst, np.linalg.norm(uu @ ss @ vv.T - u) / norm)
    dev.close()
    assert worst <= 1e-8, worst


# ------------------------------------------------------------------ T4/T5/T6
FLOORS = json.loads((GOLDEN / "floors.json").read_text())


@pytest.mark.parametrize("tag", ["rank1", "hetero", "smoke", "fp", "config1", "fp19", "slabs7"])
def test_end_to_end_dose(tag, parity_log):
    """T4/T5/T6 end to end against the reference's own run (tests/golden/
    e2e_<tag>.npz). The bound is 10 x the gauge floor: the deviation of a
    correct CPU restatement (the oracle) from the reference on the same
    inputs, with and without a 1e-15 basis rotation (tools/measure_floors.py).
    Every measured deviation is logged next to its floor ($PND_PARITY_OUT)."""
    from paper_2508_04484_b200.driver import run_bundle
    from paper_2508_04484_b200.problem import ProblemBundle

    b = ProblemBundle.load(GOLDEN / f"bundle_{tag}.npz")
    g = golden(f"e2e_{tag}.npz")
    res = run_bundle(b)
    dep = res.dose.deposited
    unc = g["uncollided"]
    ranks = np.array([r for _, _, r in res.rank_history])
    floor = FLOORS[tag]
    dev_total = rel(dep, g["deposited"])
    dev_coll = rel(dep - unc, g["deposited"] - unc)
    coll_frac = float(np.linalg.norm(g["deposited"] - unc) / np.linalg.norm(g["deposited"]))
    parity_log.append({
        "test": "end_to_end_dose", "tag": tag, "n_steps": int(len(ranks)),
        "dev_total": dev_total, "floor_total": floor["total"],
        "oracle_total": floor["impl"]["total"],
        "dev_collided": dev_coll, "floor_collided": floor["collided"],
        "oracle_collided": floor["impl"]["collided"],
        "collided_fraction_of_total": coll_frac,
        "ranks_equal": bool(np.array_equal(ranks, g["rank_history"][:, 2].astype(int))),
        "max_orthonormality_defect": float(res.diagnostics["max_orthonormality_defect"]),
    })
    np.testing.assert_array_equal(ranks, g["rank_history"][:, 2].astype(int))
    assert res.diagnostics["max_orthonormality_defect"] < 1e-10
    assert res.diagnostics["tail_violations"] == 0
    assert dev_total <= max(10.0 * floor["total"], 1e-12), (dev_total, floor)
    assert dev_coll <= max(10.0 * floor["collided"], 1e-10), (dev_coll, floor)
    if tag == "config1":
        # T4: BASELINE configs[0]'s total dose within 1e-9 of
        # the reference -- bounded below by the reference's own gauge floor:
        # a 1e-15 basis rotation of the reference moves its total dose by
        # 2.1e-9 and the oracle (the same algorithm in numpy) lands at 1.5e-9,
        # so a rounding-level change of any kernel moves this value within
        # ~[5e-10, 2e-9]. Asserted at max(1e-9, that floor),
        # without the 10x slack of the other bundles; the value is logged.
        assert dev_total <= max(1e-9, floor["eps"]["total"]), (dev_total, floor["eps"])


# ------------------------------------------------------------------ larger ranks
@pytest.mark.parametrize("r", [24, 30, 32, 40, 48, 64])
def test_streaming_step_large_rank_vs_oracle(dl, r):
    """Ranks above the bench's 20 (16-cell K-stage chunks, 8-cell Gram chunks;
    above 32 the 32-column block chains of wide.cu): a streaming step +
    truncation against the numpy oracle (pinned to the reference by
    test_oracle.py), T2 tolerances."""
    from oracle import dlra_np
    from paper_2508_04484_b200.angular import PNOperators

    ops = PNOperators.build(7)
    nx, ny, nz = 10, 9, 11
    n, m = nx * ny * nz, ops.size
    rng = np.random.default_rng(r)
    inv_s = 1.0 / rng.uniform(5.0, 12.0, n)
    u0 = np.linalg.qr(rng.standard_normal((n, r)))[0]
    v0 = np.linalg.qr(rng.standard_normal((m, r)))[0]
    s0 = np.diag(np.logspace(0, -4, r)) + 1e-3 * rng.standard_normal((r, r))
    grid = SimpleNamespace(nx=nx, ny=ny, nz=nz, dx=0.1, dy=0.12, dz=0.09)
    ctx = dl.StreamingContext(inv_s, SimpleNamespace(grid=grid), ops)
    aug = dl.streaming_step(dl.LowRankState(u0, s0, v0), 0.01, ctx)
    ou, os_, ov = dlra_np.streaming_step(u0, s0, v0, 0.01, inv_s,
                                         dlra_np.Grid(nx, ny, nz, 0.1, 0.12, 0.09),
                                         dlra_np.Ops(ops.eig_v, ops.lam_plus, ops.lam_minus))
    want = ou @ os_ @ ov.T
    assert aug.orthonormality_defect() < 1e-12
    assert rel(aug.matrix(), want) < 1e-11
    tr, _ = dl.truncate(aug, dl.TruncationPolicy(1e300, r, r))
    _, ts, _, _ = dlra_np.truncate(ou, os_, ov, 1e300, r, r)
    np.testing.assert_allclose(np.diag(tr.s), np.diag(ts), rtol=1e-9)


@pytest.mark.parametrize("r,hetero", [(40, False), (48, True), (64, False)])
def test_scattering_step_wide_rank_vs_oracle(dl, r, hetero):
    """Ranks above 32 in the scattering step (one class: the rank-one source
    path; several classes and two beams: the source-row path with per-class
    Gram passes) against the numpy oracle, T2 tolerances."""
    from oracle import dlra_np

    rng = np.random.default_rng(r)
    n, m = 700, 81
    if hetero:
        cls = rng.integers(0, 3, n)
        weights = (np.abs(rng.standard_normal((3, 12))) * 1e22)[cls]
        n_src = 2
    else:
        weights = np.tile(np.abs(rng.standard_normal(12)), (n, 1)) * 1e22
        n_src = 1
    g_diags = np.abs(rng.standard_normal((12, m))) * 1e-28
    sigma_t = g_diags[:, 0] + np.abs(rng.standard_normal(12)) * 1e-28
    inv_s = 1.0 / rng.uniform(8.0, 20.0, n)
    sources = [(np.abs(rng.standard_normal(n)), rng.standard_normal(m)) for _ in range(n_src)]
    u0 = np.linalg.qr(rng.standard_normal((n, r)))[0]
    v0 = np.linalg.qr(rng.standard_normal((m, r)))[0]
    s0 = np.diag(np.logspace(0, -1, r)) + 0.05 * rng.standard_normal((r, r))
    ctx = dl.ScatteringContext(weights, inv_s, g_diags, sigma_t, sources)
    aug = dl.scattering_step(dl.LowRankState(u0, s0, v0), 0.3, ctx)
    ou, os_, ov = dlra_np.scattering_step(u0, s0, v0, 0.3, weights, inv_s, g_diags, sigma_t,
                                          sources)
    assert aug.orthonormality_defect() < 1e-12
    assert rel(aug.matrix(), ou @ os_ @ ov.T) < 1e-11


@pytest.mark.parametrize("r", [40, 64])
def test_wide_k_rhs_and_stencil_grams_vs_oracle(dl, r):
    """The block chains of wide.cu in isolation: K' = -sum_s (D_s S^-1 K) F_s
    and the stencil Grams X^T D_s S^-1 Y for more than 32 / 64 columns,
    against the numpy oracle's stencils (T1 tolerance)."""
    from oracle import dlra_np
    from paper_2508_04484_b200.angular import PNOperators

    ops = PNOperators.build(7)
    nx, ny, nz = 7, 6, 9
    n = nx * ny * nz
    rng = np.random.default_rng(r + 1)
    grid = dlra_np.Grid(nx, ny, nz, 0.1, 0.12, 0.09)
    inv_s = 1.0 / rng.uniform(5.0, 12.0, n)
    ctx = dl.StreamingContext(inv_s, SimpleNamespace(grid=SimpleNamespace(
        nx=nx, ny=ny, nz=nz, dx=0.1, dy=0.12, dz=0.09)), ops)
    k = rng.standard_normal((n, r))
    fac = [(rng.standard_normal((r, r)), rng.standard_normal((r, r))) for _ in range(3)]
    got = ctx.k_rhs(k, fac)
    want = np.zeros_like(k)
    for i, (axis, sign) in enumerate(grid.stencils()):
        want -= dlra_np.stencil(grid, axis, sign, inv_s[:, None] * k) @ fac[axis][0 if sign > 0 else 1]
    assert relmax(got, want) < 1e-12
    x = rng.standard_normal((n, r))
    y = rng.standard_normal((n, r))
    got_g = ctx.stencil_grams(x, y)
    for i, (axis, sign) in enumerate(grid.stencils()):
        ref = x.T @ dlra_np.stencil(grid, axis, sign, inv_s[:, None] * y)
        assert relmax(got_g[i], ref) < 1e-12


# ------------------------------------------------------------------ determinism, checkpoint
def test_rerun_is_bit_identical():
    """Determinism contract (driver.py:12-13, test_driver.py:266-283): the
    same bundle run twice gives byte-identical doses and rank histories
    (fixed-order reductions everywhere, no atomics on the Gram paths)."""
    from paper_2508_04484_b200.driver import run_bundle
    from paper_2508_04484_b200.problem import ProblemBundle

    b = ProblemBundle.load(GOLDEN / "bundle_hetero.npz")
    r1 = run_bundle(b, max_steps=60)
    r2 = run_bundle(b, max_steps=60)
    assert r1.dose.deposited.tobytes() == r2.dose.deposited.tobytes()
    assert r1.rank_history == r2.rank_history


def test_checkpoint_resume_is_bit_identical(tmp_path):
    """SURVEY.md §5 checkpoint/resume: a snapshot at a step boundary, saved,
    reloaded into a fresh solver, continues to the same bytes as the
    uninterrupted run."""
    from paper_2508_04484_b200.driver import run_bundle
    from paper_2508_04484_b200.problem import ProblemBundle

    b = ProblemBundle.load(GOLDEN / "bundle_config1.npz")
    full = run_bundle(b, max_steps=40, checkpoint_at=17)
    path = tmp_path / "ckpt.npz"
    np.savez(path, **full.diagnostics["checkpoint"])
    ck = dict(np.load(path))
    rest = run_bundle(b, max_steps=40 - 17, resume=ck)
    assert rest.dose.deposited.tobytes() == full.dose.deposited.tobytes()
    assert rest.rank_history == full.rank_history[17:]


# ------------------------------------------------------------------ graded increments
@pytest.mark.parametrize("a,b,bottom", [(6, 8, 1e-12), (20, 20, 1e-11), (0, 12, 1e-13),
                                        (10, 16, 1e-9)])
def test_augmentation_keeps_graded_directions(a, b, bottom):
    """The augmentation's span on an increment whose projected singular
    values are graded from 1 down to `bottom` (below the one-pass Gram's
    1e-7 resolution): the reference's Householder QR keeps every direction
    (dlra.py:26-43), so (I - U U^T - Q Q^T) X must vanish to rounding and Q
    must be orthonormal and orthogonal to U -- the second level of the
    device augmentation (step.cu orth_complement)."""
    from paper_2508_04484_b200 import _lib
    from paper_2508_04484_b200.dlra import handle_for

    n = 3000
    rng = np.random.default_rng(a * 100 + b)
    basis = np.linalg.qr(rng.standard_normal((n, a + b)))[0]
    u, y = basis[:, :a], basis[:, a:]
    sig = np.logspace(0, np.log10(bottom), b)
    x = y @ (sig[:, None] * np.linalg.qr(rng.standard_normal((b, b)))[0])
    if a:
        x += u @ rng.standard_normal((a, b))
    h = handle_for((n, 1, 1), (1.0, 1.0, 1.0), 4)
    q = np.zeros((n, b))
    k = np.zeros(1, dtype=np.int32)
    h.call("pnd_augment_basis", _lib.ptr(np.ascontiguousarray(u)) if a else None, a,
           _lib.ptr(np.ascontiguousarray(x)), b, 0, _lib.ptr(q), _lib.ptr(k))
    k = int(k[0])
    q = q[:, :k]
    assert k == b
    assert np.abs(q.T @ q - np.eye(k)).max() < 1e-13
    if a:
        assert np.abs(u.T @ q).max() < 1e-13
    resid = x - (u @ (u.T @ x) if a else 0.0) - q @ (q.T @ x)
    assert np.linalg.norm(resid) < 1e-14 * np.linalg.norm(x)


def test_augmentation_drops_rounding_noise():
    """A rank-deficient increment (rank 3 of 10 columns, the scattering
    source's case) gives 3 directions, not normalised rounding noise."""
    from paper_2508_04484_b200 import _lib
    from paper_2508_04484_b200.dlra import handle_for

    n, a, b = 2000, 5, 10
    rng = np.random.default_rng(3)
    basis = np.linalg.qr(rng.standard_normal((n, a + 3)))[0]
    u = basis[:, :a]
    x = basis[:, a:] @ rng.standard_normal((3, b)) + u @ rng.standard_normal((a, b))
    h = handle_for((n, 1, 1), (1.0, 1.0, 1.0), 4)
    q = np.zeros((n, b))
    k = np.zeros(1, dtype=np.int32)
    h.call("pnd_augment_basis", _lib.ptr(np.ascontiguousarray(u)), a,
           _lib.ptr(np.ascontiguousarray(x)), b, 0, _lib.ptr(q), _lib.ptr(k))
    assert int(k[0]) == 3


@pytest.mark.parametrize("shape", [(7, 6, 9), (3, 4, 5), (1, 6, 7), (1, 1, 12), (5, 3, 1),
                                   (10, 9, 11)])
def test_stencil_grams_uniform_s_transpose(dl, shape):
    """One material class (1/S the same in every cell): the device forms only
    the D+ stencil Grams and takes D- = -(D+)^T + the boundary rows
    (stencil.cu minus_from_plus); every stencil Gram must still equal the
    oracle's X^T D_s S^-1 Y (T1), on grids with 3- and 4-cell axes, 2-D and 1-D."""
    from oracle import dlra_np
    from paper_2508_04484_b200.angular import PNOperators

    ops = PNOperators.build(3)
    nx, ny, nz = shape
    n = nx * ny * nz
    rng = np.random.default_rng(n)
    grid = dlra_np.Grid(nx, ny, nz, 0.1, 0.12, 0.09)
    inv_s = np.full(n, 1.0 / 7.3)
    ctx = dl.StreamingContext(inv_s, SimpleNamespace(grid=SimpleNamespace(
        nx=nx, ny=ny, nz=nz, dx=0.1, dy=0.12, dz=0.09)), ops)
    for a, b in ((5, 7), (12, 20)):
        x = rng.standard_normal((n, a))
        y = rng.standard_normal((n, b))
        got = ctx.stencil_grams(x, y)
        for i, (axis, sign) in enumerate(grid.stencils()):
            ref = x.T @ dlra_np.stencil(grid, axis, sign, inv_s[:, None] * y)
            assert relmax(got[i], ref) < 1e-12, (i, relmax(got[i], ref))
