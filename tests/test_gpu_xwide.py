"""Ranks above 64 (csrc/xwide.cu: column-blocked n-side storage) against the
numpy oracle (pinned to the reference by tests/test_oracle.py), T2
tolerances: streaming and scattering steps + truncation at r = 72 ... 200,
the narrow <-> blocked layout changes when the rank crosses 64, and a short
fixed-rank energy loop at r = 100 (SURVEY.md §8(d) configs 2 and 5 need
rank_max up to 200; the reference's default is 100, driver.py:79-81).
"""

from types import SimpleNamespace

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.fixture(scope="module")
def dl():
    from paper_2508_04484_b200 import dlra

    return dlra


def _ops(n_max):
    from paper_2508_04484_b200.angular import PNOperators

    return PNOperators.build(n_max)


@pytest.mark.parametrize("r,n_max", [(72, 11), (100, 14), (130, 17), (200, 19)])
def test_streaming_step_blocked_vs_oracle(dl, r, n_max):
    from oracle import dlra_np

    ops = _ops(n_max)
    nx, ny, nz = 9, 8, 7 if r < 200 else 9
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
    assert aug.orthonormality_defect() < 1e-12
    assert rel(aug.matrix(), ou @ os_ @ ov.T) < 1e-11
    tr, tail = dl.truncate(aug, dl.TruncationPolicy(1e300, r, r))
    _, ts, _, ttail = dlra_np.truncate(ou, os_, ov, 1e300, r, r)
    np.testing.assert_allclose(np.diag(tr.s), np.diag(ts), rtol=1e-9)
    assert tr.orthonormality_defect() < 1e-12


@pytest.mark.parametrize("r,hetero", [(80, False), (100, True)])
def test_scattering_step_blocked_vs_oracle(dl, r, hetero):
    from oracle import dlra_np

    rng = np.random.default_rng(r + 7)
    n, m = 900, 196
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


def test_rank_crossing_64_both_ways(dl):
    """Truncation of a row-major augmented state (<= 64 + 64 columns) to rank
    90 goes to the blocked layout; a later truncation to 40 comes back."""
    rng = np.random.default_rng(3)
    n, m = 700, 150
    u = np.linalg.qr(rng.standard_normal((n, 120)))[0]
    v = np.linalg.qr(rng.standard_normal((m, 120)))[0]
    s = np.diag(np.logspace(0, -6, 120)) + 1e-8 * rng.standard_normal((120, 120))
    st = dl.LowRankState(u, s, v)
    t90, _ = dl.truncate(st, dl.TruncationPolicy(1e300, 90, 90))
    p, sig, qt = np.linalg.svd(s)
    want = (u @ p[:, :90]) @ np.diag(sig[:90]) @ (v @ qt[:90].T).T
    assert rel(t90.matrix(), want) < 1e-12
    assert t90.orthonormality_defect() < 1e-13
    t40, _ = dl.truncate(t90, dl.TruncationPolicy(1e300, 40, 40))
    want40 = (u @ p[:, :40]) @ np.diag(sig[:40]) @ (v @ qt[:40].T).T
    assert rel(t40.matrix(), want40) < 1e-11


def test_fixed_rank_100_loop_vs_oracle():
    """Three energy steps at fixed rank 100 through the device loop (state,
    coefficients and dose on the GPU) against the oracle's loop, from the same
    rank-100 state: U S V^T and the dose."""
    from oracle import dlra_np
    from paper_2508_04484_b200.driver import DeviceSolver
    from paper_2508_04484_b200.problem import ProblemBundle

    b = ProblemBundle.load(GOLDEN / "bundle_fp19.npz")
    b.rank_min = b.rank_max = 100
    b.truncation_tolerance = 1e300
    n, m = b.n_cells, b.n_moments
    rng = np.random.default_rng(100)
    u = np.linalg.qr(rng.standard_normal((n, 100)))[0]
    v = np.linalg.qr(rng.standard_normal((m, 100)))[0]
    s = np.diag(np.logspace(-3, -9, 100))
    edges = b.pseudo_time_edges()
    k0 = 20
    dev = DeviceSolver(b)
    dev.h.set_state(u, s, v)
    for k in range(k0, k0 + 3):
        dev.set_coefficients(edges[k], edges[k + 1])
        out = dev.step(edges[k] - edges[k + 1])
        assert int(out[2]) == 100
    uu, ss, vv = dev.state()
    dose = dev.dose()
    dev.close()
    ref = dlra_np.run_energy_loop(b, max_steps=3, start_step=k0, state=(u, s, v))
    ou, os_, ov = ref["state"]
    assert rel(uu @ ss @ vv.T, ou @ os_ @ ov.T) < 1e-9
    assert rel(dose, ref["deposited"]) < 1e-9
