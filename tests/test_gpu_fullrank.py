"""GPU parity of the device full-rank oracle (csrc/fullrank.cu).

- fullrank_streaming_step / fullrank_scattering_step (fullrank.py:16-45)
  against the reference's own results on the steps fixtures (full_matrix,
  written by tools/make_golden.py from pndose.fullrank);
- more than one 32-column block (m = 40 and 49: a partial last block)
  against the numpy oracle (oracle/dlra_np.py, pinned by test_oracle.py);
- the "amplified" NumericalError of an unstable streaming step;
- a whole device full-rank run (driver.run_bundle(solver="fullrank"))
  against the oracle's full-rank loop on the lockstep bundle;
- T3 on the device at a size beyond the CPU lockstep test: the DLRA at
  maximal rank r = m against the device full-rank, step by step.
"""

from types import SimpleNamespace

import numpy as np
import pytest

from conftest import GOLDEN, golden

pytestmark = pytest.mark.gpu


def rel(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / nb)


def grid_ns(arr):
    nx, ny, nz = (int(v) for v in arr[:3])
    return SimpleNamespace(nx=nx, ny=ny, nz=nz, dx=float(arr[3]), dy=float(arr[4]),
                           dz=float(arr[5]))


@pytest.fixture(scope="module")
def steps_npz():
    return golden("steps.npz")


@pytest.mark.parametrize("case", ["str3d", "str2d", "strz"])
def test_fullrank_streaming_vs_reference(steps_npz, case):
    from paper_2508_04484_b200 import dlra, fullrank

    S, p = steps_npz, case + "_"
    ops = SimpleNamespace(eig_v=list(S[p + "eig_v"]), lam_plus=list(S[p + "lam_plus"]),
                          lam_minus=list(S[p + "lam_minus"]))
    ctx = dlra.StreamingContext(S[p + "inv_s"], SimpleNamespace(grid=grid_ns(S[p + "grid"])), ops)
    u = S[p + "u0"] @ S[p + "s0"] @ S[p + "v0"].T
    out = fullrank.fullrank_streaming_step(u, float(S[p + "dt"]), ctx)
    assert rel(out, S[p + "full_matrix"]) < 1e-12


@pytest.mark.parametrize("case", ["scat_h", "scat_x", "scat_max"])
def test_fullrank_scattering_vs_reference(steps_npz, case):
    from paper_2508_04484_b200 import dlra, fullrank

    S, p = steps_npz, case + "_"
    ctx = dlra.ScatteringContext(S[p + "weights"], S[p + "inv_s"], S[p + "g_diags"],
                                 S[p + "sigma_t"], list(zip(S[p + "psi"], S[p + "tm"])))
    u = S[p + "u0"] @ S[p + "s0"] @ S[p + "v0"].T
    out = fullrank.fullrank_scattering_step(u, float(S[p + "dt"]), ctx)
    assert rel(out, S[p + "full_matrix"]) < 1e-13


def random_ops(m, rng):
    vs, lp, lm = [], [], []
    for _ in range(3):
        v, _ = np.linalg.qr(rng.standard_normal((m, m)))
        lam = rng.uniform(-1.0, 1.0, m)
        vs.append(v)
        lp.append(np.maximum(lam, 0.0))
        lm.append(np.minimum(lam, 0.0))
    return vs, lp, lm


@pytest.mark.parametrize("m,shape", [(40, (5, 4, 6)), (49, (3, 5, 4))])
def test_fullrank_streaming_blocks_vs_oracle(m, shape):
    from oracle import dlra_np
    from paper_2508_04484_b200 import dlra, fullrank

    rng = np.random.default_rng(m)
    vs, lp, lm = random_ops(m, rng)
    h = (0.3, 0.25, 0.2)
    grid = dlra_np.Grid(*shape, *h)
    n = grid.n
    inv_s = rng.uniform(0.05, 0.2, n)
    u = rng.standard_normal((n, m))
    dt = 0.02
    want = dlra_np.fullrank_streaming_step(u, dt, inv_s, grid, dlra_np.Ops(vs, lp, lm))
    g = SimpleNamespace(nx=shape[0], ny=shape[1], nz=shape[2], dx=h[0], dy=h[1], dz=h[2])
    ctx = dlra.StreamingContext(inv_s, SimpleNamespace(grid=g),
                                SimpleNamespace(eig_v=vs, lam_plus=lp, lam_minus=lm))
    got = fullrank.fullrank_streaming_step(u, dt, ctx)
    assert rel(got, want) < 1e-12


def test_fullrank_amplification_error(steps_npz):
    from paper_2508_04484_b200 import dlra, fullrank
    from paper_2508_04484_b200.errors import NumericalError

    S, p = steps_npz, "str3d_"
    ops = SimpleNamespace(eig_v=list(S[p + "eig_v"]), lam_plus=list(S[p + "lam_plus"]),
                          lam_minus=list(S[p + "lam_minus"]))
    ctx = dlra.StreamingContext(S[p + "inv_s"] * 1e4,
                                SimpleNamespace(grid=grid_ns(S[p + "grid"])), ops)
    u = S[p + "u0"] @ S[p + "s0"] @ S[p + "v0"].T
    with pytest.raises(NumericalError, match="amplified"):
        fullrank.fullrank_streaming_step(u, 50.0, ctx)


def test_fullrank_run_vs_oracle():
    """The device full-rank loop (what run_bundle(solver="fullrank") drives)
    against the oracle's full-rank loop: the collided deposit, compared before
    the (much larger) uncollided dose is added."""
    from oracle import dlra_np
    from paper_2508_04484_b200.driver import DeviceSolver, run_bundle
    from paper_2508_04484_b200.problem import ProblemBundle

    b = ProblemBundle.load(GOLDEN / "bundle_lockstep.npz")
    steps = 120
    dev = DeviceSolver(b)
    dev.h.call("pnd_fullrank_reset")
    edges = b.pseudo_time_edges()
    for k in range(steps):
        dev.set_coefficients(edges[k], edges[k + 1])
        dev.h.call("pnd_fullrank_step", float(edges[k] - edges[k + 1]), 0)
    got = dev.dose()
    dev.close()
    want = dlra_np.run_energy_loop(b, solver="fullrank", max_steps=steps)
    assert rel(got, want["deposited"]) < 1e-10
    res = run_bundle(b, max_steps=4, solver="fullrank")
    assert res.rank_history[-1][2] == min(b.n_cells, b.n_moments)
    assert res.diagnostics["solver"] == "fullrank-b200"


def test_maximal_rank_dlra_vs_device_fullrank():
    """T3 (acceptance criterion 2) entirely on the device, on a grid 8x the
    CPU lockstep test's: DLRA at r = m vs the full-rank solve, <= 1e-8."""
    from paper_2508_04484_b200.driver import DeviceSolver
    from paper_2508_04484_b200.problem import ProblemBundle

    b = ProblemBundle.load(GOLDEN / "bundle_lockstep.npz")
    big = enlarge(b, 2)
    m = big.n_moments
    low = DeviceSolver(big)
    low.init_state(rank=m)
    full = DeviceSolver(big)
    full.h.call("pnd_fullrank_reset")
    edges = big.pseudo_time_edges()
    worst = 0.0
    u = np.empty((big.n_cells, m))
    from paper_2508_04484_b200 import _lib

    for k in range(min(160, len(edges) - 1)):
        dt = edges[k] - edges[k + 1]
        for s in (low, full):
            s.set_coefficients(edges[k], edges[k + 1])
        low.step(dt, want_defect=False)
        full.h.call("pnd_fullrank_step", float(dt), 0)
        if k % 20 == 19:
            uu, ss, vv = low.state()
            full.h.call("pnd_fullrank_get", _lib.ptr(u))
            nrm = np.linalg.norm(u)
            if nrm > 0:
                worst = max(worst, np.linalg.norm(uu @ ss @ vv.T - u) / nrm)
    low.close()
    full.close()
    assert worst <= 1e-8, worst


def enlarge(b, f):
    """The lockstep bundle on an f-times finer-in-count grid: the same cell
    size, f x the cells per axis, every cell of a block copying its parent's
    material and uncollided flux (a valid problem of the same physics)."""
    import dataclasses

    nx, ny, nz = b.shape
    idx = np.arange(nx * ny * nz).reshape(nz, ny, nx)
    rep = idx.repeat(f, 0).repeat(f, 1).repeat(f, 2).ravel()
    fluxes = [dataclasses.replace(fl, values=fl.values[rep], residual=fl.residual[rep])
              for fl in b.fluxes]
    return dataclasses.replace(b, shape=(nx * f, ny * f, nz * f), cell_class=b.cell_class[rep],
                               fluxes=fluxes, _log_tables=None)
