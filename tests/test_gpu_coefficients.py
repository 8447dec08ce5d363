"""GPU parity of the per-step coefficient assembly (csrc/coeff.cu).

The device evaluates, from tables uploaded once, what driver.step_contexts
(driver.py:523-538) forms on the host every step: S(E) per material class
(stopping.py:48-56, 107-120), the scattering diagonals and total cross
sections (driver.py:337-362, Boltzmann and Fokker-Planck with their
corrections) and the uncollided slices (raytracer.py:440-449). The host
restatements in problem.py are pinned to the reference's contexts by
tests/test_oracle.py; here the device must agree with them to FP64 rounding
(log/exp and the interpolation order), at table nodes, between them, at the
group-grid edges and outside the tables.
"""

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def energies(b):
    f = b.fluxes[0] if b.fluxes else None
    es = [b.e_max, b.e_min, 0.5 * (b.e_min + b.e_max), 1.37 * b.e_min + 0.11,
          float(b.mom_e[len(b.mom_e) // 2]), float(np.exp(np.log(b.stop_e[0]).mean()))]
    if f is not None:
        c = f.centers
        es += [float(c[0]), float(c[-1]), float(c[len(c) // 3]), f.e_min, f.e_max,
               f.e_max + 0.5, max(f.e_min - 0.25, 0.5 * f.e_min)]
    return [e for e in es if e > 0.0]


@pytest.mark.parametrize("tag", ["config1", "fp", "hetero", "smoke"])
def test_device_coefficients_match_host(tag):
    from paper_2508_04484_b200 import _lib
    from paper_2508_04484_b200.driver import DeviceSolver
    from paper_2508_04484_b200.problem import ProblemBundle

    b = ProblemBundle.load(GOLDEN / f"bundle_{tag}.npz")
    dev = DeviceSolver(b, device_coefficients=True)
    n, m, nb = b.n_cells, b.n_moments, len(b.fluxes)
    cs, gd, sg = np.empty(b.n_classes), np.empty((12, m)), np.empty(12)
    psi, psi_lo = np.empty((max(nb, 1), n)), np.empty((max(nb, 1), n))
    es = energies(b)
    for e_mid, e_lo in zip(es, es[1:] + es[:1]):
        dev.h.call("pnd_coefficients_at", float(e_mid), float(e_lo), 1)
        dev.h.call("pnd_get_coefficients", _lib.ptr(cs), _lib.ptr(gd), _lib.ptr(sg),
                   _lib.ptr(psi), _lib.ptr(psi_lo))
        assert rel(cs, b.class_stopping(e_mid)) < 1e-13, e_mid
        g_ref, s_ref = b.scattering_tables(e_mid)
        assert rel(gd, g_ref) < 1e-13, e_mid
        assert np.abs(sg - s_ref).max() <= 1e-13 * max(np.abs(g_ref).max(), 1.0), e_mid
        if nb:
            want, want_lo = b.psi_at(e_mid), b.psi_at(e_lo)
            scale = max(np.abs(b.fluxes[0].values).max(), 1e-300)
            assert np.abs(psi[:nb] - want).max() <= 1e-14 * scale, e_mid
            assert np.abs(psi_lo[:nb] - want_lo).max() <= 1e-14 * scale, e_lo
    dev.close()


def test_device_coefficient_steps_match_host_steps():
    """Two runs of the same bundle, host-uploaded vs device-formed coefficients:
    the same dose to rounding (the step itself is unchanged)."""
    from paper_2508_04484_b200.driver import DeviceSolver
    from paper_2508_04484_b200.problem import ProblemBundle

    b = ProblemBundle.load(GOLDEN / "bundle_smoke.npz")
    edges = b.pseudo_time_edges()
    doses = []
    for on in (False, True):
        s = DeviceSolver(b, device_coefficients=on)
        s.init_state()
        for k in range(min(12, len(edges) - 1)):
            s.set_coefficients(edges[k], edges[k + 1])
            s.step(edges[k] - edges[k + 1])
        doses.append(s.dose())
        s.close()
    assert rel(doses[1], doses[0]) < 1e-11


def test_separable_flux_matches_dense_table():
    """pnd_set_flux_separable keeps lat(x, y) and depth(z, g) on the device and forms
    each step's slices from them (no n x G table); the slices are bit-identical to
    the lerp of the expanded table, for device- and host-selected groups."""
    from paper_2508_04484_b200 import _lib
    from paper_2508_04484_b200.driver import DeviceSolver
    from paper_2508_04484_b200.problem import ProblemBundle

    b = ProblemBundle.load(GOLDEN / "bundle_hetero.npz")
    nx, ny, nz = b.shape
    n, G, nb = b.n_cells, b.fluxes[0].n_groups, len(b.fluxes)
    rng = np.random.default_rng(11)
    lats = [rng.random(nx * ny) for _ in range(nb)]
    depths = [rng.random((nz, G)) * np.exp(-rng.random((nz, G)) * 30.0) for _ in range(nb)]
    vals = [np.ascontiguousarray((d[:, None, :] * lat[None, :, None]).reshape(n, G))
            for lat, d in zip(lats, depths)]
    devs = []
    for sep in (False, True):
        dev = DeviceSolver(b, device_coefficients=True)
        for i in range(nb):
            tm = _lib.f64(b.t_ms[i])
            if sep:
                dev.h.call("pnd_set_flux_separable", i, nb, G, _lib.ptr(lats[i]),
                           _lib.ptr(depths[i]), _lib.ptr(tm))
            else:
                dev.h.call("pnd_set_flux_table", i, nb, G, _lib.ptr(vals[i]), _lib.ptr(tm))
        dev.upload_coefficient_tables()
        devs.append(dev)
    es = energies(b)
    for e_mid, e_lo in zip(es, es[1:] + es[:1]):
        got = []
        for dev in devs:
            psi, psi_lo = np.empty((nb, n)), np.empty((nb, n))
            dev.h.call("pnd_coefficients_at", float(e_mid), float(e_lo), 1)
            dev.h.call("pnd_get_coefficients", None, None, None, _lib.ptr(psi), _lib.ptr(psi_lo))
            got.append((psi, psi_lo))
        np.testing.assert_array_equal(got[0][0], got[1][0])
        np.testing.assert_array_equal(got[0][1], got[1][1])
    for j0, w0, j1, w1 in [(3, 1.0, 4, 0.0), (3, 0.25, 4, 0.75), (G - 2, 0.5, G - 1, 0.5),
                           (0, 0.7, 1, 0.0)]:
        got = []
        for dev in devs:
            psi = np.empty((nb, n))
            dev.h.call("pnd_select_flux", 0, _lib.ptr(np.full(nb, j0, np.int32)),
                       _lib.ptr(np.full(nb, w0)), _lib.ptr(np.full(nb, j1, np.int32)),
                       _lib.ptr(np.full(nb, w1)))
            dev.h.call("pnd_get_coefficients", None, None, None, _lib.ptr(psi), None)
            got.append(psi)
        np.testing.assert_array_equal(got[0], got[1])
        for i in range(nb):
            v = vals[i]
            want = w0 * v[:, j0] + w1 * v[:, j1] if w1 != 0.0 else w0 * v[:, j0]
            np.testing.assert_allclose(got[1][i], want, rtol=1e-15, atol=0)
    for dev in devs:
        dev.close()


def test_device_moment_tables_match_reference():
    """MomentTables on the device (moments.cu; driver.py:269-307 via
    moliere.py:111-147) against the reference's own tables for 1..105 MeV up
    to degree 21 (tests/golden/bench_physics.npz, written by the reference)."""
    import numpy as np

    from conftest import golden
    from paper_2508_04484_b200.moments import MomentTables

    ph = golden("bench_physics.npz")
    t = MomentTables(1.0, 105.0, 21, n_points=48, n_nodes=256, exponent=1.0)
    np.testing.assert_array_equal(t.energies, ph["mom_e"])
    g, ref = t.g, ph["mom_g"]
    assert np.abs(g - ref).max() / np.abs(ref).max() < 1e-12
    for el in range(12):  # every element to its own scale
        assert np.abs(g[el] - ref[el]).max() <= 1e-12 * np.abs(ref[el]).max()
    assert np.abs(t.xi1 - ph["mom_xi1"]).max() <= 1e-12 * np.abs(ph["mom_xi1"]).max()


def test_device_moment_tables_report_non_convergence():
    import pytest

    from paper_2508_04484_b200.errors import NumericalError
    from paper_2508_04484_b200.moments import device_moments

    with pytest.raises(NumericalError, match="did not converge"):
        device_moments([50.0], 7, n_nodes=4, rtol=1e-12)
