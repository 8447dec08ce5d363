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
