"""m-side operator assembly on the GPU.

PNOperators.build(N, device=...) forms the three P_N flux matrices by the same
exact product quadrature as the host path (angular.py; the host path is pinned
to the reference's angular.py:101-202 by tests/test_oracle.py::test_angular_operators_match_reference) with cuBLAS, and
splits them with cuSOLVER eigendecompositions. Eigenvectors are not unique
(degenerate eigenvalues), so the comparison is on what the solver consumes:
A_d^+- = V diag(lambda^+-) V^T and the spectral radius (the CFL step).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n_max", [1, 7, 19])
def test_device_flux_operators_match_host(n_max):
    from paper_2508_04484_b200.angular import PNOperators

    host = PNOperators.build(n_max)
    dev = PNOperators.build(n_max, device="cuda:0")
    assert abs(dev.spectral_radius - host.spectral_radius) <= 1e-13 * host.spectral_radius
    hp, hm = host.a_split()
    dp, dm = dev.a_split()
    scale = max(np.abs(hp).max(), np.abs(hm).max())
    assert np.abs(dp - hp).max() <= 1e-12 * scale
    assert np.abs(dm - hm).max() <= 1e-12 * scale
    for v in dev.eig_v:
        assert np.abs(v.T @ v - np.eye(v.shape[0])).max() < 1e-12
