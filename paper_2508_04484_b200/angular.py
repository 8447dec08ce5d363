"""Real spherical-harmonic P_N flux operators, host side (m-side setup).

The streaming operator needs A_d^+- = V_d diag(lambda^+-) V_d^T for the three
flux matrices A_d = Int m(Omega) m(Omega)^T Omega_d dOmega
(pkg/src/pndose/angular.py:101-202). The reference assembles them in closed
form from complex ladder identities; here they are integrated exactly with a
product quadrature -- Gauss-Legendre in mu, a uniform rule in phi -- which is
exact because every surviving integrand is a polynomial in mu times a
trigonometric polynomial in phi of degree <= 2N+1 (the same identity the
reference's own tests/oracles.py uses). The basis is the reference's: index
p = l^2 + l + k, real combinations of orthonormal harmonics with the
Condon-Shortley phase cancelled (angular.py:58-80), so V, T_M and the
degree-diagonal scattering matrices line up with it. tests/test_oracle.py::test_angular_operators_match_reference pins
A_d^+- against the reference for N = 1..7.
"""

import math
from dataclasses import dataclass

import numpy as np


def _legendre_normalised(n_max, mu):
    """bar P_l^k(mu) for 0 <= k <= l <= n_max without the Condon-Shortley phase,
    normalised so sqrt(2)*bar P_l^k cos(k phi) is orthonormal on the sphere
    (k > 0) and bar P_l^0 likewise. Returns array (n_max+1, n_max+1, len(mu))."""
    mu = np.asarray(mu, dtype=float)
    s = np.sqrt(np.maximum(0.0, 1.0 - mu * mu))
    p = np.zeros((n_max + 1, n_max + 1, mu.size))
    p[0, 0] = math.sqrt(1.0 / (4.0 * math.pi))
    for k in range(1, n_max + 1):
        p[k, k] = math.sqrt((2.0 * k + 1.0) / (2.0 * k)) * s * p[k - 1, k - 1]
    for k in range(0, n_max):
        p[k + 1, k] = math.sqrt(2.0 * k + 3.0) * mu * p[k, k]
    for k in range(0, n_max + 1):
        for ell in range(k + 2, n_max + 1):
            a = math.sqrt((4.0 * ell * ell - 1.0) / (ell * ell - k * k))
            b = math.sqrt(((ell - 1.0) ** 2 - k * k) / (4.0 * (ell - 1.0) ** 2 - 1.0))
            p[ell, k] = a * (mu * p[ell - 1, k] - b * p[ell - 2, k])
    return p


def real_basis(n_max, mu, phi):
    """m(Omega) for arrays of (mu, phi): shape ((N+1)^2, len(mu))."""
    p = _legendre_normalised(n_max, mu)
    out = np.zeros(((n_max + 1) ** 2, np.size(mu)))
    r2 = math.sqrt(2.0)
    for ell in range(n_max + 1):
        base = ell * ell + ell
        out[base] = p[ell, 0]
        for k in range(1, ell + 1):
            out[base + k] = r2 * p[ell, k] * np.cos(k * phi)
            out[base - k] = r2 * p[ell, k] * np.sin(k * phi)
    return out


def beam_projection(n_max, omega):
    """T_M = m(Omega_in) (angular.py:251-253)."""
    omega = np.asarray(omega, dtype=float)
    omega = omega / np.linalg.norm(omega)
    mu = np.array([omega[2]])
    phi = np.array([math.atan2(omega[1], omega[0])])
    return real_basis(n_max, mu, phi)[:, 0]


def _quadrature(n_max):
    nq = n_max + 2
    x, w = np.polynomial.legendre.leggauss(nq)
    nphi = 2 * n_max + 4
    phi = 2.0 * math.pi * np.arange(nphi) / nphi
    mu = np.repeat(x, nphi)
    ph = np.tile(phi, nq)
    wt = np.repeat(w, nphi) * (2.0 * math.pi / nphi)
    basis = real_basis(n_max, mu, ph)
    s = np.sqrt(1.0 - mu * mu)
    comps = (s * np.cos(ph), s * np.sin(ph), mu)
    return basis, wt, comps


def flux_matrices(n_max):
    """(A_x, A_y, A_z) by exact product quadrature."""
    basis, wt, comps = _quadrature(n_max)
    out = []
    for c in comps:
        a = (basis * (wt * c)) @ basis.T
        a = 0.5 * (a + a.T)
        a[np.abs(a) < 1e-15] = 0.0
        out.append(a)
    return tuple(out)


def _eig_jacobi(a):
    """Symmetric eigen-decomposition by the device's one-sided Jacobi SVD
    (pnd_svd_small): A + c I with c = |A|_1 + 1 is SPD, so its singular vectors
    are A's eigenvectors and sigma - c its eigenvalues (absolute error ~ eps c,
    as a dense symmetric eigensolver's)."""
    from . import _lib
    from .dlra import _generic_handle

    m = a.shape[0]
    c = float(np.abs(a).sum(axis=0).max()) + 1.0
    s = _lib.f64(a + c * np.eye(m))
    p, sig, qt = np.empty((m, m)), np.empty(m), np.empty((m, m))
    _generic_handle().call("pnd_svd_small", _lib.ptr(s), m, m, _lib.ptr(p), _lib.ptr(sig),
                           _lib.ptr(qt))
    return sig - c, p


@dataclass(frozen=True)
class PNOperators:
    """eig_v / lam_plus / lam_minus per axis, as the reference's PNOperators."""

    n_max: int
    eig_v: tuple
    lam_plus: tuple
    lam_minus: tuple

    @classmethod
    def build(cls, n_max: int, device=None) -> "PNOperators":
        """device (e.g. "cuda:0"): the three quadrature Grams on the GPU (cuBLAS
        DGEMM via torch) and their eigendecompositions by the library's own
        one-CTA Jacobi kernel (m <= 512: the SPD shift A + c I, c >= rho(A),
        has the eigenvectors of A and sigma = lambda + c; cuSOLVER syevd above
        that); SURVEY.md §8(f) row 4 -- the O(m^3) setup that takes seconds on
        the host at N >= 39."""
        if device is not None:
            return cls._build_device(n_max, device)
        vs, lp, lm = [], [], []
        for a in flux_matrices(n_max):
            lam, v = np.linalg.eigh(a)
            vs.append(v)
            lp.append(np.maximum(lam, 0.0))
            lm.append(np.minimum(lam, 0.0))
        return cls(n_max, tuple(vs), tuple(lp), tuple(lm))

    @classmethod
    def _build_device(cls, n_max, device):
        import torch

        basis, wt, comps = _quadrature(n_max)
        bd = torch.from_numpy(basis).to(device)
        vs, lp, lm = [], [], []
        m = basis.shape[0]
        for c in comps:
            a = (bd * torch.from_numpy(wt * c).to(device)) @ bd.T
            a = 0.5 * (a + a.T)
            a = torch.where(a.abs() < 1e-15, torch.zeros_like(a), a)
            if m <= 512:
                lam, v = _eig_jacobi(a.cpu().numpy())
            else:
                lam_t, v_t = torch.linalg.eigh(a)
                lam, v = lam_t.cpu().numpy(), v_t.cpu().numpy()
            vs.append(v)
            lp.append(np.maximum(lam, 0.0))
            lm.append(np.minimum(lam, 0.0))
            del a
        return cls(n_max, tuple(vs), tuple(lp), tuple(lm))

    @property
    def size(self):
        return (self.n_max + 1) ** 2

    @property
    def spectral_radius(self) -> float:
        return float(max(max(p.max(initial=0.0), -q.min(initial=0.0))
                         for p, q in zip(self.lam_plus, self.lam_minus)))

    def a_split(self):
        ap = np.stack([(v * l) @ v.T for v, l in zip(self.eig_v, self.lam_plus)])
        am = np.stack([(v * l) @ v.T for v, l in zip(self.eig_v, self.lam_minus)])
        return ap, am
