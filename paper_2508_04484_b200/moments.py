"""Device drop-in for pndose.driver.MomentTables (driver.py:269-307).

The per-element angular moments of the screened elastic-scattering kernel on
the run's energy grid -- 12 elements x n_points energies x (max_degree + 1)
Legendre moments plus xi1, each a de-peaked Gauss-Legendre quadrature with a
doubled-node convergence check (physics/moliere.py:111-147) -- evaluated on
the GPU, one CTA per (element, energy) (csrc/moments.cu, pnd_moment_tables).
The Gauss-Legendre nodes are numpy's leggauss, as the reference's. Same
constructor, attributes (energies, max_degree, g, xi1) and interpolation
methods as the reference class; `driver.run_simulation` puts it in place of
the reference's during problem assembly.
"""

import numpy as np

from . import _lib
from .dlra import _generic_handle

# (Z, A) of the 12 base elements, in the reference's canonical order
# (constants.py:42-54: H C N O Na Mg P S Cl Ar K Ca)
ELEMENT_ZA = ((1, 1), (6, 12), (7, 14), (8, 16), (11, 23), (12, 24), (15, 31), (16, 32),
              (17, 35), (18, 40), (19, 39), (20, 40))


def device_moments(energies, max_degree, n_nodes=256, exponent=1.0, rtol=1e-9):
    """(g (12, n_e, max_degree + 1), xi1 (12, n_e)) per atom [cm^2]."""
    e = _lib.f64(np.atleast_1d(energies))
    x1, w1 = np.polynomial.legendre.leggauss(n_nodes)
    x2, w2 = np.polynomial.legendre.leggauss(2 * n_nodes)
    z = np.array([za[0] for za in ELEMENT_ZA], dtype=np.int32)
    a = np.array([za[1] for za in ELEMENT_ZA], dtype=np.int32)
    g = np.empty((len(ELEMENT_ZA), e.size, max_degree + 1))
    xi1 = np.empty((len(ELEMENT_ZA), e.size))
    _generic_handle().call("pnd_moment_tables", e.size, _lib.ptr(e), len(ELEMENT_ZA),
                           _lib.ptr(z), _lib.ptr(a), int(n_nodes), _lib.ptr(_lib.f64(x1)),
                           _lib.ptr(_lib.f64(w1)), _lib.ptr(_lib.f64(x2)), _lib.ptr(_lib.f64(w2)),
                           int(max_degree), float(exponent), float(rtol), _lib.ptr(g),
                           _lib.ptr(xi1))
    return g, xi1


class MomentTables:
    """Per-element angular moments and xi1 on an energy grid (driver.py:269-307)."""

    def __init__(self, e_min, e_max, max_degree, n_points=48, n_nodes=256, exponent=1.0):
        self.energies = np.linspace(0.98 * e_min, 1.02 * e_max, n_points)
        self.max_degree = max_degree
        self.g, self.xi1 = device_moments(self.energies, max_degree, n_nodes, exponent)

    def _interp(self, table, e):
        e = np.asarray(e, dtype=float)
        idx = np.clip(np.searchsorted(self.energies, e) - 1, 0, len(self.energies) - 2)
        w = (e - self.energies[idx]) / (self.energies[idx + 1] - self.energies[idx])
        return (1.0 - w) * table[:, idx] + w * table[:, idx + 1]

    def moments_at(self, e):
        """(12, ..., max_degree+1) per-atom moments at energies e."""
        return np.moveaxis(
            np.stack([self._interp(self.g[..., d], e) for d in range(self.max_degree + 1)]),
            0, -1)

    def xi1_at(self, e):
        return self._interp(self.xi1, e)
