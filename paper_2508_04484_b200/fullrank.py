"""Full-rank oracle on the device: the drop-in for pndose.fullrank (fullrank.py:16-45).

The dense n x m moment matrix is evolved with the same Lie splitting as the
reference oracle -- RK4 on u' = F_S(u) and implicit Euler on the
per-(cell, moment) self-scattering with an explicit Euler source -- by
csrc/fullrank.cu (the K-stage kernel over 32-column blocks of u, one
elementwise scattering kernel). Same signatures, contexts and errors as the
reference ("amplified" NumericalError when a streaming step grows the
solution by more than 1e6).
"""

import numpy as np

from . import _lib
from .dlra import ScatteringContext, StreamingContext, handle_for


def fullrank_streaming_step(u: np.ndarray, dt: float, ctx: StreamingContext) -> np.ndarray:
    """One RK4 step of u' = F_S(u) on the dense moment matrix (fullrank.py:16-27)."""
    h = ctx.handle()
    u = _lib.f64(u)
    h.call("pnd_fullrank_set", _lib.ptr(u))
    h.call("pnd_fullrank_streaming_step", float(dt))
    out = np.empty_like(u)
    h.call("pnd_fullrank_get", _lib.ptr(out))
    return out


def fullrank_scattering_step(u: np.ndarray, dt: float, ctx: ScatteringContext) -> np.ndarray:
    """Implicit Euler self-scattering, then the explicit source (fullrank.py:30-45)."""
    u = _lib.f64(u)
    n, m = u.shape
    h = handle_for((n, 1, 1), (1.0, 1.0, 1.0), m)
    ctx.upload(h)
    h.call("pnd_fullrank_set", _lib.ptr(u))
    h.call("pnd_fullrank_scattering_step", float(dt))
    out = np.empty_like(u)
    h.call("pnd_fullrank_get", _lib.ptr(out))
    return out
