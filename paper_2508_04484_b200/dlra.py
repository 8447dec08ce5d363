"""Drop-in mirror of pndose.dlra (pkg/src/pndose/dlra.py) on the B200.

Same names, argument meanings and exceptions as the reference:
`LowRankState`, `TruncationPolicy`, `truncate`, `orthonormal_columns`,
`StreamingContext`, `streaming_step`, `ScatteringContext`, `scattering_step`.
Every numerical step runs in libpndose_b200.so (include/pndose_b200.h): the
factors are uploaded, the substep runs on the device, the (augmented) factors
come back. The device-resident energy loop that keeps the state on the GPU
across steps is paper_2508_04484_b200.driver.

Factor-level results are gauge-equivalent to the reference, not identical:
QR/SVD signs and rotations are not unique (BASELINE.json north_star), so the
contract is on U S V^T, singular values and ranks (tests/test_gpu_parity.py).
"""

from dataclasses import dataclass, field

import threading

import numpy as np

from . import _lib
from .errors import NumericalError

_HANDLES = {}


def _grid_of(stencils_or_grid):
    g = getattr(stencils_or_grid, "grid", stencils_or_grid)
    return (int(g.nx), int(g.ny), int(g.nz)), (float(g.dx), float(g.dy), float(g.dz))


def _a_split(ops):
    ap = np.stack([(v * lp) @ v.T for v, lp in zip(ops.eig_v, ops.lam_plus)])
    am = np.stack([(v * lm) @ v.T for v, lm in zip(ops.eig_v, ops.lam_minus)])
    return ap, am


def handle_for(shape, spacing, m):
    """Shared device handle per (grid, m, host thread) for the function-level
    API (a handle is stream-ordered state: one per thread, never shared)."""
    key = (tuple(shape), tuple(spacing), int(m), threading.get_ident())
    h = _HANDLES.get(key)
    if h is None:
        h = _lib.Handle(shape, spacing, m)
        _HANDLES[key] = h
    return h


def _generic_handle():
    return handle_for((1, 1, 1), (1.0, 1.0, 1.0), 1)


def orthonormal_columns(a: np.ndarray) -> np.ndarray:
    """Orthonormal basis of the columns of a (dlra.py:26-43), device TSQR.

    Householder-based like the reference's LAPACK QR, so rank-deficient input
    still returns min(rows, cols) orthonormal columns; a basis that fails the
    reference's defect bound raises NumericalError.
    """
    a = _lib.f64(a)
    rows, cols = a.shape
    k = min(rows, cols)
    q = np.empty((rows, k))
    r = np.empty((k, cols))
    _generic_handle().call("pnd_orthonormalize", _lib.ptr(a), rows, cols, _lib.ptr(q), _lib.ptr(r))
    defect = np.abs(q.T @ q - np.eye(k)).max()
    if defect > 1e-10:
        raise NumericalError(f"orthonormalization failed, defect {defect:.3e}")
    return q


@dataclass
class LowRankState:
    """Factored solution U S V^T (dlra.py:46-72)."""

    u: np.ndarray
    s: np.ndarray
    v: np.ndarray

    @classmethod
    def zero(cls, n: int, m: int, rank: int, seed: int = 20260809) -> "LowRankState":
        rng = np.random.default_rng(seed)
        u = orthonormal_columns(rng.standard_normal((n, rank)))
        v = orthonormal_columns(rng.standard_normal((m, rank)))
        return cls(u=u, s=np.zeros((rank, rank)), v=v)

    @property
    def rank(self) -> int:
        return min(self.s.shape)

    def matrix(self) -> np.ndarray:
        return self.u @ self.s @ self.v.T

    def orthonormality_defect(self) -> float:
        du = np.abs(self.u.T @ self.u - np.eye(self.u.shape[1])).max()
        dv = np.abs(self.v.T @ self.v - np.eye(self.v.shape[1])).max()
        return max(du, dv)


@dataclass(frozen=True)
class TruncationPolicy:
    """Tail-sum truncation threshold (dlra.py:75-87)."""

    threshold: float
    rank_min: int = 2
    rank_max: int = 100

    def __post_init__(self):
        if self.threshold < 0.0:
            raise ValueError("truncation threshold must be nonnegative")
        if not 1 <= self.rank_min <= self.rank_max:
            raise ValueError("need 1 <= rank_min <= rank_max")


def truncate(state: LowRankState, policy: TruncationPolicy):
    """Tail-rule truncation (dlra.py:90-115) on the device: Jacobi SVD of S,
    rank rule, U1 = U P, V1 = V Q. Returns (state, tail)."""
    n, m = state.u.shape[0], state.v.shape[0]
    h = handle_for((n, 1, 1), (1.0, 1.0, 1.0), m)
    h.set_state(state.u, state.s, state.v)
    tail = np.zeros(1)
    rank = np.zeros(1, dtype=np.int32)
    h.call("pnd_truncate", float(policy.threshold), int(policy.rank_min), int(policy.rank_max),
           _lib.ptr(tail), _lib.ptr(rank))
    u, s, v = h.get_state()
    return LowRankState(u=u, s=s, v=v), float(tail[0])


@dataclass
class StreamingContext:
    """Frozen per-step streaming coefficients (dlra.py:126-210).

    `stencils` is anything with a `.grid` (Grid3D-like) -- the reference's
    UpwindStencils or paper_2508_04484_b200.spatial.UpwindStencils -- and
    `ops` anything with eig_v / lam_plus / lam_minus (PNOperators). The
    upwind stencils are applied matrix-free on the device; nothing n x n is
    ever built (the reference rebuilds 2A scaled CSR matrices per step,
    dlra.py:140-145).
    """

    inv_s: np.ndarray
    stencils: object
    ops: object

    def __post_init__(self):
        shape, spacing = _grid_of(self.stencils)
        self._shape, self._spacing = shape, spacing
        self.active_axes = tuple(a for a in range(3) if shape[a] > 1)

    @property
    def m(self):
        return int(np.asarray(self.ops.eig_v[0]).shape[0])

    def handle(self):
        h = handle_for(self._shape, self._spacing, self.m)
        if h.uploaded.get("angular") is not self.ops:
            h.set_angular(*_a_split(self.ops))
            h.uploaded["angular"] = self.ops
        h.set_inv_s(self.inv_s)
        return h

    def full_rhs(self, u: np.ndarray) -> np.ndarray:
        """F_S(u) (spatial.apply_streaming) on the device."""
        u = _lib.f64(u)
        out = np.empty_like(u)
        self.handle().call("pnd_apply_streaming", _lib.ptr(u), _lib.ptr(out))
        return out

    def _moment_factors(self, w: np.ndarray):
        """[(W^T V L+ V^T W, W^T V L- V^T W)] per active axis (dlra.py:155-166)."""
        out = []
        for axis in self.active_axes:
            c = w.T @ self.ops.eig_v[axis]
            out.append(((c * self.ops.lam_plus[axis]) @ c.T, (c * self.ops.lam_minus[axis]) @ c.T))
        return out

    def k_rhs(self, k: np.ndarray, factors) -> np.ndarray:
        """-sum_s (D_s S^-1 K) F_s (dlra.py:168-174), fused stencil+contraction kernel."""
        k = _lib.f64(k)
        f = _lib.f64(np.array([fs for pair in factors for fs in pair]))
        out = np.empty_like(k)
        self.handle().call("pnd_k_rhs", _lib.ptr(k), int(k.shape[1]), _lib.ptr(f), _lib.ptr(out))
        return out

    def stencil_grams(self, x: np.ndarray, y: np.ndarray) -> np.ndarray:
        """[X^T D_s S^-1 Y] for every stencil (ns x a x b), DMMA Gram kernel."""
        x, y = _lib.f64(x), _lib.f64(y)
        ns = 2 * len(self.active_axes)
        out = np.empty((ns, x.shape[1], y.shape[1]))
        self.handle().call("pnd_stencil_grams", _lib.ptr(x), int(x.shape[1]), _lib.ptr(y),
                           int(y.shape[1]), _lib.ptr(out))
        return out

    def l_step_factors(self, u0: np.ndarray):
        """Per axis (A+, A-, (Ds+ U0)^T U0, (Ds- U0)^T U0) (dlra.py:176-186)."""
        qt = self.stencil_grams(u0, u0)
        ap, am = _a_split(self.ops)
        return [(ap[a], am[a], qt[2 * i].T, qt[2 * i + 1].T) for i, a in enumerate(self.active_axes)]

    def l_rhs(self, l: np.ndarray, factors) -> np.ndarray:
        """-sum A (L Q) (dlra.py:188-194); m-side only."""
        out = np.zeros_like(l)
        for a_plus, a_minus, q_plus, q_minus in factors:
            out -= a_plus @ (l @ q_plus)
            out -= a_minus @ (l @ q_minus)
        return out

    def s_step_factors(self, u_hat: np.ndarray, v_hat: np.ndarray):
        """Precontracted (U^T Ds U^ Grams, moment factors): the device form of
        dlra.py:196-202, which materialises n x R arrays instead."""
        return self.stencil_grams(u_hat, u_hat), self._moment_factors(v_hat)

    def s_rhs(self, s: np.ndarray, u_hat: np.ndarray, factors) -> np.ndarray:
        """-sum_s G_s S F_s (dlra.py:204-210) from the precontracted Grams."""
        grams, moment = factors
        out = np.zeros_like(s)
        for i, (f_plus, f_minus) in enumerate(moment):
            out -= grams[2 * i] @ s @ f_plus
            out -= grams[2 * i + 1] @ s @ f_minus
        return out


def streaming_step(state: LowRankState, dt: float, ctx: StreamingContext) -> LowRankState:
    """Augmented BUG step for u' = F_S(u) (dlra.py:213-225) on the device."""
    h = ctx.handle()
    h.set_state(state.u, state.s, state.v)
    h.call("pnd_streaming_step", float(dt))
    u, s, v = h.get_state()
    return LowRankState(u=u, s=s, v=v)


@dataclass
class ScatteringContext:
    """Frozen per-step scattering coefficients (dlra.py:228-267)."""

    element_weights: np.ndarray
    inv_s: np.ndarray
    g_diags: np.ndarray
    sigma_t: np.ndarray
    sources: list = field(default_factory=list)

    def classes(self):
        """Unique weight rows -> (cell_class, class_atomic)."""
        w = np.ascontiguousarray(self.element_weights, dtype=np.float64)
        uniq, inv = np.unique(w, axis=0, return_inverse=True)
        return np.asarray(inv).ravel().astype(np.int32), uniq

    def upload(self, h):
        cls, atomic = self.classes()
        h.set_materials(cls, atomic)
        h.set_inv_s(self.inv_s)
        h.set_scattering(self.g_diags, self.sigma_t)
        if self.sources:
            psi = np.array([np.asarray(p, dtype=float) for p, _ in self.sources])
            tm = np.array([np.asarray(t, dtype=float) for _, t in self.sources])
            h.set_sources(psi, tm)
        else:
            h.set_sources(np.zeros((0, h.n)), np.zeros((0, h.m)))


def scattering_step(state: LowRankState, dt: float, ctx: ScatteringContext) -> LowRankState:
    """Four-substep scattering update (dlra.py:270-322) on the device."""
    n, m = state.u.shape[0], state.v.shape[0]
    h = handle_for((n, 1, 1), (1.0, 1.0, 1.0), m)
    ctx.upload(h)
    h.set_state(state.u, state.s, state.v)
    h.call("pnd_scattering_step", float(dt))
    u, s, v = h.get_state()
    return LowRankState(u=u, s=s, v=v)
