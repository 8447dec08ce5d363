"""CPU oracle for the DLRA energy step -- TEST INFRASTRUCTURE ONLY.

A numpy restatement of the reference algorithm (pkg/src/pndose/dlra.py,
spatial.py, fullrank.py) used as the checker for the CUDA path. Only
tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import it; the product path never does.

Parity of this oracle is pinned against golden vectors written by the
reference itself (tests/golden/*.npz via tools/make_golden.py; checked in
tests/test_oracle.py).

The restatement is matrix-free: the upwind stencils (spatial.py:81-145) are
applied with array slicing on the (nz, ny, nx) cell cube instead of
Kronecker-assembled CSR matrices, and the Galerkin S-phase right-hand side
(dlra.py:196-210) is precontracted into per-stencil R x R Grams before the
RK4, which is algebraically the same map.
"""

import numpy as np


class Grid:
    """Structured grid with the flat index k*nx*ny + j*nx + i (spatial.py:62-63)."""

    def __init__(self, nx, ny, nz, dx, dy, dz):
        for n in (nx, ny, nz):
            if n == 2:
                raise ValueError("a used axis needs 1 (inactive) or >= 3 cells (3-point)")
        self.shape = (int(nx), int(ny), int(nz))
        self.h = (float(dx), float(dy), float(dz))

    @property
    def n(self):
        return self.shape[0] * self.shape[1] * self.shape[2]

    @property
    def active(self):
        return tuple(a for a in range(3) if self.shape[a] > 1)

    def stencils(self):
        """(axis, sign) pairs in the order the reference iterates them."""
        return [(a, s) for a in self.active for s in (+1, -1)]


def _axis_diff(f, n_a, h, plus):
    """Derivative along axis 0 of f (n_a, ...), one-sided (spatial.py:81-118).

    plus=True is D^+ (minus-biased, (3, -4, 1)/2h on i, i-1, i-2; first
    order at i = 1; zero-inflow ghost at i = 0). plus=False is D^- (the
    mirror image with the closure on the last two cells).
    """
    out = np.empty_like(f)
    if plus:
        out[2:] = (3.0 * f[2:] - 4.0 * f[1:-1] + f[:-2]) / (2.0 * h)
        out[1] = (f[1] - f[0]) / h
        out[0] = f[0] / h
    else:
        out[:-2] = (-3.0 * f[:-2] + 4.0 * f[1:-1] - f[2:]) / (2.0 * h)
        out[-2] = (f[-1] - f[-2]) / h
        out[-1] = -f[-1] / h
    return out


def stencil(grid, axis, sign, f):
    """D_axis^sign applied to every column of f (n, c)."""
    nx, ny, nz = grid.shape
    c = f.shape[1]
    cube = f.reshape(nz, ny, nx, c)
    ax = {0: 2, 1: 1, 2: 0}[axis]
    moved = np.moveaxis(cube, ax, 0)
    d = _axis_diff(moved, grid.shape[axis], grid.h[axis], sign > 0)
    return np.moveaxis(d, 0, ax).reshape(grid.n, c)


class Ops:
    """Angular operator data per axis: V_d, lambda_d^+, lambda_d^- (angular.py:161-202)."""

    def __init__(self, eig_v, lam_plus, lam_minus):
        self.eig_v = [np.asarray(v) for v in eig_v]
        self.lam = {+1: [np.asarray(l) for l in lam_plus], -1: [np.asarray(l) for l in lam_minus]}

    def a_mat(self, axis, sign):
        v = self.eig_v[axis]
        return (v * self.lam[sign][axis]) @ v.T

    def factor(self, w, axis, sign):
        """W^T V_d Lambda^+- V_d^T W (dlra.py:155-166)."""
        c = w.T @ self.eig_v[axis]
        return (c * self.lam[sign][axis]) @ c.T


def apply_streaming(u, inv_s, grid, ops):
    """Full-rank F_S(u) (spatial.py:148-167)."""
    if not np.all(np.isfinite(u)):
        raise FloatingPointError("non-finite streaming input")
    scaled = inv_s[:, None] * u
    out = np.zeros_like(u)
    for axis in grid.active:
        v = ops.eig_v[axis]
        w = scaled @ v
        flux = stencil(grid, axis, +1, w) * ops.lam[+1][axis] + \
            stencil(grid, axis, -1, w) * ops.lam[-1][axis]
        out -= flux @ v.T
    return out


def k_rhs(k, inv_s, grid, factors):
    """-sum_s (D_s S^-1 K) F_s (dlra.py:168-174)."""
    f = inv_s[:, None] * k
    out = np.zeros_like(k)
    for (axis, sign), fs in zip(grid.stencils(), factors):
        out -= stencil(grid, axis, sign, f) @ fs
    return out


def stencil_grams(x, y, inv_s, grid):
    """[X^T D_s S^-1 Y for each stencil s]."""
    f = inv_s[:, None] * y
    return [x.T @ stencil(grid, a, s, f) for a, s in grid.stencils()]


def rk4(f, y0, dt):
    """Classic RK4 (dlra.py:118-123)."""
    k1 = f(y0)
    k2 = f(y0 + 0.5 * dt * k1)
    k3 = f(y0 + 0.5 * dt * k2)
    k4 = f(y0 + dt * k3)
    return y0 + dt / 6.0 * (k1 + 2.0 * k2 + 2.0 * k3 + k4)


# gauge-floor experiment (SURVEY.md Appendix A.1 "eps"): when set, every basis
# is rotated by Z = qr(I + eps (X - X^T)), X seeded Gaussian -- a span-preserving
# change of basis eps away from the identity.
GAUGE = {"eps": 0.0, "rng": None}


def orthonormal_columns(a):
    """Householder QR basis (dlra.py:26-43; the pivoted fallback is the
    reference's safety net and never triggers on these inputs)."""
    q, _ = np.linalg.qr(a)
    if GAUGE["eps"] > 0.0:
        k = q.shape[1]
        x = GAUGE["rng"].standard_normal((k, k))
        z, _ = np.linalg.qr(np.eye(k) + GAUGE["eps"] * (x - x.T))
        q = q @ z
    return q


def streaming_step(u0, s0, v0, dt, inv_s, grid, ops):
    """Augmented BUG streaming step (dlra.py:213-225). Returns (U^, S^, V^)."""
    st = grid.stencils()
    kf = [ops.factor(v0, a, s) for a, s in st]
    k1 = rk4(lambda k: k_rhs(k, inv_s, grid, kf), u0 @ s0, dt)
    # Q_s = (D_s S^-1 U0)^T U0 and A_s = V Lambda V^T (dlra.py:176-194)
    q = [g.T for g in stencil_grams(u0, u0, inv_s, grid)]
    amats = [ops.a_mat(a, s) for a, s in st]

    def l_rhs(l):
        out = np.zeros_like(l)
        for am, qs in zip(amats, q):
            out -= am @ (l @ qs)
        return out

    l1 = rk4(l_rhs, v0 @ s0.T, dt)
    u_hat = orthonormal_columns(np.hstack([k1, u0]))
    v_hat = orthonormal_columns(np.hstack([l1, v0]))
    s_hat0 = (u_hat.T @ u0) @ s0 @ (v0.T @ v_hat)
    g = stencil_grams(u_hat, u_hat, inv_s, grid)
    fh = [ops.factor(v_hat, a, s) for a, s in st]

    def s_rhs(s):
        out = np.zeros_like(s)
        for gs, fs in zip(g, fh):
            out -= gs @ s @ fs
        return out

    s_hat = rk4(s_rhs, s_hat0, dt)
    return u_hat, s_hat, v_hat


def truncate(u, s, v, threshold, rank_min, rank_max):
    """Tail-sum truncation (dlra.py:90-115). Returns (U1, S1, V1, tail)."""
    p, sigma, qt = np.linalg.svd(s, full_matrices=False)
    tails = np.append(np.cumsum(sigma[::-1])[::-1], 0.0)
    r1 = int(np.argmax(tails <= threshold))
    if r1 > rank_max:
        raise ArithmeticError(f"adaptive rank {r1} exceeds rank_max={rank_max}")
    r1 = min(max(r1, rank_min), rank_max, sigma.size)
    return u @ p[:, :r1], np.diag(sigma[:r1]), v @ qt[:r1].T, float(tails[r1])


def scattering_step(u0, s0, v0, dt, weights, inv_s, g_diags, sigma_t, sources):
    """Four-substep scattering update (dlra.py:270-322). Returns (U^, S^, V^)."""
    r = u0.shape[1]
    spatial = weights * inv_s[:, None]
    b = np.stack([(u0 * spatial[:, i:i + 1]).T @ u0 for i in range(spatial.shape[1])])
    coeffs = sigma_t[:, None] - g_diags
    l_cols = s0 @ v0.T
    l_new = np.empty_like(l_cols)
    for q in range(l_cols.shape[1]):
        mat = np.eye(r) + dt * np.einsum("i,ijk->jk", coeffs[:, q], b)
        l_new[:, q] = np.linalg.solve(mat, l_cols[:, q])
    v_t, r_t = np.linalg.qr(l_new.T)
    s_t = r_t.T
    src = np.zeros_like(u0)
    proj = np.zeros((r, v0.shape[0]))
    for psi, tm in sources:
        x = weights * (inv_s * psi)[:, None]
        gt = g_diags * tm[None, :]
        src += x @ (gt @ v0)
        proj += (u0.T @ x) @ gt
    u_hat = orthonormal_columns(np.hstack([u0 @ s0 + dt * src, u0]))
    v_hat = orthonormal_columns(np.hstack([v_t @ s_t.T + dt * proj.T, v_t]))
    s1 = (u_hat.T @ u0) @ s_t @ (v_t.T @ v_hat)
    for psi, tm in sources:
        x = weights * (inv_s * psi)[:, None]
        s1 = s1 + dt * (u_hat.T @ x) @ ((g_diags * tm[None, :]) @ v_hat)
    return u_hat, s1, v_hat


def fullrank_streaming_step(u, dt, inv_s, grid, ops):
    """RK4 on the dense n x m matrix (fullrank.py:16-26)."""
    return rk4(lambda x: apply_streaming(x, inv_s, grid, ops), u, dt)


def fullrank_scattering_step(u, dt, weights, inv_s, g_diags, sigma_t, sources):
    """Scalar implicit self-scattering plus explicit source (fullrank.py:29-40)."""
    rates = (weights * inv_s[:, None]) @ (sigma_t[:, None] - g_diags)
    out = u / (1.0 + dt * rates)
    for psi, tm in sources:
        out = out + dt * (weights * (inv_s * psi)[:, None]) @ (g_diags * tm[None, :])
    return out


def run_energy_loop(bundle, solver="dlra", max_steps=None, start_step=0, state=None):
    """Pseudo-time loop + dose trapezoid (driver.py:541-625) on a ProblemBundle.

    Returns dict(deposited, rank_history, state). `max_steps`/`start_step`
    bound the run (used for the timed CPU baseline sample).
    """
    nx, ny, nz = bundle.shape
    grid = Grid(nx, ny, nz, *bundle.spacing)
    ops = Ops(bundle.eig_v, bundle.lam_plus, bundle.lam_minus)
    n, m = bundle.n_cells, bundle.n_moments
    edges = bundle.pseudo_time_edges()
    n_steps = len(edges) - 1
    stop = n_steps if max_steps is None else min(n_steps, start_step + max_steps)
    weights = bundle.atomic_densities
    if state is None:
        if solver == "dlra":
            r0 = min(bundle.rank_min, n, m)
            rng = np.random.default_rng(bundle.seed)
            u = orthonormal_columns(rng.standard_normal((n, r0)))
            v = orthonormal_columns(rng.standard_normal((m, r0)))
            state = (u, np.zeros((r0, r0)), v)
        else:
            state = np.zeros((n, m))
    deposited = np.zeros(n)
    prev = np.zeros(n)
    ranks = []
    th, rmin, rmax = bundle.truncation_tolerance, bundle.rank_min, bundle.rank_max
    for k in range(start_step, stop):
        e_hi, e_lo = edges[k], edges[k + 1]
        dt = e_hi - e_lo
        e_mid = 0.5 * (e_hi + e_lo)
        s_field = bundle.stopping_field(e_mid)
        inv_s = 1.0 / s_field
        g_diags, sigma_t = bundle.scattering_tables(e_mid)
        sources = list(zip(bundle.psi_at(e_mid), bundle.t_ms))
        if solver == "dlra":
            u, s, v = state
            u, s, v = streaming_step(u, s, v, dt, inv_s, grid, ops)
            if bundle.truncate_after in ("streaming", "both"):
                u, s, v, _ = truncate(u, s, v, th, rmin, rmax)
            u, s, v = scattering_step(u, s, v, dt, weights, inv_s, g_diags, sigma_t, sources)
            if bundle.truncate_after in ("scattering", "both"):
                u, s, v, _ = truncate(u, s, v, th, rmin, rmax)
            state = (u, s, v)
            ranks.append(s.shape[0])
            u0m = u @ (s @ v[0, :])
        else:
            x = fullrank_streaming_step(state, dt, inv_s, grid, ops)
            state = fullrank_scattering_step(x, dt, weights, inv_s, g_diags, sigma_t, sources)
            ranks.append(min(n, m))
            u0m = state[:, 0]
        integrand = np.sqrt(4.0 * np.pi) * u0m
        if bundle.uncollided_tally == "steps":
            integrand = integrand + s_field * bundle.psi_at(e_lo).sum(axis=0)
        deposited += 0.5 * dt * (prev + integrand)
        prev = integrand
    return {"deposited": deposited, "rank_history": ranks, "state": state}
