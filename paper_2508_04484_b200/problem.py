"""Problem data and the per-step frozen coefficients, host side.

This is the host half of the drop-in boundary: the energy loop on the device
needs, per step, the stopping-power field at mid-step (1/S), the corrected
per-element scattering diagonals g (12 x m) and sigma_t (12), and the
uncollided flux slice psi_u per beam. The reference computes these in
`driver.step_contexts` (/root/reference/pkg/src/pndose/driver.py:523-538)
from an assembled `Problem` (driver.py:310-362) and the traced fluxes
(raytracer.py:440-449).

`ProblemBundle` is a compact, self-contained form of that assembled problem
(material classes instead of a dense n x 12 weight field, the stopping-power
and angular-moment tables instead of closures), so the device loop can run
where the reference package is absent. `export_problem` builds a bundle from
a reference `Problem`; `ProblemBundle.load` reads one from .npz.

Every coefficient function below restates the reference formula it cites;
the CPU tests pin them against contexts produced by the reference itself
(tests/golden/e2e_*.npz, keys ctx*).
"""

from dataclasses import dataclass, field, replace

import numpy as np

SQRT_4PI = float(np.sqrt(4.0 * np.pi))
N_ELEMENTS = 12


def pn_degrees(n_max: int) -> np.ndarray:
    """Degree l of every real-harmonic index p = l^2 + l + k (angular.py:39-42)."""
    return np.concatenate([np.full(2 * l + 1, l) for l in range(n_max + 1)])


@dataclass
class UncollidedSlices:
    """Group-sampled uncollided flux of one beam (raytracer.UncollidedFlux).

    Dense (cells = None): values (n, G), residual (n,). Ray-footprint form
    (cells = the strictly increasing cells the beam's rays touched): values
    (nnz, G), residual (nnz,), zero in every other cell of the n_cells."""

    values: np.ndarray        # (n, G) or (nnz, G) group representatives
    residual: np.ndarray      # (n,) or (nnz,) below-cutoff energy density
    e_min: float
    e_max: float
    cells: np.ndarray = None  # (nnz,) int32 footprint cells, or None (dense)
    n_cells: int = 0          # grid cells (footprint form)

    def dense(self) -> "UncollidedSlices":
        if self.cells is None:
            return self
        v = np.zeros((self.n_cells, self.values.shape[1]))
        r = np.zeros(self.n_cells)
        v[self.cells] = self.values
        r[self.cells] = self.residual
        return UncollidedSlices(v, r, self.e_min, self.e_max)

    @property
    def n_groups(self) -> int:
        return self.values.shape[1]

    @property
    def centers(self) -> np.ndarray:
        edges = np.linspace(self.e_min, self.e_max, self.n_groups + 1)
        return 0.5 * (edges[:-1] + edges[1:])

    @property
    def width(self) -> float:
        return (self.e_max - self.e_min) / self.n_groups

    def lerp_weights(self, e: float):
        """(j0, w0, j1, w1) with at_energy(e) = w0 v[:, j0] + w1 v[:, j1].

        Restates UncollidedFlux.at_energy (raytracer.py:440-449): linear
        interpolation between group centers, the edge group held flat inside
        [e_min, e_max], zero outside.
        """
        c = self.centers
        g = self.n_groups
        if e <= c[0] or e >= c[-1]:
            j = 0 if e <= c[0] else g - 1
            inside = self.e_min <= e <= self.e_max
            return (j, 1.0 if inside else 0.0, j, 0.0)
        j = int(np.searchsorted(c, e)) - 1
        w = (e - c[j]) / (c[j + 1] - c[j])
        return (j, 1.0 - w, j + 1, w)

    def at_energy(self, e: float) -> np.ndarray:
        if self.cells is not None:
            out = np.zeros(self.n_cells)
            out[self.cells] = UncollidedSlices(self.values, self.residual, self.e_min,
                                               self.e_max).at_energy(e)
            return out
        j0, w0, j1, w1 = self.lerp_weights(e)
        if w0 == 0.0 and w1 == 0.0:
            return np.zeros(self.values.shape[0])
        if w1 == 0.0:
            return self.values[:, j0] if w0 == 1.0 else w0 * self.values[:, j0]
        return w0 * self.values[:, j0] + w1 * self.values[:, j1]


@dataclass
class ProblemBundle:
    """Assembled inputs of one simulation in compact form."""

    shape: tuple                 # (nx, ny, nz)
    spacing: tuple               # (dx, dy, dz)
    origin: tuple
    cell_class: np.ndarray       # (n,) int32 material class per cell
    class_density: np.ndarray    # (M,)
    class_weights: np.ndarray    # (M, 12) mass fractions
    class_atomic: np.ndarray     # (M, 12) atomic densities N_i
    stop_e: np.ndarray           # (12, K) stopping-table energies
    stop_s: np.ndarray           # (12, K) mass stopping powers
    mom_e: np.ndarray            # (P,) moment-table energies
    mom_g: np.ndarray            # (12, P, N+2) per-atom Legendre moments
    mom_xi1: np.ndarray          # (12, P)
    eig_v: np.ndarray            # (3, m, m)
    lam_plus: np.ndarray         # (3, m)
    lam_minus: np.ndarray        # (3, m)
    t_ms: np.ndarray             # (B, m) beam projections
    fluxes: list                 # [UncollidedSlices] per beam
    model: str = "boltzmann"
    pn_order: int = 7
    boltzmann_correction: bool = True
    fp_correction_scale: float = 0.5
    e_min: float = 1.0
    e_max: float = 10.0
    cfl_number: float = 0.7
    truncation_tolerance: float = 0.01
    rank_min: int = 2
    rank_max: int = 100
    truncate_after: str = "both"
    uncollided_tally: str = "groups"
    seed: int = 20260809
    name: str = "run"
    _log_tables: tuple = field(default=None, repr=False)

    # ------------------------------------------------------------ sizes
    @property
    def n_cells(self) -> int:
        return int(np.prod(self.shape))

    @property
    def n_moments(self) -> int:
        return (self.pn_order + 1) ** 2

    @property
    def n_classes(self) -> int:
        return self.class_density.shape[0]

    @property
    def density(self) -> np.ndarray:
        return self.class_density[self.cell_class]

    @property
    def atomic_densities(self) -> np.ndarray:
        """(n, 12) N_i per cell (materials.py:176-184)."""
        return self.class_atomic[self.cell_class]

    @property
    def spectral_radius(self) -> float:
        """max |lambda| over the three flux matrices (angular.py:196-202)."""
        return float(
            max(
                max(lp.max(initial=0.0), -lm.min(initial=0.0))
                for lp, lm in zip(self.lam_plus, self.lam_minus)
            )
        )

    def a_split(self):
        """Gauge-free A_d^+- = V_d diag(lambda^+-) V_d^T per axis (dlra.py:181-182)."""
        ap = np.stack([(v * lp) @ v.T for v, lp in zip(self.eig_v, self.lam_plus)])
        am = np.stack([(v * lm) @ v.T for v, lm in zip(self.eig_v, self.lam_minus)])
        return ap, am

    # ----------------------------------------------- per-step coefficients
    def class_stopping(self, e_mev: float) -> np.ndarray:
        """S(E) per material class [MeV/cm].

        Restates mix_stopping_power (stopping.py:107-120): log-log linear
        interpolation of each element table (stopping.py:48-56), Bragg
        additivity rho * sum_i w_i s_i(E).
        """
        if self._log_tables is None:
            self._log_tables = (np.log(self.stop_e), np.log(self.stop_s))
        log_e, log_s = self._log_tables
        x = np.log(e_mev)
        s_elem = np.array(
            [np.exp(np.interp(x, log_e[i], log_s[i])) for i in range(N_ELEMENTS)]
        )
        return self.class_density * (self.class_weights @ s_elem)

    def stopping_field(self, e_mev: float) -> np.ndarray:
        """S(E, cell) (driver.py:331-335)."""
        return self.class_stopping(e_mev)[self.cell_class]

    def _interp_moments(self, table, e):
        """MomentTables._interp (driver.py:290-296)."""
        en = self.mom_e
        idx = int(np.clip(np.searchsorted(en, e) - 1, 0, len(en) - 2))
        w = (e - en[idx]) / (en[idx + 1] - en[idx])
        return (1.0 - w) * table[:, idx] + w * table[:, idx + 1]

    def scattering_tables(self, e_mev: float):
        """Corrected per-element (g_diags (12, m), sigma_t (12,)) at one energy.

        Restates Problem.scattering_tables (driver.py:337-362) with the
        Boltzmann transport correction (angular.py:229-235) and the FP
        Laplace-Beltrami diagonal plus its correction (angular.py:217-248).
        """
        n_max = self.pn_order
        degrees = pn_degrees(n_max)
        if self.model == "boltzmann":
            moments = np.stack(
                [self._interp_moments(self.mom_g[..., d], e_mev)
                 for d in range(self.mom_g.shape[-1])],
                axis=-1,
            )
            g_diags = moments[:, degrees]
            sigma_t = moments[:, 0].copy()
            if self.boltzmann_correction:
                g_next = moments[:, n_max + 1]
                g_diags = g_diags - g_next[:, None]
                sigma_t = sigma_t - g_next
            return g_diags, sigma_t
        xi1 = self._interp_moments(self.mom_xi1, e_mev)
        lb = degrees * (degrees + 1.0)
        g_diags = np.stack([-(x / 2.0) * lb for x in xi1])
        sigma_t = np.zeros(N_ELEMENTS)
        scale = self.fp_correction_scale
        if scale > 0.0:
            lam_next = -(xi1 / 2.0) * (n_max + 1.0) * (n_max + 2.0)
            g_diags = g_diags - (scale * lam_next)[:, None]
            sigma_t = sigma_t - scale * lam_next
        return g_diags, sigma_t

    def psi_at(self, e_mev: float) -> np.ndarray:
        """(B, n) uncollided flux per beam at e (raytracer.py:440-449)."""
        return np.array([f.at_energy(e_mev) for f in self.fluxes])

    def cfl_step(self) -> float:
        """driver._cfl_step (driver.py:503-512)."""
        s_at_emax = self.class_stopping(self.e_max)[np.unique(self.cell_class)]
        active = [h for n, h in zip(self.shape, self.spacing) if n > 1]
        if not active:
            from .errors import ConfigError

            raise ConfigError("grid has no active axis")
        return self.cfl_number * min(active) * float(s_at_emax.min()) / self.spectral_radius

    def pseudo_time_edges(self) -> np.ndarray:
        """driver.pseudo_time_edges (driver.py:515-520)."""
        de = self.cfl_step()
        n_steps = max(1, int(np.ceil((self.e_max - self.e_min) / de)))
        return np.linspace(self.e_max, self.e_min, n_steps + 1)

    def uncollided_dose(self) -> np.ndarray:
        """Group-sum tally sum_g S(E_g) psi_g h + residual (driver.py:452-461)."""
        deposited = np.zeros(self.n_cells)
        for flux in self.fluxes:
            rows = slice(None) if flux.cells is None else flux.cells
            cls = self.cell_class[rows]  # S(E_g) per cell = the class value, gathered
            for g, e_g in enumerate(flux.centers):
                deposited[rows] += self.class_stopping(e_g)[cls] * flux.values[:, g] * flux.width
            deposited[rows] += flux.residual
        return deposited

    def subset_beams(self, beams) -> "ProblemBundle":
        """The same problem with only the given beams' sources: one subset of
        a beam-batched run (slabs.beam_partition). The energy grid (e_max) is
        the whole problem's, as in the joint run."""
        beams = [int(i) for i in beams]
        return replace(self, t_ms=self.t_ms[beams], fluxes=[self.fluxes[i] for i in beams],
                       _log_tables=None)

    # ----------------------------------------------------------------- io
    def to_arrays(self) -> dict:
        out = {
            "shape": np.array(self.shape),
            "spacing": np.array(self.spacing, dtype=float),
            "origin": np.array(self.origin, dtype=float),
            "cell_class": self.cell_class.astype(np.int32),
            "class_density": self.class_density,
            "class_weights": self.class_weights,
            "class_atomic": self.class_atomic,
            "stop_e": self.stop_e,
            "stop_s": self.stop_s,
            "mom_e": self.mom_e,
            "mom_g": self.mom_g,
            "mom_xi1": self.mom_xi1,
            "eig_v": self.eig_v,
            "lam_plus": self.lam_plus,
            "lam_minus": self.lam_minus,
            "t_ms": self.t_ms,
            "flux_values": np.stack([f.dense().values for f in self.fluxes]),
            "flux_residual": np.stack([f.dense().residual for f in self.fluxes]),
            "flux_range": np.array([[f.e_min, f.e_max] for f in self.fluxes]),
            "scalars": np.array(
                [self.pn_order, float(self.boltzmann_correction), self.fp_correction_scale,
                 self.e_min, self.e_max, self.cfl_number, self.truncation_tolerance,
                 self.rank_min, self.rank_max, self.seed]
            ),
            "strings": np.array([self.model, self.truncate_after, self.uncollided_tally,
                                 self.name]),
        }
        return out

    @classmethod
    def from_arrays(cls, a) -> "ProblemBundle":
        sc = a["scalars"]
        st = [str(s) for s in a["strings"]]
        fluxes = [
            UncollidedSlices(v, r, float(rg[0]), float(rg[1]))
            for v, r, rg in zip(a["flux_values"], a["flux_residual"], a["flux_range"])
        ]
        return cls(
            shape=tuple(int(v) for v in a["shape"]),
            spacing=tuple(float(v) for v in a["spacing"]),
            origin=tuple(float(v) for v in a["origin"]),
            cell_class=np.asarray(a["cell_class"], dtype=np.int32),
            class_density=a["class_density"],
            class_weights=a["class_weights"],
            class_atomic=a["class_atomic"],
            stop_e=a["stop_e"],
            stop_s=a["stop_s"],
            mom_e=a["mom_e"],
            mom_g=a["mom_g"],
            mom_xi1=a["mom_xi1"],
            eig_v=a["eig_v"],
            lam_plus=a["lam_plus"],
            lam_minus=a["lam_minus"],
            t_ms=a["t_ms"],
            fluxes=fluxes,
            model=st[0],
            pn_order=int(sc[0]),
            boltzmann_correction=bool(sc[1]),
            fp_correction_scale=float(sc[2]),
            e_min=float(sc[3]),
            e_max=float(sc[4]),
            cfl_number=float(sc[5]),
            truncation_tolerance=float(sc[6]),
            rank_min=int(sc[7]),
            rank_max=int(sc[8]),
            seed=int(sc[9]),
            truncate_after=st[1],
            uncollided_tally=st[2],
            name=st[3],
        )

    @classmethod
    def load(cls, path) -> "ProblemBundle":
        with np.load(path, allow_pickle=False) as a:
            return cls.from_arrays({k: a[k] for k in a.files})


def export_problem(problem, fluxes, t_ms) -> dict:
    """Compact arrays of a reference `Problem` + traced fluxes (export_bundle's
    ProblemBundle as .npz-able arrays; footprint tables densified)."""
    return export_bundle(problem, fluxes, t_ms).to_arrays()


def export_bundle(problem, fluxes, t_ms) -> "ProblemBundle":
    """A reference `Problem` + traced fluxes as a ProblemBundle.

    `problem` is duck-typed on pndose.driver.Problem (driver.py:310-321);
    material classes are the unique (density, weights) rows, exactly the
    grouping trace_all_beams uses (driver.py:400-403).
    """
    mat = problem.material
    rows = np.column_stack([mat.density, mat.weights])
    uniq, inverse = np.unique(rows, axis=0, return_inverse=True)
    inverse = np.asarray(inverse).ravel()
    first = np.array([int(np.argmax(inverse == k)) for k in range(uniq.shape[0])])
    atomic = np.asarray(mat.atomic_densities)[first]
    lib = problem.stopping
    symbols = list(lib.tables)
    lengths = {len(lib.tables[s].energies) for s in symbols}
    if len(lengths) != 1:
        raise ValueError("stopping tables must share one grid length for a bundle")
    stop_e = np.stack([lib.tables[s].energies for s in symbols])
    stop_s = np.stack([lib.tables[s].values for s in symbols])
    cfg = problem.config
    grid = problem.grid
    bundle = ProblemBundle(
        shape=grid.shape,
        spacing=grid.spacings,
        origin=tuple(grid.origin),
        cell_class=inverse.astype(np.int32),
        class_density=np.asarray(mat.density)[first],
        class_weights=np.asarray(mat.weights)[first],
        class_atomic=atomic,
        stop_e=stop_e,
        stop_s=stop_s,
        mom_e=problem.moments.energies,
        mom_g=problem.moments.g,
        mom_xi1=problem.moments.xi1,
        eig_v=np.stack(problem.ops.eig_v),
        lam_plus=np.stack(problem.ops.lam_plus),
        lam_minus=np.stack(problem.ops.lam_minus),
        t_ms=np.stack(t_ms),
        fluxes=[
            UncollidedSlices(f.values, f.residual_energy, f.space.e_min, f.space.e_max,
                             getattr(f, "cells", None), int(getattr(f, "n_cells", 0) or 0))
            for f in fluxes
        ],
        model=cfg.model,
        pn_order=cfg.pn_order,
        boltzmann_correction=cfg.boltzmann_correction,
        fp_correction_scale=cfg.fp_correction_scale,
        e_min=cfg.e_min_mev,
        e_max=cfg.e_max_mev,
        cfl_number=cfg.cfl_number,
        truncation_tolerance=cfg.truncation_tolerance,
        rank_min=cfg.rank_min,
        rank_max=cfg.rank_max,
        truncate_after=cfg.truncate_after,
        uncollided_tally=cfg.uncollided_tally,
        seed=cfg.seed,
        name=cfg.name,
    )
    return bundle
