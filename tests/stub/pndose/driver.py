"""Stub of pndose.driver's host API over a committed problem bundle.

A config names a bundle fixture (tests/golden/bundle_<tag>.npz, the
reference's own assembled problem + traced fluxes) and optional transport
overrides; assemble_problem / trace_all_beams rebuild the reference-shaped
objects export_problem and the result consumers read."""

import json
from dataclasses import dataclass
from pathlib import Path
from types import SimpleNamespace

import numpy as np

from . import angular
from .errors import ConfigError, OutputIOError

GOLDEN = Path(__file__).resolve().parents[2] / "golden"


@dataclass
class Grid3D:
    nx: int
    ny: int
    nz: int
    dx: float
    dy: float
    dz: float
    origin: tuple = (0.0, 0.0, 0.0)

    @property
    def shape(self):
        return (self.nx, self.ny, self.nz)

    @property
    def spacings(self):
        return (self.dx, self.dy, self.dz)

    @property
    def n_cells(self):
        return self.nx * self.ny * self.nz


@dataclass
class ProblemConfig:
    bundle: str
    transport: dict
    output_directory: Path
    name: str = "stub"
    resolved: dict = None
    beams: list = None

    @classmethod
    def load(cls, path):
        path = Path(path)
        try:
            raw = json.loads(path.read_text())
        except FileNotFoundError as exc:
            raise ConfigError(f"config file not found: {path}") from exc
        return cls(bundle=raw["bundle"], transport=raw.get("transport", {}),
                   output_directory=Path(raw["output"]), name=raw.get("name", "stub"),
                   resolved=raw)


@dataclass
class DoseGrid:
    grid: Grid3D
    deposited: np.ndarray
    dose: np.ndarray

    @property
    def negativity(self):
        neg = self.deposited < 0.0
        return {"min_value": float(self.deposited.min(initial=0.0)),
                "negative_cells": int(np.count_nonzero(neg))}


@dataclass
class SimulationResult:
    problem: object
    dose: DoseGrid
    rank_history: list
    diagnostics: dict
    fluxes: list


def _bundle(config):
    return np.load(GOLDEN / config.bundle, allow_pickle=False)


def assemble_problem(config):
    a = _bundle(config)
    sc = a["scalars"]
    strings = [str(s) for s in a["strings"]]
    t = dict(config.transport)
    cfg = SimpleNamespace(
        model=strings[0], pn_order=int(sc[0]), boltzmann_correction=bool(sc[1]),
        fp_correction_scale=float(sc[2]), e_min_mev=float(sc[3]), e_max_mev=float(sc[4]),
        cfl_number=float(sc[5]),
        truncation_tolerance=float(t.get("truncation_tolerance", sc[6])),
        rank_min=int(t.get("rank_min", sc[7])), rank_max=int(t.get("rank_max", sc[8])),
        seed=int(sc[9]), truncate_after=t.get("truncate_after", strings[1]),
        uncollided_tally=strings[2], name=config.name, resolved=config.resolved,
        output_directory=config.output_directory)
    cls = a["cell_class"]
    material = SimpleNamespace(density=a["class_density"][cls],
                               weights=a["class_weights"][cls],
                               atomic_densities=a["class_atomic"][cls])
    tables = {f"e{i}": SimpleNamespace(energies=a["stop_e"][i], values=a["stop_s"][i])
              for i in range(a["stop_e"].shape[0])}
    sh, sp, org = a["shape"], a["spacing"], a["origin"]
    grid = Grid3D(int(sh[0]), int(sh[1]), int(sh[2]), float(sp[0]), float(sp[1]), float(sp[2]),
                  tuple(float(v) for v in org))
    beams = []
    for i, tm in enumerate(a["t_ms"]):
        direction = (0.0, 0.0, 1.0 + i)  # a registry key per beam
        angular._T_MS[(cfg.pn_order, direction)] = tm
        beams.append(SimpleNamespace(direction=direction))
    config.beams = beams
    config.pn_order = cfg.pn_order
    cfg.beams = beams
    return SimpleNamespace(
        config=cfg, grid=grid, material=material, stopping=SimpleNamespace(tables=tables),
        moments=SimpleNamespace(energies=a["mom_e"], g=a["mom_g"], xi1=a["mom_xi1"]),
        ops=SimpleNamespace(eig_v=list(a["eig_v"]), lam_plus=list(a["lam_plus"]),
                            lam_minus=list(a["lam_minus"])),
        n_cells=grid.n_cells, n_moments=int(a["eig_v"].shape[1]))


@dataclass
class UncollidedFlux:
    space: object
    values: np.ndarray
    residual_energy: np.ndarray
    n_rays: int

    @property
    def undershoot(self):
        return float(min(self.values.min(initial=0.0), 0.0))


def trace_beam(*args, **kwargs):  # replaced by the device tracer during run_simulation
    raise AssertionError("run_simulation must route trace_beam to the device tracer")


# --- the reference's straggling model (physics/stopping.py:123-165), restated
_E_CHARGE, _EPS0, _ME_KG, _MEV_J, _C = (1.602176634e-19, 8.8541878128e-12, 9.1093837015e-31,
                                        1.602176634e-13, 2.99792458e8)
_Z = np.array([1, 6, 7, 8, 11, 12, 15, 16, 17, 18, 19, 20], dtype=float)
_I_J = np.array([19.2, 78.0, 82.0, 95.0, 149.0, 156.0, 173.0, 180.0, 174.0, 188.0, 190.0,
                 191.0]) * _E_CHARGE
_PREF = 4.0 * np.pi * _E_CHARGE ** 4 / (4.0 * np.pi * _EPS0) ** 2


def _straggling_t(n_i, e):
    p = np.sqrt(e * (e + 2.0 * 938.272))
    v = p / (e + 938.272) * _C
    me_v2 = _ME_KG * v * v
    log_arg = 2.0 * me_v2 / _I_J
    term = np.where(log_arg > 1.0, 4.0 * _I_J / (3.0 * me_v2) * np.log(log_arg), 0.0)
    return (n_i * 1e6 @ (_PREF * _Z * term)) / _MEV_J ** 2 / 100.0


def _straggling_dt(n_i, e, rel_step=1e-4):
    h = rel_step * max(abs(e), 1.0)
    return (_straggling_t(n_i, e + h) - _straggling_t(n_i, e - h)) / (2.0 * h)


def trace_all_beams(problem):
    """driver.py:398-449: one energy-operator closure triple per unique
    material row, then trace_beam per beam (the device tracer once
    run_simulation has routed it). The closures restate the reference's
    (stopping power by Bragg mixing of the log-log element tables, Williams
    straggling, the corrected total cross section) over the bundle's class
    tables -- the paper_2508_04484_b200.problem restatements, pinned to the
    reference's contexts by tests/test_oracle.py."""
    from paper_2508_04484_b200.problem import ProblemBundle

    cfg = problem.config
    if not cfg.resolved.get("trace"):
        a = np.load(GOLDEN / cfg.resolved["bundle"], allow_pickle=False)
        return [UncollidedFlux(space=SimpleNamespace(e_min=float(r[0]), e_max=float(r[1])),
                               values=v, residual_energy=res, n_rays=441)
                for v, res, r in zip(a["flux_values"], a["flux_residual"], a["flux_range"])]
    b = ProblemBundle.load(GOLDEN / cfg.resolved["bundle"])
    keys = b.cell_class
    coefficients = {}
    for key in range(b.n_classes):
        n_i = b.class_atomic[key]

        def s_star(e, key=key, n_i=n_i):
            e = np.asarray(e, dtype=float)
            s = np.array([b.class_stopping(float(x))[key] for x in np.atleast_1d(e).ravel()])
            dt = np.array([_straggling_dt(n_i, float(x)) for x in np.atleast_1d(e).ravel()])
            return (s + 0.5 * dt).reshape(np.shape(e))

        def t_coeff(e, n_i=n_i):
            e = np.asarray(e, dtype=float)
            return np.array([_straggling_t(n_i, float(x))
                             for x in np.atleast_1d(e).ravel()]).reshape(np.shape(e))

        def sigma_t_fn(e, n_i=n_i):
            e = np.asarray(e, dtype=float)
            return np.array([float(n_i @ b.scattering_tables(float(x))[1])
                             for x in np.atleast_1d(e).ravel()]).reshape(np.shape(e))

        coefficients[key] = (s_star, t_coeff, sigma_t_fn)
    t = cfg.resolved["trace"]
    space = SimpleNamespace(e_min=b.fluxes[0].e_min, e_max=b.fluxes[0].e_max,
                            n_groups=b.fluxes[0].n_groups, degree=2)
    out = []
    for bm in t["beams"]:
        beam = SimpleNamespace(direction=tuple(bm["direction"]), energy_mev=bm["energy_mev"],
                               position_cm=tuple(bm["position_cm"]), weight=bm.get("weight", 1.0),
                               sigma_xy_cm=bm.get("sigma_xy_cm", 0.3),
                               sigma_e_mev=0.01 * bm["energy_mev"])
        out.append(trace_beam(beam, problem.grid, space, keys, coefficients,
                              n_side=t["n_side"], span_sigmas=3.0, max_step=0.01))
    return out


def run_simulation(config, solver="dlra"):
    raise AssertionError("the stub has no CPU solver; install() routes this to the device")


def write_outputs(result):
    """The reads of driver.py:809-849: result.problem.config / .grid, the dose
    arrays, the rank history, the diagnostics (JSON manifest)."""
    config = result.problem.config
    out = Path(config.output_directory)
    try:
        out.mkdir(parents=True, exist_ok=True)
    except OSError as exc:
        raise OutputIOError(f"output directory {out} is not writable: {exc}") from exc
    grid = result.problem.grid
    np.save(out / "deposited.npy", result.dose.deposited.reshape(grid.nz, grid.ny, grid.nx))
    np.save(out / "dose.npy", result.dose.dose)
    with open(out / "rank_history.csv", "w") as fh:
        fh.write("step,E_MeV,rank\n")
        for step, e_mev, rank in result.rank_history:
            fh.write(f"{step},{e_mev:.9g},{rank}\n")
    (out / "manifest.json").write_text(json.dumps(
        {"name": config.name, "diagnostics": result.diagnostics}, sort_keys=True, default=str))
    return out
