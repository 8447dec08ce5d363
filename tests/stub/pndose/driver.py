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
    raise AssertionError("the stub never traces; fluxes come from the fixture")


def trace_all_beams(problem):
    a = np.load(GOLDEN / problem.config.resolved["bundle"], allow_pickle=False)
    return [UncollidedFlux(space=SimpleNamespace(e_min=float(r[0]), e_max=float(r[1])),
                           values=v, residual_energy=res, n_rays=441)
            for v, res, r in zip(a["flux_values"], a["flux_residual"], a["flux_range"])]


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
