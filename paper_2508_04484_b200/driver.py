"""Device-resident energy loop: the hot path of pndose.driver.run_simulation.

`run_bundle(bundle)` is the loop of driver.py:541-666 with the state kept on
the GPU for the whole run: per step the host computes only the frozen
coefficients of driver.step_contexts (a few hundred doubles: S per material
class, the 12 x m scattering diagonals, the at_energy interpolation weights)
and one `pnd_step` call does streaming -> truncate -> scattering ->
truncate -> dose trapezoid on the device. The per-cell 1/S and S fields and
the psi_u slices are formed on the device from those scalars.

`run_simulation(config, solver="dlra")` is the drop-in entry point for a
reference `ProblemConfig`: it assembles and ray-traces with the reference's
own host code (which stays unchanged) and hands the energy
loop to the device. It needs the reference package importable; on the GPU
box the tests and the benchmark drive `run_bundle` with committed bundles.
"""

import math
import time
import warnings
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .dlra import LowRankState, orthonormal_columns
from .errors import ConfigError, NumericalError
from .problem import SQRT_4PI, ProblemBundle, UncollidedSlices, export_bundle, export_problem

TRUNCATE_FLAGS = {"streaming": 1, "scattering": 2, "both": 3}
# largest factor rank the step kernels take (an augmented state holds 2x this;
# above 64 the n-side factors are column-blocked, csrc/xwide.cu)
MAX_RANK = 256


@dataclass
class DoseGrid:
    deposited: np.ndarray
    dose: np.ndarray

    @property
    def negativity(self):
        neg = self.deposited < 0.0
        return {
            "min_value": float(self.deposited.min(initial=0.0)),
            "negative_cells": int(np.count_nonzero(neg)),
        }


@dataclass
class SimulationResult:
    bundle: ProblemBundle
    dose: DoseGrid
    rank_history: list
    diagnostics: dict
    uncollided: np.ndarray = field(default=None, repr=False)


class DeviceSolver:
    """One bundle's device state: operators, flux tables, low-rank factors."""

    def __init__(self, bundle: ProblemBundle, device: int = 0, slab=None, comm_id=None,
                 device_coefficients: bool = True):
        """slab: a slabs.Slab (this process's z-planes of a multi-GPU solve)
        with comm_id the world's NCCL id; None = the whole grid on one GPU.
        device_coefficients: evaluate the per-step coefficients on the GPU from
        tables uploaded once (no host->device copy per step); False = the host
        restatement (problem.py) uploads them every step."""
        self.bundle = bundle
        b = bundle
        self.slab = slab
        lo, hi = (0, b.n_cells) if slab is None else slab.rows
        shape = b.shape if slab is None else (b.shape[0], b.shape[1], slab.planes)
        self.rows = (lo, hi)
        self.h = _lib.Handle(shape, b.spacing, b.n_moments, device)
        if slab is not None:
            self.h.set_slab(slab.z0, b.shape[2], comm_id, slab.rank, slab.world)
        self.h.set_angular(*b.a_split())
        self.h.set_materials(b.cell_class[lo:hi], b.class_atomic)
        nb = len(b.fluxes)
        sparse = any(f.cells is not None for f in b.fluxes)
        for i, (f, tm) in enumerate(zip(b.fluxes, b.t_ms)):
            t = _lib.f64(tm)
            if sparse:  # ray-footprint tables (pnd_set_flux_table_sparse)
                f = f if f.cells is not None else UncollidedSlices(
                    f.values, f.residual, f.e_min, f.e_max,
                    np.arange(b.n_cells, dtype=np.int32), b.n_cells)
                sel = (f.cells >= lo) & (f.cells < hi)
                cells = np.ascontiguousarray(f.cells[sel] - lo, dtype=np.int32)
                vals = _lib.f64(f.values[sel])
                self.h.call("pnd_set_flux_table_sparse", i, nb, int(f.values.shape[1]),
                            len(cells), _lib.ptr(cells), _lib.ptr(vals), _lib.ptr(t))
                continue
            vals = _lib.f64(f.values[lo:hi])
            self.h.call("pnd_set_flux_table", i, nb, int(vals.shape[1]), _lib.ptr(vals),
                        _lib.ptr(t))
        self.h.call("pnd_dose_reset")
        self.device_coefficients = False
        if device_coefficients:
            self.upload_coefficient_tables()

    def upload_coefficient_tables(self):
        """Stopping-power, moment and group tables for pnd_coefficients_at (once)."""
        b = self.bundle
        log_e, log_s = np.log(b.stop_e), np.log(b.stop_s)  # problem.class_stopping's tables
        p = len(b.mom_e)
        mom_g = b.mom_g if b.mom_g is not None else np.zeros((12, p, b.pn_order + 2))
        xi1 = b.mom_xi1 if b.mom_xi1 is not None else np.zeros((12, p))
        fr = np.array([[f.e_min, f.e_max] for f in b.fluxes], dtype=np.float64).reshape(-1)
        arrs = [_lib.f64(x) for x in (log_e, log_s, b.class_density, b.class_weights, b.mom_e,
                                      mom_g, xi1, fr if fr.size else np.zeros(2))]
        self.h.call("pnd_set_coefficient_tables", int(log_e.shape[1]), _lib.ptr(arrs[0]),
                    _lib.ptr(arrs[1]), _lib.ptr(arrs[2]), _lib.ptr(arrs[3]), p,
                    _lib.ptr(arrs[4]), int(mom_g.shape[2]), _lib.ptr(arrs[5]),
                    _lib.ptr(arrs[6]), 0 if b.model == "boltzmann" else 1, int(b.pn_order),
                    1 if b.boltzmann_correction else 0, float(b.fp_correction_scale),
                    len(b.fluxes), _lib.ptr(arrs[7]))
        self.device_coefficients = True

    def init_state(self, rank=None, seed=None):
        """LowRankState.zero (dlra.py:54-60): seeded Gaussian bases, S = 0."""
        b = self.bundle
        n, m = b.n_cells, b.n_moments
        r0 = min(b.rank_min if rank is None else rank, n, m)
        st = LowRankState.zero(n, m, r0, seed=b.seed if seed is None else seed)
        lo, hi = self.rows
        self.h.set_state(st.u[lo:hi], st.s, st.v)

    def select_flux(self, which: int, e_mev: float):
        fl = self.bundle.fluxes
        if not fl:
            return
        w = [f.lerp_weights(e_mev) for f in fl]
        j0 = np.array([x[0] for x in w], dtype=np.int32)
        w0 = np.array([x[1] for x in w])
        j1 = np.array([x[2] for x in w], dtype=np.int32)
        w1 = np.array([x[3] for x in w])
        self.h.call("pnd_select_flux", which, _lib.ptr(j0), _lib.ptr(w0), _lib.ptr(j1),
                    _lib.ptr(w1))

    def set_coefficients(self, e_hi: float, e_lo: float):
        """driver.step_contexts (driver.py:523-538), coefficients only."""
        b = self.bundle
        e_mid = 0.5 * (e_hi + e_lo)
        if self.device_coefficients:
            self.h.call("pnd_coefficients_at", e_mid, e_lo,
                        1 if b.uncollided_tally == "steps" else 0)
            return
        self.h.set_class_stopping(b.class_stopping(e_mid))
        g, s = b.scattering_tables(e_mid)
        self.h.set_scattering(g, s)
        self.select_flux(0, e_mid)
        if b.uncollided_tally == "steps":
            self.select_flux(1, e_lo)

    def step(self, dt: float, want_defect: bool = True):
        b = self.bundle
        out = np.zeros(8)
        self.h.call(
            "pnd_step", float(dt), float(b.truncation_tolerance), int(b.rank_min),
            int(b.rank_max), TRUNCATE_FLAGS[b.truncate_after],
            1 if b.uncollided_tally == "steps" else 0, 1 if want_defect else 0, _lib.ptr(out),
        )
        return out

    def checkpoint(self, step: int) -> dict:
        """Snapshot at a step boundary: the factors, the dose
        trapezoid state and the next step index; np.savez-able."""
        u, s_, v = self.state()
        n = self.rows[1] - self.rows[0]
        dep, prev = np.empty(n), np.empty(n)
        self.h.call("pnd_dose_state", _lib.ptr(dep), _lib.ptr(prev))
        return {"u": u, "s": s_, "v": v, "deposited": dep, "prev": prev,
                "step": np.array(int(step))}

    def restore(self, ckpt) -> int:
        """Resume from checkpoint(): returns the step to continue from."""
        self.h.set_state(ckpt["u"], ckpt["s"], ckpt["v"])
        dep, prev = _lib.f64(ckpt["deposited"]), _lib.f64(ckpt["prev"])
        self.h.call("pnd_dose_restore", _lib.ptr(dep), _lib.ptr(prev))
        return int(ckpt["step"])

    def dose(self) -> np.ndarray:
        """Deposited energy of this device's cells (the slab's rows)."""
        out = np.empty(self.rows[1] - self.rows[0])
        self.h.call("pnd_get_dose", _lib.ptr(out))
        return out

    def state(self):
        return self.h.get_state()

    def close(self):
        self.h.close()


def augmented_sizes(n, m, a0, b0, a1, b1):
    """state.u.size + state.s.size + state.v.size right after each substep,
    as the reference's loop records them (driver.py:583-596): the sizes of
    its Householder bases, which depend only on the incoming ranks --
    streaming: U^ = orth([K1, U0]) (n x min(n, a+b)), V^ = orth([L1, V0])
    (m x min(m, a+b)), dlra.py:213-225; scattering: U^ = orth([K1, U0])
    (n x min(n, 2a)), V^ = orth([l3, V~]) with V~ m x min(m, a), dlra.py:270-322."""
    cu, cv = min(n, a0 + b0), min(m, a0 + b0)
    du, dv = min(n, 2 * a1), min(m, a1 + min(m, a1))
    return n * cu + cu * cv + m * cv, n * du + du * dv + m * dv


def check_rank_cap(bundle: ProblemBundle):
    """Ranks the device kernels support: refuse a run whose
    rank_max cannot be reached before it starts, not at the step where the
    adaptive rank first passes the cap (the whole run would be lost)."""
    cap = MAX_RANK if bundle.truncate_after == "both" else MAX_RANK // 2
    if bundle.rank_max > cap and bundle.truncation_tolerance < 1e300:
        warnings.warn(
            f"rank_max={bundle.rank_max} exceeds the device's rank capacity {cap} for "
            f"truncate_after='{bundle.truncate_after}': an adaptive rank above {cap} "
            f"stops the run with a NumericalError naming the step", stacklevel=3)
    if bundle.rank_min > cap:
        raise ConfigError(f"rank_min={bundle.rank_min} exceeds the device's rank capacity {cap}")


def run_bundle(bundle: ProblemBundle, max_steps=None, want_defect=True, device=0,
               solver="dlra", slab=None, comm_id=None, resume=None,
               checkpoint_at=None) -> SimulationResult:
    """The pseudo-time loop of run_simulation (driver.py:541-666) on the device.

    slab / comm_id: this process's z-slab of a multi-GPU solve (slabs.plan)
    and the world's communicator id; the dose then covers the slab's cells.
    resume: a DeviceSolver.checkpoint() dict to continue from; checkpoint_at:
    a step index whose boundary snapshot is returned in
    diagnostics["checkpoint"]. max_steps counts from the start (or resume) step."""
    if solver not in ("dlra", "fullrank"):
        raise ConfigError(f"unknown solver '{solver}'")
    if solver == "fullrank":
        return _run_fullrank(bundle, max_steps, device, slab, comm_id)
    t_start = time.perf_counter()
    b = bundle
    check_rank_cap(b)
    n, m = b.n_cells, b.n_moments
    solver_ = DeviceSolver(b, device, slab=slab, comm_id=comm_id)
    solver_.init_state()
    edges = b.pseudo_time_edges()
    k0 = solver_.restore(resume) if resume is not None else 0
    n_steps = len(edges) - 1
    if max_steps is not None:
        n_steps = min(n_steps, k0 + int(max_steps))
    de = float(edges[0] - edges[1])
    ranks, max_tail, violations, max_defect = [], 0.0, 0, 0.0
    peak_state = 0
    peak_transient = 0
    snapshot = None
    for k in range(k0, n_steps):
        if checkpoint_at is not None and k == int(checkpoint_at):
            snapshot = solver_.checkpoint(k)
        e_hi, e_lo = edges[k], edges[k + 1]
        solver_.set_coefficients(e_hi, e_lo)
        try:
            out = solver_.step(e_hi - e_lo, want_defect)
        except ConfigError as exc:  # the rank capacity, reached mid-run
            raise NumericalError(f"energy step {k} (E = {e_hi:.4f} MeV): {exc}") from exc
        r = int(out[2])
        peak_transient = max(peak_transient, *augmented_sizes(n, m, *out[4:8].astype(int)))
        for idx, flag in ((0, 1), (1, 2)):
            if TRUNCATE_FLAGS[b.truncate_after] & flag:
                tail = float(out[idx])
                max_tail = max(max_tail, tail)
                violations += tail > b.truncation_tolerance + 1e-15
        max_defect = max(max_defect, float(out[3]))
        ranks.append((k, float(e_lo), r))
        peak_state = max(peak_state, n * r + r * r + m * r)
    deposited = solver_.dose()
    lo, hi = solver_.rows
    unc = None
    if b.uncollided_tally == "groups":
        unc = b.uncollided_dose()[lo:hi]
        deposited = deposited + unc
    solver_.close()
    density = b.density[lo:hi]
    dose = DoseGrid(deposited=deposited, dose=deposited / density)
    full = n * m
    diagnostics = {
        "solver": "dlra-b200",
        "n_cells": n,
        "n_moments": m,
        "n_steps": n_steps,
        "energy_step_mev": de,
        "max_orthonormality_defect": max_defect,
        "max_truncation_tail": max_tail,
        "tail_violations": int(violations),
        "mean_rank": float(np.mean([r for _, _, r in ranks])) if ranks else 0.0,
        "max_rank": int(max((r for _, _, r in ranks), default=0)),
        "peak_state_numbers": int(peak_state),
        "peak_transient_numbers": int(peak_transient),
        "fullrank_numbers": int(full),
        "state_memory_fraction": float(peak_state / full),
        "negativity": dose.negativity,
        "runtime_s": time.perf_counter() - t_start,
    }
    if snapshot is not None:
        diagnostics["checkpoint"] = snapshot
    return SimulationResult(bundle=b, dose=dose, rank_history=ranks, diagnostics=diagnostics,
                            uncollided=unc)


@dataclass
class BatchedResult:
    """A beam-batched run (SURVEY.md §8(e) "Beams"): independent solves per
    beam subset, doses summed."""

    dose: DoseGrid
    parts: list                 # beam indices of every subset
    rank_histories: dict        # subset index -> [(step, E_MeV, rank)] (this rank's subsets)
    diagnostics: dict


def run_beam_batched(bundle: ProblemBundle, parts=None, device=0, dist=None, max_steps=None,
                     solve=None) -> BatchedResult:
    """Multi-beam run as independent low-rank solves per beam subset.

    parts: beam indices per subset (default: one subset per beam,
    slabs.beam_partition). With torch.distributed initialised (`dist`), the
    subsets go to groups of ranks (slabs.assign_parts): a group of g ranks
    z-slab shards its subset over an NCCL communicator of its own (its rank-0
    makes the id; the world broadcast carries every group's id), a lone rank
    solves its subsets one after another on its GPU; the doses are summed
    over the world. Not numerically the joint solve (driver.py:549-550 solves
    all sources together): its parity reference is the reference run per
    subset, summed (tests/test_gpu_beams.py). `solve(sub_bundle, slab,
    comm_id)` replaces the device solve (the CPU tests pass the oracle)."""
    from . import slabs as _slabs

    t_start = time.perf_counter()
    b = bundle
    if parts is None:
        parts = _slabs.beam_partition(len(b.fluxes))
    parts = [tuple(int(i) for i in p) for p in parts]
    world = dist.get_world_size() if dist is not None else 1
    rank = dist.get_rank() if dist is not None else 0
    mine = _slabs.assign_parts(world, rank, len(parts))
    # one NCCL id per multi-rank group, made by the group's first rank
    ids = [None] * len(parts)
    grouped = world >= len(parts) and world // len(parts) > 1  # the same on every rank
    if dist is not None and grouped and solve is None:
        local_id = _lib.comm_unique_id() if mine.local_rank == 0 else None
        gathered = [None] * world
        dist.all_gather_object(gathered, (mine.parts, local_id))
        for ps, cid in gathered:
            if cid is not None:
                for p in ps:
                    ids[p] = cid
    if solve is None:
        def solve(sub, slab, cid):
            return run_bundle(sub, device=device, slab=slab, comm_id=cid, max_steps=max_steps)
    total = np.zeros(b.n_cells)
    histories = {}
    for p in mine.parts:
        sub = b.subset_beams(parts[p])
        slab = None
        if mine.local_world > 1:
            slab = _slabs.plan(*b.shape, mine.local_world, mine.local_rank)
        res = solve(sub, slab, ids[p])
        lo, hi = (0, b.n_cells) if slab is None else slab.rows
        total[lo:hi] += res.dose.deposited
        histories[p] = res.rank_history
    if dist is not None:
        total = _slabs.sum_doses(total, dist=dist)
    dose = DoseGrid(deposited=total, dose=total / b.density)
    diagnostics = {"solver": "dlra-beam-batched", "n_cells": b.n_cells,
                   "n_moments": b.n_moments, "parts": parts, "world": world,
                   "group_size": mine.local_world,
                   "negativity": dose.negativity,
                   "runtime_s": time.perf_counter() - t_start}
    return BatchedResult(dose=dose, parts=parts, rank_histories=histories,
                         diagnostics=diagnostics)


def _run_fullrank(b: ProblemBundle, max_steps, device, slab, comm_id) -> SimulationResult:
    """The solver="fullrank" branch of the loop (driver.py:607-621) on the device:
    the dense n x m matrix from zero, streaming RK4 + scattering + dose per step."""
    t_start = time.perf_counter()
    n, m = b.n_cells, b.n_moments
    solver_ = DeviceSolver(b, device, slab=slab, comm_id=comm_id)
    solver_.h.call("pnd_fullrank_reset")
    edges = b.pseudo_time_edges()
    n_steps = len(edges) - 1 if max_steps is None else min(len(edges) - 1, int(max_steps))
    tally = 1 if b.uncollided_tally == "steps" else 0
    ranks = []
    for k in range(n_steps):
        e_hi, e_lo = edges[k], edges[k + 1]
        solver_.set_coefficients(e_hi, e_lo)
        solver_.h.call("pnd_fullrank_step", float(e_hi - e_lo), tally)
        ranks.append((k, float(e_lo), min(n, m)))
    deposited = solver_.dose()
    lo, hi = solver_.rows
    unc = None
    if b.uncollided_tally == "groups":
        unc = b.uncollided_dose()[lo:hi]
        deposited = deposited + unc
    solver_.close()
    dose = DoseGrid(deposited=deposited, dose=deposited / b.density[lo:hi])
    diagnostics = {
        "solver": "fullrank-b200",
        "n_cells": n,
        "n_moments": m,
        "n_steps": n_steps,
        "energy_step_mev": float(edges[0] - edges[1]),
        "fullrank_numbers": int(n * m),
        "negativity": dose.negativity,
        "runtime_s": time.perf_counter() - t_start,
    }
    return SimulationResult(bundle=b, dose=dose, rank_history=ranks, diagnostics=diagnostics,
                            uncollided=unc)


def write_dose_volume(result: SimulationResult, path, binary: bool = True, slab=None):
    """The dose.vtk of driver.write_outputs (driver.py:672-690) for a run_bundle
    result: binary legacy VTK by default (output.py; binary=False is the
    reference's ASCII form). slab: this rank's slabs.Slab of a multi-GPU run,
    whose result holds only its cells -- each rank then writes its own byte
    ranges of the one file (output.write_volume_slab)."""
    from .output import VolumeGrid, write_volume, write_volume_slab

    b = result.bundle
    grid = VolumeGrid(*b.shape, *b.spacing, tuple(b.origin))
    arrays = {"deposited_energy": result.dose.deposited, "dose": result.dose.dose}
    if slab is None:
        write_volume(path, grid, arrays, binary=binary)
    else:
        write_volume_slab(path, grid, list(arrays), arrays, slab.rows[0], slab.rank)


def run_simulation(config, solver: str = "dlra"):
    """Drop-in for pndose.driver.run_simulation(config, solver) (driver.py:541-666).

    `config` is a reference ProblemConfig and the return value is the
    reference's own SimulationResult (problem, DoseGrid(grid, deposited,
    dose), rank_history, diagnostics with every key the reference sets,
    fluxes), so write_outputs (driver.py:809-849) and the CLI (cli.py:18-37)
    consume it unchanged. Problem assembly and the per-beam tracer setup
    (material keys, coefficient closures; driver.py:398-436) are the
    reference's host code; every beam's march and deposit (raytracer.
    trace_beam) and the energy loop run on the GPU. solver="fullrank" runs
    the dense oracle on the device (fullrank.cu); solver="dlra-cpu" hands
    the whole run back to the reference. Errors are the reference's classes
    (errors.py binds pndose.errors when it is importable), so cli.py:130 maps
    them to its exit codes.
    """
    from pndose import driver as ref_driver  # the reference package
    from pndose.angular import beam_projection

    from . import raytracer as dev_tracer

    if solver == "dlra-cpu":
        if _REFERENCE_RUN is not None:  # routed by install(): the original function
            return _REFERENCE_RUN(config, solver="dlra")
        try:  # routed by the source edit of INTEGRATION.md §2, which keeps "dlra-cpu"
            return ref_driver.run_simulation(config, solver="dlra-cpu")
        except ConfigError as exc:  # not routed at all: the reference's own "dlra"
            if "unknown solver" not in str(exc):
                raise
            return ref_driver.run_simulation(config, solver="dlra")
    if solver not in ("dlra", "fullrank"):
        raise ConfigError(f"unknown solver '{solver}'")
    from .moments import MomentTables as DeviceMomentTables

    t_start = time.perf_counter()
    # problem assembly is the reference's host code, with its moment tables
    # (driver.py:269-307) evaluated on the device
    ref_tables = getattr(ref_driver, "MomentTables", None)
    if ref_tables is not None:
        ref_driver.MomentTables = DeviceMomentTables
    try:
        problem = ref_driver.assemble_problem(config)
    finally:
        if ref_tables is not None:
            ref_driver.MomentTables = ref_tables
    ref_trace = ref_driver.trace_beam
    ref_driver.trace_beam = dev_tracer.trace_beam
    try:
        fluxes = ref_driver.trace_all_beams(problem)
    finally:
        ref_driver.trace_beam = ref_trace
    t_ms = [beam_projection(config.pn_order, bm.direction) for bm in config.beams]
    bundle = export_bundle(problem, fluxes, t_ms)  # keeps ray-footprint tables sparse
    res = run_bundle(bundle, solver=solver)
    return reference_result(ref_driver, problem, fluxes, res, solver, t_start)


_REFERENCE_RUN = None


def install():
    """Route the reference's run_simulation to the device
    without editing its source: pndose.driver.run_simulation -- and the name
    pndose.cli imported from it -- become this module's run_simulation;
    solver="dlra-cpu" still reaches the original CPU function."""
    global _REFERENCE_RUN
    from pndose import driver as ref_driver

    if getattr(ref_driver.run_simulation, "_pnd_b200", False):
        return
    _REFERENCE_RUN = ref_driver.run_simulation

    def routed(config, solver: str = "dlra"):
        return run_simulation(config, solver)

    routed._pnd_b200 = True
    routed.__doc__ = run_simulation.__doc__
    ref_driver.run_simulation = routed
    try:
        from pndose import cli as ref_cli
    except ImportError:
        return
    ref_cli.run_simulation = routed


def reference_result(ref_driver, problem, fluxes, res: SimulationResult, solver: str,
                     t_start: float):
    """The reference's SimulationResult (driver.py:494-500) for a device run:
    DoseGrid with the problem's grid, the reference's diagnostics keys and
    order (driver.py:634-659; solver named as the caller asked), the traced
    fluxes, runtime over the whole pipeline."""
    d = res.diagnostics
    n, m = d["n_cells"], d["n_moments"]
    full = n * m
    dose = ref_driver.DoseGrid(grid=problem.grid, deposited=res.dose.deposited,
                               dose=res.dose.dose)
    ranks = [r for _, _, r in res.rank_history]
    dlra = solver == "dlra"
    diagnostics = {
        "solver": solver,
        "n_cells": n,
        "n_moments": m,
        "n_steps": d["n_steps"],
        "energy_step_mev": d["energy_step_mev"],
        "max_orthonormality_defect": float(d.get("max_orthonormality_defect", 0.0)),
        "max_truncation_tail": float(d.get("max_truncation_tail", 0.0)),
        "tail_violations": int(d.get("tail_violations", 0)),
        "mean_rank": float(np.mean(ranks)),
        "max_rank": int(max(ranks)),
        "peak_state_numbers": int(d["peak_state_numbers"] if dlra else full),
        "peak_transient_numbers": int(d["peak_transient_numbers"] if dlra else full),
        "fullrank_numbers": int(full),
        "state_memory_fraction": float((d["peak_state_numbers"] if dlra else full) / full),
        "negativity": dose.negativity,
        "uncollided_undershoot": float(min((f.undershoot for f in fluxes), default=0.0)),
        "runtime_s": time.perf_counter() - t_start,
        "rays_per_beam": [f.n_rays for f in fluxes],
    }
    return ref_driver.SimulationResult(problem=problem, dose=dose,
                                       rank_history=res.rank_history,
                                       diagnostics=diagnostics, fluxes=fluxes)


__all__ = ["DeviceSolver", "run_bundle", "run_beam_batched", "BatchedResult", "run_simulation",
           "reference_result", "install",
           "SimulationResult", "DoseGrid", "SQRT_4PI", "math", "orthonormal_columns"]
