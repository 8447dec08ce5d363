"""Host half of the drop-in boundary against the REAL reference (CPU).

Runs where /root/reference exists (the build container; skipped elsewhere):
the result that `driver.run_simulation` builds around a device run
(`driver.reference_result`) is fed to the reference's own consumers --
`write_outputs` (driver.py:809-849) and the CLI's exit-code mapping
(cli.py:115-133) -- and its diagnostics must carry exactly the keys of the
reference's run_simulation (driver.py:634-659). The device run itself is
stood in for by the reference's dose (no GPU here); tests/test_gpu_dropin.py
covers the device path through a stub of the same API on the GPU box.
"""

import json
import subprocess
import sys
import time
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT, golden

REF = Path("/root/reference/pkg/src")
pytestmark = pytest.mark.skipif(not REF.exists(), reason="reference tree not present")


def _smoke_config(out):
    sys.path.insert(0, str(REF))
    from pndose import driver as ref_driver

    raw = {
        "name": "smoke",
        "grid": {"nx": 8, "ny": 8, "nz": 12,
                 "delta_x_cm": 0.25, "delta_y_cm": 0.25, "delta_z_cm": 0.25},
        "phantom": {"background_hu": 0.0},
        "beams": [{"direction": [0, 0, 1], "energy_mev": 20.0, "position_cm": [1.0, 1.0, 0.0]}],
        "pn_order": 3,
        "transport": {"cfl_number": 0.2},
        "energy": {"groups": 64},
        "rays": {"n_side": 5},
        "output": {"directory": str(out)},
    }
    return ref_driver, ref_driver.ProblemConfig.from_dict(raw)


def test_reference_result_feeds_reference_write_outputs(tmp_path):
    from paper_2508_04484_b200 import driver as dev

    ref_driver, config = _smoke_config(tmp_path / "out")
    problem = ref_driver.assemble_problem(config)
    fluxes = ref_driver.trace_all_beams(problem)
    g = golden("e2e_smoke.npz")
    dep = g["deposited"]
    hist = [(int(k), float(e), int(r)) for k, e, r in g["rank_history"]]
    n, m = problem.n_cells, problem.n_moments
    fake = dev.SimulationResult(
        bundle=None, dose=dev.DoseGrid(deposited=dep, dose=dep / problem.material.density),
        rank_history=hist,
        diagnostics={"n_cells": n, "n_moments": m, "n_steps": len(hist),
                     "energy_step_mev": 0.1, "max_orthonormality_defect": 1e-15,
                     "max_truncation_tail": 0.0, "tail_violations": 0,
                     "peak_state_numbers": n * 2 + 4 + m * 2,
                     "peak_transient_numbers": n * 4 + 16 + m * 4})
    res = dev.reference_result(ref_driver, problem, fluxes, fake, "dlra", time.perf_counter())
    assert isinstance(res, ref_driver.SimulationResult)
    assert isinstance(res.dose, ref_driver.DoseGrid) and res.dose.grid is problem.grid
    assert set(res.diagnostics) == set(json.loads(str(g["diagnostics"])))
    assert list(res.diagnostics) == list(json.loads(str(g["diagnostics"])))  # same order
    out = ref_driver.write_outputs(res)
    man = json.loads((out / "manifest.json").read_text())
    assert man["diagnostics"]["solver"] == "dlra"
    assert man["diagnostics"]["rays_per_beam"] == [f.n_rays for f in fluxes]
    _, vol = ref_driver.read_volume(out / "dose.vtk")
    np.testing.assert_allclose(vol["deposited_energy"], dep, rtol=1e-11)


def test_errors_are_the_reference_classes_when_importable():
    """With pndose importable, the package raises pndose.errors' own classes,
    so the reference CLI (cli.py:130) maps them to its exit codes."""
    code = (
        "import sys; sys.path[:0] = [sys.argv[1], sys.argv[2]]\n"
        "import pndose.errors as re\n"
        "from paper_2508_04484_b200 import errors, _lib\n"
        "assert errors.REFERENCE_CLASSES\n"
        "assert errors.ConfigError is re.ConfigError and errors.NumericalError is re.NumericalError\n"
        "assert issubclass(errors.DeviceError, re.PnDoseError) and errors.DeviceError.exit_code == 6\n"
        "assert _lib.errors.BY_CODE[4] is re.NumericalError if hasattr(_lib, 'errors') else True\n"
        "print('ok')\n")
    proc = subprocess.run([sys.executable, "-c", code, str(REF), str(ROOT)], capture_output=True,
                          text=True, timeout=120)
    assert proc.returncode == 0 and "ok" in proc.stdout, proc.stderr
