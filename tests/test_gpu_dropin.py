"""The drop-in boundary end to end on the GPU box.

The reference is absent on the GPU box, so a child process puts the stub of
its host API (tests/stub/pndose, fed from the reference-written bundles) on
sys.path, routes pndose.driver.run_simulation to the device with
`paper_2508_04484_b200.driver.install()`, and drives the reference CLI's
`run` / `oracle` commands: the result must be the reference's
SimulationResult type that write_outputs consumes, carry every diagnostics
key the reference's own run wrote (tests/golden/e2e_smoke.npz), raise the
reference's error classes, and map them to its exit codes.
"""

import json
import subprocess
import sys

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, golden

pytestmark = pytest.mark.gpu

CHILD = r'''
import json, sys
sys.path[:0] = [sys.argv[1], sys.argv[2]]
import pndose.cli, pndose.driver, pndose.errors
from paper_2508_04484_b200 import driver as dev, errors
assert errors.REFERENCE_CLASSES and errors.NumericalError is pndose.errors.NumericalError
dev.install()
assert pndose.cli.run_simulation is pndose.driver.run_simulation
out = {"rc": [pndose.cli.main([cmd, path]) for cmd, path in json.loads(sys.argv[3])]}
cfg = pndose.driver.ProblemConfig.load(json.loads(sys.argv[3])[0][1])
res = pndose.driver.run_simulation(cfg)
out["type"] = type(res).__module__ + "." + type(res).__name__
out["dose_type"] = type(res.dose).__name__
out["grid_is_problem_grid"] = res.dose.grid is res.problem.grid
out["n_fluxes"] = len(res.fluxes)
print("RESULT " + json.dumps(out))
'''


def _config(tmp_path, name, bundle, transport=None):
    out = tmp_path / name
    path = tmp_path / f"{name}.json"
    path.write_text(json.dumps({"bundle": bundle, "transport": transport or {},
                                "output": str(out), "name": name}))
    return str(path), out


TRACE_CHILD = r'''
import json, sys
sys.path[:0] = [sys.argv[1], sys.argv[2]]
import numpy as np
import pndose.driver
from paper_2508_04484_b200 import driver as dev
dev.install()
cfg = pndose.driver.ProblemConfig.load(sys.argv[3])
res = pndose.driver.run_simulation(cfg)
ref = np.load(sys.argv[4])
dev_v = max(float(np.abs(f.values - v).max() / np.abs(v).max())
            for f, v in zip(res.fluxes, ref["flux_values"]))
np.save(sys.argv[5], res.dose.deposited)
print("RESULT " + json.dumps({"flux_dev": dev_v, "n_fluxes": len(res.fluxes),
                              "rays": [f.n_rays for f in res.fluxes]}))
'''


def test_trace_all_beams_coupling_through_device_tracer(tmp_path):
    """driver.py:398-449 (d5): the per-material closure triples and the
    per-beam trace_beam calls of trace_all_beams, with trace_beam routed to
    the device tracer by run_simulation -- the two-beam heterogeneous phantom
    (three material classes, an axial and an oblique beam): the traced tables
    equal the reference-traced ones the bundle carries, and the dose the
    reference's run (T5 floors)."""
    g = golden("e2e_hetero.npz")
    path = tmp_path / "hetero.json"
    path.write_text(json.dumps({
        "bundle": "bundle_hetero.npz", "output": str(tmp_path / "out"), "name": "hetero",
        "trace": {"n_side": 5, "beams": [
            {"direction": [0, 0, 1], "energy_mev": 25.0, "position_cm": [1.0, 1.0, 0.0]},
            {"direction": [0, 0.6, 0.8], "energy_mev": 22.0, "position_cm": [1.0, 0.3, 0.0],
             "weight": 0.5}]}}))
    dose_path = tmp_path / "dose.npy"
    proc = subprocess.run([sys.executable, "-c", TRACE_CHILD, str(ROOT / "tests" / "stub"),
                           str(ROOT), str(path), str(GOLDEN / "bundle_hetero.npz"),
                           str(dose_path)], capture_output=True, text=True, timeout=600)
    assert proc.returncode == 0, proc.stderr[-3000:]
    res = json.loads([x for x in proc.stdout.splitlines() if x.startswith("RESULT ")][-1][7:])
    assert res["n_fluxes"] == 2
    assert res["flux_dev"] < 1e-10, res
    dep = np.load(dose_path)
    floors = json.loads((GOLDEN / "floors.json").read_text())["hetero"]
    assert np.linalg.norm(dep - g["deposited"]) / np.linalg.norm(g["deposited"]) <= \
        max(10 * floors["total"], 1e-12)


def test_run_simulation_dropin_through_reference_cli(tmp_path):
    ok, ok_out = _config(tmp_path, "ok", "bundle_smoke.npz")
    fr, fr_out = _config(tmp_path, "fr", "bundle_smoke.npz")
    bad, _ = _config(tmp_path, "bad", "bundle_smoke.npz",
                     {"truncation_tolerance": 0.0, "rank_min": 1, "rank_max": 2})
    cmds = [["run", ok], ["oracle", fr], ["run", bad]]
    proc = subprocess.run([sys.executable, "-c", CHILD, str(ROOT / "tests" / "stub"), str(ROOT),
                           json.dumps(cmds)], capture_output=True, text=True, timeout=600)
    assert proc.returncode == 0, proc.stderr[-3000:]
    line = [x for x in proc.stdout.splitlines() if x.startswith("RESULT ")][-1]
    res = json.loads(line[7:])
    # exit codes: success, success, NumericalError (rank_max, cli.py:130 mapping)
    assert res["rc"] == [0, 0, 4], (res, proc.stderr[-2000:])
    assert "rank_max" in proc.stderr
    assert res["type"] == "pndose.driver.SimulationResult"
    assert res["dose_type"] == "DoseGrid" and res["grid_is_problem_grid"]
    assert res["n_fluxes"] == 1
    # write_outputs wrote the reference's outputs; the manifest's diagnostics
    # carry exactly the keys of the reference's own run
    g = golden("e2e_smoke.npz")
    ref_keys = set(json.loads(str(g["diagnostics"])))
    for out, solver in ((ok_out, "dlra"), (fr_out, "fullrank")):
        man = json.loads((out / "manifest.json").read_text())
        assert set(man["diagnostics"]) == ref_keys, set(man["diagnostics"]) ^ ref_keys
        assert man["diagnostics"]["solver"] == solver
    dep = np.load(ok_out / "deposited.npy").ravel()
    floors = json.loads((GOLDEN / "floors.json").read_text())["smoke"]
    assert np.linalg.norm(dep - g["deposited"]) / np.linalg.norm(g["deposited"]) <= \
        10 * floors["total"]
    hist = (ok_out / "rank_history.csv").read_text().splitlines()[1:]
    assert [int(r.split(",")[2]) for r in hist] == g["rank_history"][:, 2].astype(int).tolist()
