"""Gauge floors of the end-to-end fixtures: dev(oracle, reference).

The DLRA trajectory at rank >= 2 is ill-conditioned in the basis gauge
(SURVEY.md §0.4): two correct CPU implementations that differ only in
rounding already disagree on the collided dose. This script measures, per
fixture, the relative L2 deviation of the numpy oracle (oracle/dlra_np.py)
from the reference's own output, for the total and the collided dose, and
writes tests/golden/floors.json. The GPU parity tests accept
dev(GPU, reference) <= 10 x floor (tier T5 of SURVEY.md §8(c)).

    OPENBLAS_NUM_THREADS=1 python tools/measure_floors.py
"""

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle import dlra_np  # noqa: E402
from paper_2508_04484_b200.problem import ProblemBundle  # noqa: E402


def rel(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / nb) if nb > 0 else float(np.linalg.norm(a))


def main():
    out = {}
    for tag in ("smoke", "config1", "hetero", "fp", "rank1", "fp19", "slabs7", "hetero_b0", "hetero_b1"):
        b = ProblemBundle.load(ROOT / f"tests/golden/bundle_{tag}.npz")
        g = np.load(ROOT / f"tests/golden/e2e_{tag}.npz")
        unc = b.uncollided_dose()
        entry = {}
        for label, eps in (("impl", 0.0), ("eps", 1e-15)):
            dlra_np.GAUGE.update(eps=eps, rng=np.random.default_rng(7))
            res = dlra_np.run_energy_loop(b)
            dep = res["deposited"] + (unc if b.uncollided_tally == "groups" else 0.0)
            entry[label] = {
                "total": rel(dep, g["deposited"]),
                "collided": rel(dep - unc, g["deposited"] - g["uncollided"]),
                "ranks_equal": bool(np.array_equal(np.array(res["rank_history"]),
                                                   g["rank_history"][:, 2].astype(int))),
            }
        dlra_np.GAUGE.update(eps=0.0, rng=None)
        entry["total"] = max(entry["impl"]["total"], entry["eps"]["total"])
        entry["collided"] = max(entry["impl"]["collided"], entry["eps"]["collided"])
        out[tag] = entry
        print(tag, out[tag])
    (ROOT / "tests/golden/floors.json").write_text(json.dumps(out, indent=2) + "\n")


if __name__ == "__main__":
    main()
