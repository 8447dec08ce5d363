"""Beam-batched mode on the device against the reference run per subset.

SURVEY.md §8(e) "Beams": a multi-beam problem split into independent
low-rank solves per beam subset, doses summed. Not the joint solve, so the
parity reference is the reference itself run on each subset with the joint
run's energy grid (tests/golden/e2e_hetero_b{0,1}.npz, tools/make_golden.py
hetero_beam_raw), summed; tolerance 10 x the subsets' gauge floors (T5).
"""

import json

import numpy as np
import pytest

from conftest import GOLDEN, golden

pytestmark = pytest.mark.gpu

FLOORS = json.loads((GOLDEN / "floors.json").read_text())


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def test_beam_batched_matches_reference_per_subset(parity_log):
    from paper_2508_04484_b200.driver import run_beam_batched
    from paper_2508_04484_b200.problem import ProblemBundle

    b = ProblemBundle.load(GOLDEN / "bundle_hetero.npz")
    res = run_beam_batched(b, parts=[(0,), (1,)])
    refs = [golden(f"e2e_hetero_b{i}.npz") for i in (0, 1)]
    want = refs[0]["deposited"] + refs[1]["deposited"]
    unc = refs[0]["uncollided"] + refs[1]["uncollided"]
    for i in (0, 1):
        np.testing.assert_array_equal([r for _, _, r in res.rank_histories[i]],
                                      refs[i]["rank_history"][:, 2].astype(int))
    floor_t = max(FLOORS[f"hetero_b{i}"]["total"] for i in (0, 1))
    floor_c = max(FLOORS[f"hetero_b{i}"]["collided"] for i in (0, 1))
    dev_t = rel(res.dose.deposited, want)
    dev_c = rel(res.dose.deposited - unc, want - unc)
    joint = golden("e2e_hetero.npz")["deposited"]
    parity_log.append({"test": "beam_batched", "tag": "hetero {0},{1}", "dev_total": dev_t,
                       "floor_total": floor_t, "dev_collided": dev_c, "floor_collided": floor_c,
                       "batched_vs_joint_reference": rel(want, joint)})
    assert dev_t <= max(10 * floor_t, 1e-12), (dev_t, floor_t)
    assert dev_c <= max(10 * floor_c, 1e-10), (dev_c, floor_c)


def test_beam_batched_single_subset_is_the_joint_run():
    """One subset holding every beam is the joint solve, bit for bit."""
    from paper_2508_04484_b200.driver import run_beam_batched, run_bundle
    from paper_2508_04484_b200.problem import ProblemBundle

    b = ProblemBundle.load(GOLDEN / "bundle_hetero.npz")
    res = run_beam_batched(b, parts=[(0, 1)], max_steps=30)
    joint = run_bundle(b, max_steps=30)
    assert res.dose.deposited.tobytes() == joint.dose.deposited.tobytes()
