"""Speculative steps (pnd_step on small grids): the host predicts the step's
augmentation and truncation ranks, the device checks them, one
synchronisation per step. The result must be bit-identical to the
synchronous path -- accepted steps and steps recomputed after a rejected
prediction alike (PND_SPEC_TEST_MISS forces rejections)."""
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

STEPS = 30


def _run(env):
    from paper_2508_04484_b200 import _lib
    from paper_2508_04484_b200.driver import DeviceSolver
    from paper_2508_04484_b200.problem import ProblemBundle

    old = {k: os.environ.get(k) for k in ("PND_NO_SPEC", "PND_SPEC_TEST_MISS")}
    for k in old:
        os.environ.pop(k, None)
    os.environ.update(env)
    try:
        b = ProblemBundle.load(GOLDEN / "bundle_config1.npz")
        s = DeviceSolver(b)
        s.init_state()
        edges = b.pseudo_time_edges()
        outs = []
        for k in range(STEPS):
            s.set_coefficients(edges[k], edges[k + 1])
            outs.append(s.step(edges[k] - edges[k + 1]))
        u, sv, v = s.h.get_state()
        dep = np.empty(b.n_cells)
        s.h.call("pnd_get_dose", _lib.ptr(dep))
        hm = np.zeros(2, dtype=np.int64)
        s.h.call("pnd_spec_stats", _lib.ptr(hm))
        return np.array(outs), u @ sv @ v.T, dep, hm
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def test_speculative_steps_are_bit_identical(parity_log):
    ref = _run({"PND_NO_SPEC": "1"})
    spec = _run({})
    miss = _run({"PND_SPEC_TEST_MISS": "3"})
    assert ref[3][0] == 0 and ref[3][1] == 0
    assert spec[3][0] >= STEPS - 5, spec[3]  # all but the first few steps speculative
    assert miss[3][1] >= 5, miss[3]          # the restore path ran
    parity_log.append({"test": "speculative_steps", "steps": STEPS,
                       "spec_hits_misses": spec[3].tolist(),
                       "forced_miss_hits_misses": miss[3].tolist()})
    for run in (spec, miss):
        np.testing.assert_array_equal(run[0], ref[0])
        np.testing.assert_array_equal(run[1], ref[1])
        np.testing.assert_array_equal(run[2], ref[2])
