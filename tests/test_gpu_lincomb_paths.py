"""LINCOMB variants against the paths they replace, step by step:
- the one-column LINCOMB (lincomb1_kernel: the rank-one scattering
  augmentation's CGS passes and the Q^T diag(1/S) psi Gram, FP64 FMAs on the
  CUDA cores) against the tensor-core per-warp path (PND_LINCOMB1_OFF);
- the symmetric Gram-only pass (tiles below the diagonal mirrored, used on
  large grids; forced here with PND_LINCOMB_SYM) against the full one.
Both compute the same sums in different orders, so each
energy step taken from the same state agrees to rounding: the gauge-free
product U S V^T within 1e-11 relative (T2's bound), step by step over 30
config-1 steps. (Over a whole trajectory the two orders drift apart like
any two roundings of the reference: the collided dose is basis-gauge
sensitive.)"""
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

STEPS = 30


def _set(var, on):
    if on:
        os.environ[var] = "1"
    else:
        os.environ.pop(var, None)


@pytest.mark.parametrize("var,label", [("PND_LINCOMB1_OFF", "lincomb1_vs_dmma_per_step"),
                                       ("PND_LINCOMB_SYM", "sym_gram_vs_full_per_step")])
def test_lincomb_variant_matches_per_step(parity_log, var, label):
    from paper_2508_04484_b200.driver import DeviceSolver
    from paper_2508_04484_b200.problem import ProblemBundle

    old = os.environ.get(var)
    try:
        b = ProblemBundle.load(GOLDEN / "bundle_config1.npz")
        s = DeviceSolver(b)
        s.init_state()
        edges = b.pseudo_time_edges()
        worst = 0.0
        for k in range(STEPS):
            u0, s0, v0 = s.h.get_state()
            prods = []
            for on in (True, False):
                s.h.set_state(u0, s0, v0)
                _set(var, on)
                s.set_coefficients(edges[k], edges[k + 1])
                s.step(edges[k] - edges[k + 1])
                u, sv, v = s.h.get_state()
                prods.append(u @ sv @ v.T)
            dev = float(np.abs(prods[1] - prods[0]).max() / np.abs(prods[0]).max())
            worst = max(worst, dev)
        parity_log.append({"test": label, "steps": STEPS, "state_rel_dev_max": worst})
        assert worst <= 1e-11, worst
    finally:
        _set(var, False)
        if old is not None:
            os.environ[var] = old
