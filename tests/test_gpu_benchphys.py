"""T2 parity at the benchmarked physics, step by step, against the reference.

tests/golden/lock_<tag>.npz holds, for a few steps k of a reference run, the
input state, the frozen contexts and the reference's factors after each
substep and truncation (tools/make_golden.py run_lockstep_record):

  fp19:   water, P19 Fokker-Planck (m = 400), fixed rank 20 -- BASELINE
          configs[1]'s physics on 10 x 10 x 12 cells: the m = 400 split-K
          m-side GEMMs, the one-CTA m-side QR at 400 rows, the K-stage/S-Gram
          kernels at r = 20 / R = 40;
  slabs7: water / bone / lung z-slabs, Boltzmann P7, fixed rank 20 --
          BASELINE configs[2]'s physics on 10 x 10 x 24 cells: the
          three-class scattering path (per-class weighted Grams, materialised
          source rows) at r = 20.

Every substep starts from the reference's own previous output, so each one is
checked in isolation (no accumulated gauge drift). Compared: U S V^T
(gauge-invariant), singular values and the tail; never individual factors.
"""

from types import SimpleNamespace

import numpy as np
import pytest

from conftest import golden

pytestmark = pytest.mark.gpu

CASES = [("fp19", k) for k in (2, 25, 50)] + [("slabs7", k) for k in (2, 150, 300)]


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def mat(L, p):
    return L[p + "_u"] @ L[p + "_s"] @ L[p + "_v"].T


@pytest.fixture(scope="module")
def dl():
    from paper_2508_04484_b200 import dlra

    return dlra


def _ctx(dl, L, tag, k):
    g = L["grid"]
    grid = SimpleNamespace(nx=int(g[0]), ny=int(g[1]), nz=int(g[2]), dx=float(g[3]),
                           dy=float(g[4]), dz=float(g[5]))
    B = golden(f"bundle_{tag}.npz")  # the same run's P_N operators
    ops = SimpleNamespace(eig_v=list(B["eig_v"]), lam_plus=list(B["lam_plus"]),
                          lam_minus=list(B["lam_minus"]))
    p = f"k{k}_"
    sc = dl.StreamingContext(L[p + "inv_s"], SimpleNamespace(grid=grid), ops)
    cc = dl.ScatteringContext(L["weights"], L[p + "inv_s"], L[p + "g_diags"],
                              L[p + "sigma_t"], list(zip(L[p + "psi"], L["t_ms"])))
    return sc, cc, float(L[p + "dt"])


def _truncation_bound(sig, r):
    """Rank-r truncation of a perturbed S^: the kept subspace moves by about
    |dS| / (sigma_r - sigma_r+1) (Wedin), so the T2 bound is scaled by the
    relative gap of the reference's own spectrum at the cut."""
    if sig.size <= r or sig[r] == 0.0:
        return 1.0
    return max(1.0, sig[0] / max(sig[r - 1] - sig[r], 1e-300))


@pytest.mark.parametrize("tag,k", CASES)
def test_streaming_substep(dl, tag, k, parity_log):
    L = golden(f"lock_{tag}.npz")
    sc, _, dt = _ctx(dl, L, tag, k)
    p = f"k{k}"
    st = dl.LowRankState(L[p + "_u"], L[p + "_s"], L[p + "_v"])
    aug = dl.streaming_step(st, dt, sc)
    dev = rel(aug.matrix(), mat(L, p + "_sa"))
    r = st.s.shape[0]
    tr, tail = dl.truncate(aug, dl.TruncationPolicy(1e300, r, r))
    dev_t = rel(tr.matrix(), mat(L, p + "_st"))
    ref_sig = np.linalg.svd(L[p + "_sa_s"], compute_uv=False)
    amp = _truncation_bound(ref_sig, r)
    parity_log.append({"test": "streaming_substep", "tag": tag, "step": k, "dev_aug": dev,
                       "dev_truncated": dev_t, "gap_amplification": amp,
                       "aug_rank_ref": int(L[p + "_sa_s"].shape[0]),
                       "aug_rank_gpu": int(min(aug.s.shape)),
                       "tail_ref": float(L[p + "_st_tail"]), "tail_gpu": tail})
    assert aug.orthonormality_defect() < 1e-12
    assert dev < 1e-11, dev
    assert dev_t < 1e-11 * amp, (dev_t, amp)
    assert tail == pytest.approx(float(L[p + "_st_tail"]), rel=1e-8 * amp)


@pytest.mark.parametrize("tag,k", CASES)
def test_scattering_substep(dl, tag, k, parity_log):
    L = golden(f"lock_{tag}.npz")
    _, cc, dt = _ctx(dl, L, tag, k)
    p = f"k{k}"
    st = dl.LowRankState(L[p + "_st_u"], L[p + "_st_s"], L[p + "_st_v"])
    aug = dl.scattering_step(st, dt, cc)
    dev = rel(aug.matrix(), mat(L, p + "_ca"))
    ref_sig = np.linalg.svd(L[p + "_ca_s"], compute_uv=False)
    # the reference's Householder QR turns the rank-deficient source
    # augmentation's rounding noise into extra directions (sigma ~ 1e-16 of
    # the largest); compare on the numerical rank
    numerical = int(np.count_nonzero(ref_sig > 1e-12 * ref_sig[0]))
    sig = np.linalg.svd(aug.s, compute_uv=False)
    r = st.s.shape[0]
    tr, tail = dl.truncate(aug, dl.TruncationPolicy(1e300, r, r))
    dev_t = rel(tr.matrix(), mat(L, p + "_ct"))
    amp = _truncation_bound(ref_sig, r)
    parity_log.append({"test": "scattering_substep", "tag": tag, "step": k, "dev_aug": dev,
                       "dev_truncated": dev_t, "gap_amplification": amp,
                       "numerical_rank_ref": numerical, "aug_rank_gpu": int(min(aug.s.shape)),
                       "sigma_dev": float(np.abs(sig[:numerical] - ref_sig[:numerical]).max()
                                          / ref_sig[0])})
    assert aug.orthonormality_defect() < 1e-12
    assert numerical <= min(aug.s.shape)
    assert np.abs(sig[:numerical] - ref_sig[:numerical]).max() < 1e-11 * ref_sig[0]
    assert dev < 1e-11, dev
    assert dev_t < 1e-11 * amp, (dev_t, amp)
