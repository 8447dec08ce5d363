"""Wall time of the one-CTA Jacobi SVD (pnd_svd_small) on the shapes the step
uses; a 2 x 2 call gives the copy + launch overhead to subtract."""
import sys
import time

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

from paper_2508_04484_b200 import _lib  # noqa: E402
from paper_2508_04484_b200.dlra import _generic_handle  # noqa: E402


def run(s, reps=2):
    p, q = s.shape
    k = min(p, q)
    pm, sig, qt = np.empty((p, k)), np.empty(k), np.empty((k, q))
    h = _generic_handle()
    s = np.ascontiguousarray(s)
    h.call("pnd_svd_small", _lib.ptr(s), p, q, _lib.ptr(pm), _lib.ptr(sig), _lib.ptr(qt))
    t0 = time.perf_counter()
    for _ in range(reps):
        h.call("pnd_svd_small", _lib.ptr(s), p, q, _lib.ptr(pm), _lib.ptr(sig), _lib.ptr(qt))
    return (time.perf_counter() - t0) / reps * 1e6


rng = np.random.default_rng(0)
base = run(np.eye(2))
print(f"overhead (2x2): {base:.1f} us")
for n in (20, 40, 64):
    g = rng.standard_normal((n, n))
    graded = g * np.exp(-0.5 * np.arange(n))
    u, _ = np.linalg.qr(rng.standard_normal((n, n)))
    gram = u @ np.diag(np.logspace(0, -14, n)) @ u.T
    for name, m in (("gaussian", g), ("graded", graded), ("psd gram", gram)):
        print(f"{n:3d} {name:9s} {run(m) - base:8.1f} us")
