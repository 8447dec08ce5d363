"""Small dense-kernel microbenchmark. Truncation SVD on augmented S^ matrices captured from the
config-1 reference trajectory (oracle run, tools/data/svd_caps_config1.npy):
accuracy against numpy and wall time per call of pnd_svd_small, for the
QR-preconditioned kernel and (PND_SVD_PLAIN=1) the plain Jacobi kernel.
Then the one-CTA m-side QR (pnd_orthonormalize) at 64 x 40 and 400 x 40 (the
P7 and P19 moment counts at rank 20). Kernel durations come from an ncu
launch list of this script."""
import os
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2508_04484_b200 import _lib  # noqa: E402
from paper_2508_04484_b200.dlra import _generic_handle  # noqa: E402


def run(s):
    p, q = s.shape
    k = min(p, q)
    pm, sig, qt = np.empty((p, k)), np.empty(k), np.empty((k, q))
    _generic_handle().call("pnd_svd_small", _lib.ptr(np.ascontiguousarray(s)), p, q,
                           _lib.ptr(pm), _lib.ptr(sig), _lib.ptr(qt))
    return pm, sig, qt


def main():
    caps = np.load(Path(__file__).resolve().parent / "data" / "svd_caps_config1.npy")
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    for mode in ("qrj", "plain"):
        if mode == "plain":
            os.environ["PND_SVD_PLAIN"] = "1"
        worst = [0.0, 0.0, 0.0]
        for s in caps:
            pm, sig, qt = run(s)
            ref = np.linalg.svd(s, compute_uv=False)
            k = sig.size
            worst[0] = max(worst[0], float(np.abs(sig - ref).max() / ref[0]))
            worst[1] = max(worst[1], float(np.abs(pm.T @ pm - np.eye(k)).max()),
                           float(np.abs(qt @ qt.T - np.eye(k)).max()))
            worst[2] = max(worst[2], float(np.linalg.norm(pm @ np.diag(sig) @ qt - s)
                                           / np.linalg.norm(s)))
        t0 = time.perf_counter()
        for _ in range(reps):
            for s in caps:
                run(s)
        dt = (time.perf_counter() - t0) / (reps * len(caps))
        print(f"{mode}: sigma dev {worst[0]:.2e} orth {worst[1]:.2e} recon {worst[2]:.2e} "
              f"wall/call {dt * 1e6:.1f} us", flush=True)


def qr_cases(reps):
    rng = np.random.default_rng(7)
    for rows, cols in ((64, 40), (400, 40)):
        a = rng.standard_normal((rows, cols)) * np.exp(-0.5 * np.arange(cols))
        q, r = np.empty((rows, cols)), np.empty((cols, cols))
        h = _generic_handle()
        for _ in range(reps):
            h.call("pnd_orthonormalize", _lib.ptr(a), rows, cols, _lib.ptr(q), _lib.ptr(r))
        print(f"qr {rows}x{cols}: orth {np.abs(q.T @ q - np.eye(cols)).max():.2e} "
              f"recon {np.abs(q @ r - a).max() / np.abs(a).max():.2e}", flush=True)


if __name__ == "__main__":
    main()
    qr_cases(int(sys.argv[1]) if len(sys.argv) > 1 else 3)
