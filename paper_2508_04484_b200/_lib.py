"""ctypes binding of libpndose_b200.so (include/pndose_b200.h).

There is no CPU fallback: if the shared library is missing or no CUDA device
is usable, every call raises DeviceError. Status codes map onto the
reference's exception classes (pkg/src/pndose/errors.py) with the message
the library produced.
"""

import ctypes
from pathlib import Path

import numpy as np

from .errors import BY_CODE, DeviceError, PnDoseError

LIB_PATH = Path(__file__).resolve().parent / "libpndose_b200.so"

_P = ctypes.c_void_p
_I = ctypes.c_int
_D = ctypes.c_double

# name -> argtypes (every function returns int)
SIGNATURES = {
    "pnd_create": [ctypes.POINTER(_P), _I, _I, _I, _D, _D, _D, _I, _I],
    "pnd_destroy": [_P],
    "pnd_last_error": [_P, ctypes.c_char_p, ctypes.c_size_t],
    "pnd_synchronize": [_P],
    "pnd_device_bytes": [_P, _P],
    "pnd_set_angular": [_P, _P, _P],
    "pnd_set_materials": [_P, _P, _I, _P],
    "pnd_set_inv_s": [_P, _P],
    "pnd_set_class_stopping": [_P, _P],
    "pnd_set_scattering": [_P, _P, _P],
    "pnd_set_sources": [_P, _I, _P, _P],
    "pnd_set_flux_table": [_P, _I, _I, _I, _P, _P],
    "pnd_select_flux": [_P, _I, _P, _P, _P, _P],
    "pnd_set_flux_table_sparse": [_P, _I, _I, _I, _I, _P, _P, _P],
    "pnd_moment_tables": [_P, _I, _P, _I, _P, _P, _I, _P, _P, _P, _P, _I, _D, _D, _P, _P],
    "pnd_state_set": [_P, _I, _I, _P, _P, _P],
    "pnd_state_shape": [_P, _P, _P],
    "pnd_state_get": [_P, _P, _P, _P],
    "pnd_streaming_step": [_P, _D],
    "pnd_scattering_step": [_P, _D],
    "pnd_truncate": [_P, _D, _I, _I, _P, _P],
    "pnd_step": [_P, _D, _D, _I, _I, _I, _I, _I, _P],
    "pnd_dose_reset": [_P],
    "pnd_dose_accumulate": [_P, _D, _I],
    "pnd_get_dose": [_P, _P],
    "pnd_dose_state": [_P, _P, _P],
    "pnd_dose_restore": [_P, _P, _P],
    "pnd_orth_defect": [_P, _P],
    "pnd_apply_streaming": [_P, _P, _P],
    "pnd_stencil_grams": [_P, _P, _I, _P, _I, _P],
    "pnd_k_rhs": [_P, _P, _I, _P, _P],
    "pnd_augment_basis": [_P, _P, _I, _P, _I, _I, _P, _P],
    "pnd_orthonormalize": [_P, _P, _I, _I, _P, _P],
    "pnd_svd_small": [_P, _P, _I, _I, _P, _P, _P],
    "pnd_set_coefficient_tables": [_P, _I, _P, _P, _P, _P, _I, _P, _I, _P, _P, _I, _I, _I, _D,
                                   _I, _P],
    "pnd_coefficients_at": [_P, _D, _D, _I],
    "pnd_fullrank_reset": [_P],
    "pnd_fullrank_set": [_P, _P],
    "pnd_fullrank_get": [_P, _P],
    "pnd_fullrank_streaming_step": [_P, _D],
    "pnd_fullrank_scattering_step": [_P, _D],
    "pnd_fullrank_step": [_P, _D, _I],
    "pnd_get_coefficients": [_P, _P, _P, _P, _P, _P],
    "pnd_traverse": [_P, _P, _I, _P, _P, _P, _P, _P, _P, _P],
    "pnd_timing": [_P, _I],
    "pnd_timing_get": [_P, _I, _P, _P],
    "pnd_event_record": [_P, _I],
    "pnd_event_elapsed": [_P, _I, _I, _P],
    "pnd_launch_count": [_P, _P],
    "pnd_spec_stats": [_P, _P],
    "pnd_set_flux_separable": [_P, _I, _I, _I, _P, _P, _P],
    "pnd_state_random": [_P, _I, ctypes.c_ulonglong],
    "pnd_march": [_P, _I, _I, _I, _P, _P, _P, _D, _P, _P, _I, _P, _P, _I, _P, _P, _P, _P, _P,
                  _P, _P, _P],
    "pnd_deposit": [_P, _I, _I, _P, _P, _P, _P, _P, _P, _D, _I, _P, _P, _P, _P],
    "pnd_comm_unique_id": [ctypes.c_char_p],
    "pnd_set_slab": [_P, _I, _I, ctypes.c_char_p, _I, _I],
}

PHASES = ["kstage", "l_gram", "l_side", "tsqr_n", "tsqr_m", "s_gram", "s_rk4", "svd",
          "rotate", "scat_k1", "scat_gram", "scat_small", "dose", "defect"]

_lib = None


def lib():
    """Load the native library once; raise DeviceError when it is absent."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise DeviceError(
                f"{LIB_PATH.name} is not built; run `python -m paper_2508_04484_b200.build` "
                "(there is no CPU fallback)"
            )
        handle = ctypes.CDLL(str(LIB_PATH))
        for name, argtypes in SIGNATURES.items():
            fn = getattr(handle, name)
            fn.argtypes = argtypes
            fn.restype = _I
        _lib = handle
    return _lib


def ptr(a):
    return None if a is None else a.ctypes.data_as(_P)


def f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


class Handle:
    """One device-resident solve (grid, moments) behind a pnd_handle."""

    def __init__(self, shape, spacing, m, device=0):
        self._h = _P()
        self.shape = tuple(int(v) for v in shape)
        self.spacing = tuple(float(v) for v in spacing)
        self.m = int(m)
        self.n = self.shape[0] * self.shape[1] * self.shape[2]
        rc = lib().pnd_create(ctypes.byref(self._h), *self.shape, *self.spacing, self.m,
                              int(device))
        if rc != 0:
            msg = self._message()
            lib().pnd_destroy(self._h)
            self._h = None
            raise BY_CODE.get(rc, PnDoseError)(msg)
        self.uploaded = {}

    def _message(self):
        buf = ctypes.create_string_buffer(2048)
        lib().pnd_last_error(self._h, buf, len(buf))
        return buf.value.decode(errors="replace")

    def call(self, name, *args):
        rc = getattr(lib(), name)(self._h, *args)
        if rc != 0:
            raise BY_CODE.get(rc, PnDoseError)(self._message())

    def close(self):
        if self._h:
            lib().pnd_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------ helpers
    def set_slab(self, z0, nz_global, comm_id=None, rank=0, world=1):
        """This handle holds planes [z0, z0 + nz) of a grid of nz_global planes
        (comm.cu); comm_id: the 128-byte NCCL id shared by the world."""
        cid = comm_id if comm_id is not None else bytes(128)
        self.call("pnd_set_slab", int(z0), int(nz_global), ctypes.c_char_p(bytes(cid)),
                  int(rank), int(world))

    def set_angular(self, a_plus, a_minus):
        ap, am = f64(a_plus), f64(a_minus)
        self.call("pnd_set_angular", ptr(ap), ptr(am))

    def set_inv_s(self, inv_s):
        v = f64(inv_s)
        self.call("pnd_set_inv_s", ptr(v))

    def set_materials(self, cell_class, class_atomic):
        c, a = i32(cell_class), f64(class_atomic)
        self.call("pnd_set_materials", ptr(c), int(a.shape[0]), ptr(a))

    def set_class_stopping(self, class_s):
        v = f64(class_s)
        self.call("pnd_set_class_stopping", ptr(v))

    def set_scattering(self, g_diags, sigma_t):
        g, s = f64(g_diags), f64(sigma_t)
        self.call("pnd_set_scattering", ptr(g), ptr(s))

    def set_sources(self, psi, t_m):
        p, t = f64(psi), f64(t_m)
        self.call("pnd_set_sources", int(p.shape[0]), ptr(p), ptr(t))

    def set_state(self, u, s, v):
        u, s, v = f64(u), f64(s), f64(v)
        self.call("pnd_state_set", int(s.shape[0]), int(s.shape[1]), ptr(u), ptr(s), ptr(v))

    def get_state(self):
        ru, rv = _I(), _I()
        self.call("pnd_state_shape", ctypes.byref(ru), ctypes.byref(rv))
        u = np.empty((self.n, ru.value))
        s = np.empty((ru.value, rv.value))
        v = np.empty((self.m, rv.value))
        self.call("pnd_state_get", ptr(u), ptr(s), ptr(v))
        return u, s, v


def comm_unique_id():
    """A fresh NCCL unique id (128 bytes) for pnd_set_slab."""
    buf = ctypes.create_string_buffer(128)
    rc = lib().pnd_comm_unique_id(buf)
    if rc != 0:
        raise BY_CODE.get(rc, PnDoseError)("cannot create an NCCL unique id")
    return buf.raw
