"""The C-ABI library loads on a CPU-only host and exports every symbol that
include/pndose_b200.h declares (no compute calls here -- those need a GPU)."""

import ctypes
import re

from conftest import ROOT


def declared_symbols():
    text = (ROOT / "include" / "pndose_b200.h").read_text()
    return sorted(set(re.findall(r"^int (pnd_\w+)\(", text, flags=re.M)))


def test_header_declares_the_boundary():
    names = declared_symbols()
    for required in ("pnd_create", "pnd_streaming_step", "pnd_scattering_step", "pnd_truncate",
                     "pnd_step", "pnd_traverse", "pnd_apply_streaming"):
        assert required in names


def test_library_exports_every_declared_symbol():
    from paper_2508_04484_b200 import _lib
    from paper_2508_04484_b200.build import build

    build()
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    missing = [n for n in declared_symbols() if not hasattr(lib, n)]
    assert not missing, missing
    # the ctypes signature table covers the same set
    assert sorted(_lib.SIGNATURES) == declared_symbols()


def test_no_gpu_means_loud_failure():
    import pytest

    from paper_2508_04484_b200 import _lib
    from paper_2508_04484_b200.errors import PnDoseError

    try:
        import torch

        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    with pytest.raises(PnDoseError):
        _lib.Handle((4, 4, 4), (0.1, 0.1, 0.1), 4)
