"""Exception hierarchy with the reference's CLI exit categories.

When the reference package is importable (the drop-in deployment: pndose's
driver routed to this package) these ARE its classes
(pkg/src/pndose/errors.py:4-31), so `except PnDoseError` in cli.py:130 and
the reference's tests' `pytest.raises(NumericalError, match="rank_max")` see
the device's errors unchanged. Without it (the GPU box, where only this
package travels) an identical hierarchy with the same names, exit codes and
message fragments ("column", "rank_max", "3-point") stands in. The C-ABI
returns the exit code as its status (include/pndose_b200.h) and the Python
shim raises the class registered for that code.
"""

try:  # the reference's own classes when it is installed
    from pndose.errors import (  # type: ignore  # noqa: F401
        ConfigError,
        NumericalError,
        OutputIOError,
        PhysicsDataError,
        PnDoseError,
    )

    REFERENCE_CLASSES = True
except ImportError:
    REFERENCE_CLASSES = False

    class PnDoseError(Exception):
        exit_code = 1

    class ConfigError(PnDoseError):
        exit_code = 2

    class PhysicsDataError(PnDoseError):
        exit_code = 3

    class NumericalError(PnDoseError):
        exit_code = 4

    class OutputIOError(PnDoseError):
        exit_code = 5


class DeviceError(PnDoseError):
    """CUDA runtime failure or missing native library (no CPU fallback)."""

    exit_code = 6


BY_CODE = {
    2: ConfigError,
    3: PhysicsDataError,
    4: NumericalError,
    5: OutputIOError,
    6: DeviceError,
}
