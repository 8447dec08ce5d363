"""Exception hierarchy with the reference's CLI exit categories.

Mirrors /root/reference/pkg/src/pndose/errors.py:4-31 so callers that catch
the reference classes by name (and tests that match message fragments such
as "column", "rank_max", "3-point") see the same behaviour. The C-ABI
returns the exit code as its status (include/pndose_b200.h) and the Python
shim raises the class registered for that code.
"""


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
