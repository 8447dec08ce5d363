"""Test-side stand-in for the reference package `pndose` on the GPU box.

/root/reference is absent there, so tests/test_gpu_dropin.py drives the
drop-in run_simulation through this stub of the reference's HOST API: the
names and fields the device path and the reference's result consumers
touch (driver.py:310-321 Problem, 476-500 DoseGrid / SimulationResult,
398-449 trace_all_beams, 809-849 write_outputs; cli.py:18-37, 115-133;
errors.py:4-31), fed from the committed fixtures (tests/golden/bundle_*.npz
written by the real reference). Not product code; only that test imports it.
"""

__version__ = "0.1.0+stub"
