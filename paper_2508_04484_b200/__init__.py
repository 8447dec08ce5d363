"""B200-native collided-flux DLRA energy stepper (arXiv 2508.04484).

Drop-in for the hot path of the reference package `pndose`: the low-rank
streaming/scattering substeps, the truncation, the energy loop with its dose
tally, and the uncollided ray traversal run as sm_100a CUDA kernels behind the
C-ABI in include/pndose_b200.h. The Python modules here mirror the reference
API (dlra, spatial, raytracer, driver); they hold no numerical fallback --
every compute call goes through libpndose_b200.so and raises DeviceError when
it is missing.
"""

__version__ = "0.1.0"
