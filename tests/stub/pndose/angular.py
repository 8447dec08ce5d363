"""beam_projection (angular.py:251-253) served from the fixture's T_M rows."""

import numpy as np

_T_MS = {}


def beam_projection(n_max, direction):
    return np.asarray(_T_MS[(int(n_max), tuple(float(v) for v in direction))])
