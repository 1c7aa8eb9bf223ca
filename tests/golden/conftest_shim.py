"""Signed in-band values for SR fixtures (same recipe as the reference's
tests/conftest.py:19-27 helper, restated here)."""

import numpy as np


def in_band_values(shape, seed, lo_exp=-7.0, hi_exp=-3.5):
    rng = np.random.default_rng(seed)
    mag = 10.0 ** rng.uniform(lo_exp, hi_exp, size=shape)
    sign = np.where(rng.random(shape) < 0.5, -1.0, 1.0)
    return mag * sign
