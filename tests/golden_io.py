"""Load the golden fixtures written by tests/golden/make_golden.py."""
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    z = np.load(os.path.join(GOLDEN, name), allow_pickle=False)
    cases = {}
    for key in z.files:
        case, field = key.split(".", 1)
        v = z[key]
        cases.setdefault(case, {})[field] = v.item() if v.ndim == 0 else v
    return cases


SYSTEMS = {
    # golden name -> (oracle system, fwave, reversed, reference equation kind)
    "ac2d": ("acoustics-2d", False, False),
    "ac2d_adj_rev": ("acoustics-2d", True, True),
    "ac2d_adj": ("acoustics-2d", True, False),
    "ac2d_rev": ("acoustics-2d", False, True),
    "swe_wet": ("swe-linear-2d", False, False),
    "swe_dry": ("swe-linear-2d", False, False),
    "swe_adj_rev": ("swe-linear-2d", True, True),
    "swe_wet_adj_rev": ("swe-linear-2d", True, True),
    "ac1d": ("acoustics-1d", False, False),
    "ac1d_adj_rev": ("acoustics-1d", True, True),
}
