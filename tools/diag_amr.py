"""Diagnostic: exact-variant AMR run vs golden, per level, first step."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1511_03645_b200 import _lib  # noqa: E402
from tests.golden_io import load  # noqa: E402
from tests import test_gpu_amr as T  # noqa: E402

AMR = load("amr.npz")
for name in ("ac2d_hetero", "ac2d_adjoint"):
    out = T.run(name, _lib.VARIANT_EXACT)
    g = AMR[name]
    for step, snap in enumerate(out):
        for lev in range(1, snap["nlev"] + 1):
            got, want = snap[f"L{lev}_q"], g[f"s{step}_L{lev}_q"]
            d = np.argwhere(got != want)
            print(name, "step", step, "lev", lev, "ndiff", len(d), "max", float(np.max(np.abs(got - want))) if len(d) else 0.0,
                  "first", d[:3].tolist())
        if any(not np.array_equal(snap[f"L{l}_q"], g[f"s{step}_L{l}_q"]) for l in range(1, snap["nlev"] + 1)):
            break
