import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from tests.test_gpu_stream import _patch
from paper_1511_03645_b200 import _lib, solver
sides = ("wall", "outflow", "outflow", "wall")
shape = (301, 263)
h, p, eq, bc, dt = _patch("swe", *shape, sides)
start = np.array(p.state, copy=True)
st = solver.store_of(p)
print("tiles (device path):", st.tiles(_lib.VARIANT_FAST)[1:2], "strip len", st._strip_length(128, 28))
solver.fill_ghost_physical(p, bc, eq, shape)
solver.step_patch(p, dt, eq, "MC", variant=_lib.VARIANT_FAST)
want = np.array(p.state, copy=True)
h2, p2, eq2, bc2, dt2 = _patch("swe", *shape, sides)
host = torch.from_numpy(start.copy()).pin_memory()
solver.step_patch_host(p2, host, dt, eq2, bc2, shape, "MC", slabs=1)
got = host.numpy()
d = np.abs(got - want)
idx = np.argwhere(d > 0)
print("ndiff", len(idx), "max", d.max())
for c in range(3):
    ii = idx[idx[:, 0] == c]
    if len(ii):
        print("comp", c, "rows", np.unique(ii[:, 1])[:20], "cols", np.unique(ii[:, 2])[:40])
