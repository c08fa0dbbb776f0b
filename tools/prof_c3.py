import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1511_03645_b200 import _lib, device, solver
h, p, eq, bc, dt = bench.build_c3(2048)
st = solver.store_of(p)
solver.advance_uniform(p, eq, bc, (2048, 2048), dt, 2, "MC", _lib.VARIANT_FAST, graph=False)
torch.cuda.synchronize()
ts = []
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    out = st._free(st.cur, -1)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    device.launch_step(st, dt, eq, "MC", _lib.VARIANT_FAST, out,
                       phys_in=(bc, eq, (2048, 2048)) if "physin" in sys.argv else None)   # physin: the bench's launch
    b.record()
    st.ghost_src = st.cur; st.cur = out
    ts.append((a, b))
torch.cuda.synchronize()
print("k1 ms", [round(a.elapsed_time(b), 4) for a, b in ts])
if len(sys.argv) > 2 and sys.argv[2] == "flag":      # the C3 flagging launch (k3_direct), as bench_c3 runs it
    import numpy as np
    from paper_1511_03645_b200 import adjoint
    ring = bench.adjoint_ring_c3(50, 2048)
    T = 200 * dt
    idx = adjoint.window_indices(100 * dt, adjoint.TimeWindow(0.0, T), np.linspace(0.0, T, 50))
    device.launch_flag(st, ring, (2048, 2048), (0.0, 0.0), 1.0 / 2048, 1.0 / 2048, (0.0, 0.0), 1.0 / 2048,
                       1.0 / 2048, idx, 0.05)
    torch.cuda.synchronize()
    print("flag ok", len(idx))
