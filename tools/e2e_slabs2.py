"""e2e C4 chained steps (step_patch_host(wait=False)) over slab counts."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1511_03645_b200 import solver
h, p, eq, bc, dt = bench.build_c4(4096)
st = solver.store_of(p)
st.sync_in()
host = torch.empty(tuple(st.view(p._slot).shape), dtype=torch.float64, pin_memory=True)
host.copy_(st.view(p._slot))
for slabs in (2, 3, 4, 6, 8, 12, 16):
    solver.step_patch_host(p, host, dt, eq, bc, (4096, 4096), "MC", slabs=slabs)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        solver.step_patch_host(p, host, dt, eq, bc, (4096, 4096), "MC", slabs=slabs, wait=False)
    solver.host_stream_finish(p)
    el = (time.perf_counter() - t0) / 10
    print("slabs", slabs, "ms", round(el * 1e3, 2), "G/s", round(4096 * 4096 / el / 1e9, 3), flush=True)
