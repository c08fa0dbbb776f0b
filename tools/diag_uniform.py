import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1511_03645_b200 import _lib, solver
h, p, eq, bc, dt = bench.build_c4()
st = solver.store_of(p)
for n in (5, 20, 20, 20, 21, 20):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = time.perf_counter()
    e0.record()
    solver.advance_uniform(p, eq, bc, (bench.N, bench.N), dt, n, "MC", _lib.VARIANT_FAST)
    e1.record(); torch.cuda.synchronize()
    print(n, "ms/step", e0.elapsed_time(e1) / n, "host ms/step", (time.perf_counter() - t) * 1e3 / n,
          "graphs", [k[-1] for k in st._scratch if isinstance(k, tuple) and k and k[0] == "uniform_graph"])
for n in (20,):
    torch.cuda.synchronize()
    e0.record()
    solver.advance_uniform(p, eq, bc, (bench.N, bench.N), dt, n, "MC", _lib.VARIANT_FAST, graph=False)
    e1.record(); torch.cuda.synchronize()
    print("eager", n, "ms/step", e0.elapsed_time(e1) / n)
