import cProfile, io, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1511_03645_b200 import _lib, amr, device
h, eq, ctx, dt = bench.build_c5(_lib.VARIANT_FAST)
for _ in range(2):
    amr.advance_hierarchy(h, 1, dt, ctx)
g = amr.SweepGraph(h, dt, ctx)
g.advance(2)
torch.cuda.synchronize()
# pure replay time (no shadow): GPU-side cost of a pair
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    g.graph.replay()
e1.record(); torch.cuda.synchronize()
print("pure replay ms per coarse step", e0.elapsed_time(e1) / 20)
pr = cProfile.Profile()
t = time.perf_counter()
pr.enable()
g.advance(10)
pr.disable()
torch.cuda.synchronize()
print("advance(10) wall ms per coarse step", (time.perf_counter() - t) * 100)
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(35)
print(s.getvalue())
