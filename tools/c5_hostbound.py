"""C5: is the graph-replayed sweep host-bound?  Device time of g.advance(N)
vs host wall time, raw back-to-back graph replays (no shadow orchestration:
device time only), and the shadow orchestration alone (host time)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1511_03645_b200 import _lib, amr, device
h, eq, ctx, dt = bench.build_c5(_lib.VARIANT_FAST)
for _ in range(4):
    amr.advance_hierarchy(h, 1, dt, ctx)
g = amr.SweepGraph(h, dt, ctx)
g.advance(2)
torch.cuda.synchronize()
for n in (2, 10, 20):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w = time.perf_counter(); e0.record(); g.advance(n); e1.record(); torch.cuda.synchronize()
    print(f"advance({n}): device {e0.elapsed_time(e1) / n:.4f} ms/coarse, host wall {(time.perf_counter() - w) * 1e3 / n:.4f}")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    g.graph.replay()
e1.record(); torch.cuda.synchronize()
print(f"raw replays: device {e0.elapsed_time(e1) / 20:.4f} ms/coarse")
w = time.perf_counter()
for _ in range(10):
    device.SHADOW = True; device.PARAMS = g.params; g.params.rewind(); ctx._defer_checks = True
    for _ in range(2):
        amr.advance_hierarchy(h, 1, dt, ctx)
    device.SHADOW = False; device.PARAMS = None; ctx._defer_checks = False
    g.params.upload()
print(f"shadow only: host {(time.perf_counter() - w) * 1e3 / 20:.4f} ms/coarse")
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for _ in range(5):
    device.SHADOW = True; device.PARAMS = g.params; g.params.rewind(); ctx._defer_checks = True
    for _ in range(2):
        amr.advance_hierarchy(h, 1, dt, ctx)
    device.SHADOW = False; device.PARAMS = None; ctx._defer_checks = False
    g.params.upload()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
