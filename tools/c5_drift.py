"""C5: device / host time per coarse step over successive g.advance(10) calls (drift check)."""
import gc, os, sys, time
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
if len(sys.argv) > 1:
    gc.disable()
for rep in range(8):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    w = time.perf_counter(); e0.record(); g.advance(10); e1.record(); torch.cuda.synchronize()
    print(f"rep {rep}: device {e0.elapsed_time(e1) / 10:.4f} ms/coarse, host {(time.perf_counter() - w) * 1e2:.4f}")
    e0.record()
    for _ in range(5):
        g.graph.replay()
    e1.record(); torch.cuda.synchronize()
    print(f"       raw replay {e0.elapsed_time(e1) / 10:.4f}")
