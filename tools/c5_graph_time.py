"""C5: graph replay time per coarse step (the bench's number) and an eager
run, for comparison with a warm-cache ncu launch list of the same command."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1511_03645_b200 import _lib, amr
h, eq, ctx, dt = bench.build_c5(_lib.VARIANT_FAST)
for _ in range(4):
    amr.advance_hierarchy(h, 1, dt, ctx)
g = amr.SweepGraph(h, dt, ctx)
g.advance(2)
torch.cuda.synchronize()
if os.environ.get("NCU_ONE"):
    g.advance(2)
    torch.cuda.synchronize()
    sys.exit(0)
for rep in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.advance(10); e1.record(); torch.cuda.synchronize()
    print("graph ms/coarse step", e0.elapsed_time(e1) / 10)
