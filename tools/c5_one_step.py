import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1511_03645_b200 import _lib, amr
h, eq, ctx, dt = bench.build_c5(_lib.VARIANT_FAST)
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
    amr.advance_hierarchy(h, 1, dt, ctx)
torch.cuda.synchronize()
print("ok")
