"""C5: per-level ghost plan sizes (entries, coarse-interpolated entries) and patch counts."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1511_03645_b200 import _lib, amr
h, eq, ctx, dt = bench.build_c5(_lib.VARIANT_FAST)
for _ in range(2):
    amr.advance_hierarchy(h, 1, dt, ctx)
torch.cuda.synchronize()
for lev in range(1, h.num_levels() + 1):
    pl = amr._plan(h, lev)
    gp = getattr(pl, "gplan", None) or getattr(pl, "plan", None)
    print(lev, len(h.patches(lev)), {k: getattr(v, "n", None) for k, v in vars(pl).items() if hasattr(v, "nc")},
          {k: getattr(v, "nc", None) for k, v in vars(pl).items() if hasattr(v, "nc")})
