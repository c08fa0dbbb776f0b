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
    for key, gp in pl._gather.items():
        meta = gp.meta[:gp.n].cpu().numpy()
        nphys_coarse = int(((meta & 1) != 0).sum()) - gp.nc
        print(f"L{lev}: patches {len(h.patches(lev))} ghost entries {gp.n} coarse rect cells {gp.nc} "
              f"physical mirroring coarse {nphys_coarse} copy+physical {gp.n - gp.nc - nphys_coarse}")
