"""cProfile of the host work of creating one regridded level: make_patches
(material sampling) and LevelStore construction, on ~300 patches of mixed
shapes like a C5 L3 regrid."""
import cProfile, io, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_1511_03645_b200 import _lib, amr, device

h, eq, ctx, dt = bench.build_c5(_lib.VARIANT_FAST)
rng = np.random.default_rng(0)
boxes = []
for k in range(300):
    lo = rng.integers(0, 3900, 2) // 4 * 4
    sh = rng.integers(2, 17, 2) * 4
    boxes.append((tuple(int(v) for v in lo), tuple(int(a + b - 1) for a, b in zip(lo, sh))))
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ps = amr.make_patches(h, 3, boxes, ctx, 0.0)
    t1 = time.perf_counter()
    st = device.LevelStore(ps)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"make_patches {1e3 * (t1 - t0):.2f} ms  LevelStore {1e3 * (t2 - t1):.2f} ms")
pr = cProfile.Profile()
pr.enable()
for rep in range(3):
    ps = amr.make_patches(h, 3, boxes, ctx, 0.0)
    st = device.LevelStore(ps)
torch.cuda.synchronize()
pr.disable()
s = io.StringIO()
pstats.Stats(pr, stream=s).sort_stats("tottime").print_stats(25)
print(s.getvalue()[:7000])
