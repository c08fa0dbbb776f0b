import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1511_03645_b200 import _lib, amr
from tests.test_gpu_graph import small_hierarchy

def cmp(ha, hb, tag):
    for lev in (1, 2, 3):
        d = [float(np.max(np.abs(pa.interior() - pb.interior()))) for pa, pb in zip(ha.patches(lev), hb.patches(lev))]
        print(tag, "lev", lev, "maxdiff", max(d), "npatch_diff", sum(x > 0 for x in d), "t", ha.patches(lev)[0].time, hb.patches(lev)[0].time)

# eager vs eager
ha, ca, dt = small_hierarchy(_lib.VARIANT_FAST)
hb, cb, _ = small_hierarchy(_lib.VARIANT_FAST)
for _ in range(4):
    amr.advance_hierarchy(ha, 1, dt, ca)
    amr.advance_hierarchy(hb, 1, dt, cb)
cmp(ha, hb, "eager/eager")
# graph: warmup 2 + capture 2 (replayed once) == 4 steps
ha, ca, dt = small_hierarchy(_lib.VARIANT_FAST)
hb, cb, _ = small_hierarchy(_lib.VARIANT_FAST)
for _ in range(4):
    amr.advance_hierarchy(ha, 1, dt, ca)
g = amr.SweepGraph(hb, dt, cb)
cmp(ha, hb, "after capture (4 steps)")
for _ in range(2):
    amr.advance_hierarchy(ha, 1, dt, ca)
g.advance(2)
cmp(ha, hb, "after 1 replay pair (6 steps)")
print("slots", len(g.params.vals), g.params.vals[:12])
