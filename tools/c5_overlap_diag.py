"""Where the overlapped capture first differs from the sequential one: one
replayed pair, states per level; overlap limited to levels <= maxlev."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1511_03645_b200 import _lib, amr


def run(overlap, maxlev=99, pairs=1):
    amr.USE_LEVEL_OVERLAP = overlap
    amr._OVERLAP_MAX_LEVEL = maxlev
    h, eq, ctx, dt = bench.build_c5(_lib.VARIANT_FAST)
    for _ in range(2):
        amr.advance_hierarchy(h, 1, dt, ctx)
    g = amr.SweepGraph(h, dt, ctx)      # replays the captured pair once
    torch.cuda.synchronize()
    print("capture slots", ["%.3g" % v for v in g.params.vals])
    for k in range(4):
        g._shadow_pair()
        print("pair", k, "slots", ["%.3g" % v for v in g.params.vals])
    if pairs > 1:
        g.advance(2 * (pairs - 1)); torch.cuda.synchronize()
    out = []
    for lev in range(1, h.num_levels() + 1):
        st = amr._plan(h, lev).st
        out.append((st.buf[st.cur].clone(), st.cur, st.old, st.ghost_src))
    return out


def cmp(tag, a, b):
    msg = []
    for lev, (x, y) in enumerate(zip(a, b), start=1):
        d = (x[0] - y[0]).abs()
        msg.append(f"L{lev}: {int((d > 0).sum())} diff max {float(d.max()):.2e} roles {x[1:]} {y[1:]}")
    print(tag, " | ".join(msg), flush=True)


ref = run(False)
cmp("seq vs seq", ref, run(False))
cmp("ov vs seq ", run(True), ref)
cmp("ov vs ov  ", run(True), run(True))
cmp("ov L1 only", run(True, 1), ref)
