"""C5: the captured sweep with level overlap (parent steps on side streams)
against the sequential capture -- bitwise equal states after N coarse steps,
and the replay time per coarse step of each (ADJAMR_LEVEL_OVERLAP switch)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_1511_03645_b200 import _lib, amr

STEPS = int(os.environ.get("C5_STEPS", "20"))


def run(overlap):
    amr.USE_LEVEL_OVERLAP = overlap
    h, eq, ctx, dt = bench.build_c5(_lib.VARIANT_FAST)
    for _ in range(4):
        amr.advance_hierarchy(h, 1, dt, ctx)
    g = amr.SweepGraph(h, dt, ctx)
    g.advance(2)
    torch.cuda.synchronize()
    ts = []
    for rep in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.advance(STEPS); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / STEPS)
    states = []
    for lev in range(1, h.num_levels() + 1):
        st = amr._plan(h, lev).st
        states.append(st.buf[st.cur].clone())
    print(f"overlap={overlap}: graph ms/coarse step", " ".join(f"{t:.4f}" for t in ts),
          "skip slots", g.skip_slots, "sequential replays", g.seq_replays, flush=True)
    del g
    return states, dict(ctx.cell_steps)


a, ca = run(False)
b, cb = run(True)
same = all(torch.equal(x, y) for x, y in zip(a, b))
print("bitwise equal:", same, "cell_steps equal:", ca == cb)
if not same:
    for lev, (x, y) in enumerate(zip(a, b), start=1):
        d = (x - y).abs()
        print(f"level {lev}: {int((d > 0).sum())} differing, max {float(d.max()):.3e}")
    sys.exit(1)
