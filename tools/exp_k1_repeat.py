"""Experiment: C5's finest level, R K1 launches vs one launch of R concatenated
job tables (same work, no fills, results not meaningful) -- the cost of the
kernel boundaries and per-launch tails of small-patch levels."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
from paper_1511_03645_b200 import _lib, amr, device

h, eq, ctx, dt = bench.build_c5(_lib.VARIANT_FAST)
for _ in range(2):
    amr.advance_hierarchy(h, 1, dt, ctx)
torch.cuda.synchronize()
FAST = _lib.VARIANT_FAST
for lev in (3, 2):
    st = amr._plan(h, lev).st
    tiles, ntile, jobs, njob = st.tiles(FAST)
    rows = np.frombuffer(tiles.cpu().numpy().tobytes(), dtype=_lib.TILE_DTYPE)[:ntile].copy()
    offs = jobs.cpu().numpy().astype(np.int64)
    out = st._free(st.cur, st.old if st.old is not None else -1)
    dtl = dt / (h.ratio_to_finer(1) if lev == 2 else h.ratio_to_finer(1) * h.ratio_to_finer(2))

    def timed(reps_in_graph, tabs):
        saved = st._tiles[FAST]
        st._tiles[FAST] = tabs
        try:
            device.launch_step(st, dtl, eq, "MC", FAST, out, accumulate=True)
            torch.cuda.synchronize()
            side = torch.cuda.Stream()
            side.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(side):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=side):
                    for _ in range(reps_in_graph):
                        device.launch_step(st, dtl, eq, "MC", FAST, out, accumulate=True)
            torch.cuda.current_stream().wait_stream(side)
            g.replay(); torch.cuda.synchronize()
            ts = []
            for _ in range(5):
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(); g.replay(); b.record(); torch.cuda.synchronize()
                ts.append(a.elapsed_time(b))
            return sorted(ts)[2]
        finally:
            st._tiles[FAST] = saved

    for R in (1, 2, 4, 8):
        rr = np.concatenate([rows] * R)
        oo = np.concatenate([offs[:-1] + r * ntile for r in range(R)] + [np.array([R * ntile])])
        tabs = (device._dev_table(rr), len(rr), torch.from_numpy(oo.astype(np.int32)).to("cuda"), len(oo) - 1)
        one = timed(1, tabs)
        sep = timed(R, (tiles, ntile, jobs, njob))
        print(f"L{lev} R={R}: one launch of R tables {one * 1e3:8.1f} us   R launches {sep * 1e3:8.1f} us "
              f"  per-substep {one * 1e3 / R:6.1f} vs {sep * 1e3 / R:6.1f}", flush=True)
