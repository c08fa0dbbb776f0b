"""Per-kernel totals over the last N launches of my library in an ncu launch-list CSV."""
import collections, csv, sys
path, per = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 2
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
hdr, data = rows[0], rows[1:]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
U = {'msecond': 1e3, 'usecond': 1, 'nsecond': 1e-3, 'ms': 1e3, 'us': 1, 'ns': 1e-3}
seq = [(r[ki].split('(')[0][-34:], float(r[vi].replace(',', '')) * U[r[ui]]) for r in data]
mine = [x for x in seq if 'at::' not in x[0]]
n = int(sys.argv[3]) if len(sys.argv) > 3 else len(mine) // 4
tail = mine[-n:]
t = collections.defaultdict(float); c = collections.Counter()
for k, v in tail:
    t[k] += v; c[k] += 1
for k in sorted(t, key=lambda k: -t[k]):
    print(f"{k:36s} n={c[k]:3d} per-unit={t[k] / per:8.1f} us avg={t[k] / c[k]:6.2f}")
print('sum per unit', round(sum(t.values()) / per, 1), 'launches per unit', len(tail) / per)
