"""Aggregate an ncu source page (SASS) by opcode: executed warp instructions
and stall samples.  usage: ncu_sass_stats.py report.ncu-rep [kernel-regex]"""
import collections
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"]
if len(sys.argv) > 2:
    cmd += ["-k", "regex:" + sys.argv[2]]
out = subprocess.run(cmd, capture_output=True, text=True).stdout
lines = [l for l in out.splitlines() if l.startswith('"0x') or l.startswith('"Address"')]
rows = list(csv.reader(io.StringIO("\n".join(lines))))
hdr, rows = rows[0], rows[1:]
ci = {h: i for i, h in enumerate(hdr)}
ex = collections.Counter()
st = collections.Counter()
tot_ex = tot_st = 0
for r in rows:
    src = r[ci["Source"]].strip()
    op = re.sub(r"^@!?U?P\w+\s+", "", src).split()[0] if src else "?"
    op = op.split(".")[0]
    n = int(r[ci["Instructions Executed"]] or 0)
    s = int(r[ci["Warp Stall Sampling (All Samples)"]] or 0)
    ex[op] += n
    st[op] += s
    tot_ex += n
    tot_st += s
print(f"warp instructions executed {tot_ex}, stall samples {tot_st}")
for op, n in ex.most_common(30):
    print(f"{op:10s} exec {n:12d} ({100 * n / tot_ex:5.1f}%)  samples {st[op]:8d} ({100 * st[op] / max(tot_st, 1):5.1f}%)")
