"""Top SASS instructions of an ncu source page by stall samples, with the
dominant stall reasons.  usage: ncu_stall_lines.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = []
for l in out.splitlines():          # first kernel of the report only
    if l.startswith('"Address"') and lines:
        break
    if l.startswith('"0x') or l.startswith('"Address"'):
        lines.append(l)
rows = list(csv.reader(io.StringIO("\n".join(lines))))
hdr, rows = rows[0], rows[1:]
ci = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = {r: 0 for r in reasons}
for r in rows:
    for k in reasons:
        tot[k] += int(r[ci[k]] or 0)
T = sum(tot.values())
print("total samples", T, ":", ", ".join(f"{k[6:]} {100 * v / T:.1f}%" for k, v in sorted(tot.items(), key=lambda x: -x[1]) if v))
rows.sort(key=lambda r: -int(r[ci["Warp Stall Sampling (All Samples)"]] or 0))
for idx, r in enumerate(rows[:top]):
    s = int(r[ci["Warp Stall Sampling (All Samples)"]] or 0)
    rs = sorted(((int(r[ci[k]] or 0), k[6:]) for k in reasons), reverse=True)[:3]
    print(f"{r[0][-5:]} {s:6d} {100 * s / T:5.1f}%  {r[1].strip()[:60]:60s} " + " ".join(f"{n}:{v}" for v, n in rs if v))
