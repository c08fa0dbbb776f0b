"""Registers / stack bytes of every k1_fast instantiation in an object or library:
<SYS FORM REV LIM CFL RST PFILL> -> REG, STACK (cuobjdump -res-usage)."""
import re, subprocess, sys
out = subprocess.run(["cuobjdump", "-res-usage", sys.argv[1]], capture_output=True, text=True).stdout
lines = out.splitlines()
for i, l in enumerate(lines):
    m = re.search(r"Function (\S*k1_fast(2?)I(\S*)E\S*v11AdjStepArgs)", l)
    if m and i + 1 < len(lines):
        args = re.findall(r"L([ib])(\d+)E", m.group(3))
        r = re.search(r"REG:(\d+) STACK:(\d+)", lines[i + 1])
        print("k1_fast" + m.group(2), " ".join(v for _, v in args), "REG", r.group(1), "STACK", r.group(2))
