"""Instruction mix per column of K1's inner march loop (the backward-branch body with the
cp.async prefetches; three columns per cp.async wait, so columns = 3 x its DEPBAR count)."""
import collections, re, subprocess, sys
lib, pat = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs = re.split(r"\n\s+Function : ", out)
body = next(f for f in funcs if re.match(r"\S*" + pat, f))
ins = []
for l in body.splitlines():
    m = re.match(r"\s+/\*([0-9a-f]+)\*/\s+(.*?);", l)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
loops = []
for a, t in ins:
    m = re.search(r"BRA (?:\S+ )?0x([0-9a-f]+)", t)
    if m and int(m.group(1), 16) < a:
        loops.append((int(m.group(1), 16), a))
# inner march loop: backward-branch body with the cp.async prefetches (LDGSTS), no divergent fallback
def body_of(l):
    return [t for a, t in ins if l[0] <= a <= l[1]]
cands = [l for l in loops if any("LDGSTS" in t for t in body_of(l)) and not any("WARPSYNC" in t for t in body_of(l))]
lo, hi = min(cands, key=lambda l: l[1] - l[0])
loop = [t for a, t in ins if lo <= a <= hi]
ncol = 3 * max(1, sum(1 for t in loop if t.startswith("DEPBAR")))
ops = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", t).split()[0] for t in loop)
base = collections.Counter()
for k, v in ops.items():
    base[k.split(".")[0] if not k.startswith("IMAD.MOV") else "IMAD.MOV"] += v
fp64 = sum(base[k] for k in ("DADD", "DMUL", "DFMA", "DSETP"))
loc = sum(v for k, v in ops.items() if k.startswith(("LDL", "STL")))
print(f"loop {hex(lo)}-{hex(hi)} ({ncol} columns): {len(loop) / ncol:.1f} instr/column, FP64 {fp64 / ncol:.1f}/column, "
      f"local ld/st {loc}")
print(", ".join(f"{k} {v / ncol:.1f}" for k, v in base.most_common(16)))
