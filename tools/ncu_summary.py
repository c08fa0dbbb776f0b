"""Summarise ncu reports / launch lists into text for profiles/ (run in the
build container on files brought back in gpurun_out/)."""
import collections
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "sm__cycles_elapsed.avg.per_second"]


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units, vals = rows[0], rows[1], rows[2]
    lines = [f"# {path}", f"kernel: {vals[hdr.index('Kernel Name')]}"]
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            lines.append(f"{k:62s} {vals[i]:>20s} {units[i]}")
    stalls = [(h, vals[i]) for i, h in enumerate(hdr) if h.startswith("smsp__pcsamp_warps_issue_stalled_")
              and not h.endswith("not_issued")]
    stalls = sorted(((h.split("stalled_")[1], float(v.replace(",", "") or 0)) for h, v in stalls), key=lambda x: -x[1])
    tot = sum(v for _, v in stalls) or 1
    lines.append("stall samples (share): " + ", ".join(f"{h} {100 * v / tot:.1f}%" for h, v in stalls[:8]))
    return "\n".join(lines)


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr, data = rows[0], rows[1:]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in data:
        name = r[ki].split("(")[0]
        v = float(r[vi].replace(",", ""))
        v *= {"msecond": 1e6, "usecond": 1e3, "nsecond": 1.0}.get(r[ui], 1.0)
        tot[name] += v
        cnt[name] += 1
    T = sum(tot.values())
    lines = [f"# launch list {path}: {len(data)} launches, {T / 1e6:.3f} ms total (cold-cache, serialised)"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        lines.append(f"{k[:70]:70s} n={cnt[k]:5d} total={v / 1e6:9.3f} ms share={100 * v / T:5.1f}% avg={v / cnt[k] / 1e3:9.2f} us")
    return "\n".join(lines)


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(launches(p) if p.endswith(".csv") else report(p))
        print()
