"""Summarise an ncu report: key metrics + the hottest SASS lines.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--top 30]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 30
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(det)))
hdr = rows[0]
keep = ("Duration", "Elapsed Cycles", "SM Frequency", "Executed Ipc Active", "Issue Slots Busy",
        "Registers Per Thread", "Achieved Active Warps Per SM", "Executed Instructions", "DRAM Throughput",
        "L1/TEX Cache Throughput", "Compute (SM) Throughput", "Max Active Clusters", "No Eligible",
        "Warp Cycles Per Issued Instruction", "Memory Throughput")
for r in rows[1:]:
    d = dict(zip(hdr, r))
    if d.get("Metric Name") in keep:
        print(f"{d['Metric Name']:40s} {d['Metric Value']} {d['Metric Unit']}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = rows[2:]


def f(r, k):
    try:
        return float(r[ix[k]])
    except Exception:
        return 0.0


tot = sum(f(r, "Instructions Executed") for r in data)
samp = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data)
print(f"instructions executed {tot:.0f}, stall samples {samp:.0f}")
print("--- hottest by stall samples (addr, sass, executed, samples)")
for r in sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:top]:
    print(r[0][-5:], r[1][:64].ljust(64), int(f(r, "Instructions Executed")),
          int(f(r, "Warp Stall Sampling (All Samples)")))

if "--exec" in sys.argv:   # list lines executed exactly N times, in address order (e.g. the tail warp)
    n = float(sys.argv[sys.argv.index("--exec") + 1])
    sel = [r for r in data if abs(f(r, "Instructions Executed") - n) <= 0.02 * n]
    print(f"--- {len(sel)} lines executed ~{n:.0f} times; stall samples {sum(f(r, 'Warp Stall Sampling (All Samples)') for r in sel):.0f}")
    for r in sel:
        print(r[0][-5:], r[1][:70].ljust(70), int(f(r, "Warp Stall Sampling (All Samples)")))

if "--range" in sys.argv:   # all lines whose address suffix lies in [lo, hi] (hex, last 5 digits)
    lo, hi = (int(v, 16) for v in sys.argv[sys.argv.index("--range") + 1].split(":"))
    for r in data:
        a = int(r[0][-5:], 16)
        if lo <= a <= hi:
            print(r[0][-5:], r[1][:70].ljust(70), int(f(r, "Instructions Executed")),
                  int(f(r, "Warp Stall Sampling (All Samples)")))
