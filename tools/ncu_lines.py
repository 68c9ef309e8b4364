"""Per-source-line instruction counts and stall samples of one kernel in an ncu report,
by mapping the report's SASS addresses (relative to the function start) to CUDA lines
with nvdisasm's line table of the same cubin (tools only).

    python tools/ncu_lines.py REP.ncu-rep LIB.so KERNEL_SUBSTRING SRC_BASENAME [units]
units: divide instruction counts by this (e.g. warps x samples) for per-unit numbers.
"""
import collections
import csv
import glob
import io
import os
import re
import subprocess
import sys
import tempfile

rep, lib, kname, srcname = sys.argv[1:5]
lib = os.path.abspath(lib)
units = float(sys.argv[5]) if len(sys.argv) > 5 else 1.0
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[hi]
ix = {h: i for i, h in enumerate(hdr)}
prof = []
for r in rows[hi + 1:]:
    if len(r) < len(hdr):
        continue
    prof.append((int(r[0], 16), r[ix["Source"]], float(r[ix["Instructions Executed"]] or 0),
                 float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)))
base = prof[0][0]
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=tmp, capture_output=True)
line_of = {}
for cub in glob.glob(os.path.join(tmp, "*.cubin")):
    dis = subprocess.run(["nvdisasm", "--print-line-info-inline", cub], capture_output=True, text=True).stdout
    fn, cur = None, None
    for l in dis.split("\n"):
        m = re.match(r"\s*\.text\.(\S+):", l)
        if m:
            fn = m.group(1)
            continue
        if fn is None or kname not in fn:
            continue
        m = re.search(srcname + r'", line (\d+)', l)
        if m:
            cur = int(m.group(1))
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(\S.*?);", l)
        if m and cur is not None:
            line_of.setdefault(fn, {})[int(m.group(1), 16)] = (cur, m.group(2))
# pick the function whose instruction sequence matches the profile
best = None
for fn, mp in line_of.items():
    ok = sum(1 for a, s, _, _ in prof[:200] if (a - base) in mp and mp[a - base][1].split()[0] in s)
    if best is None or ok > best[0]:
        best = (ok, fn)
mp = line_of[best[1]]
agg = collections.defaultdict(lambda: [0.0, 0.0])
for a, s, ie, st in prof:
    ln = mp.get(a - base, (None, ""))[0]
    agg[ln][0] += ie
    agg[ln][1] += st
srcl = {}
for f in glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2304_09590_b200", "csrc", srcname)):
    srcl = dict(enumerate(open(f).read().split("\n"), 1))
tot_i = sum(v[0] for v in agg.values())
tot_s = sum(v[1] for v in agg.values())
print(f"function {best[1]} (matched {best[0]}/200); instructions {tot_i / units:.1f} per unit, stall samples {tot_s:.0f}")
for ln, (ie, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:50]:
    print(f"{str(ln):>5} {ie / units:8.1f} {st / tot_s * 100:5.1f}%  {srcl.get(ln, '').strip()[:90]}")
