"""Spill (LDL/STL) counts per source line of one kernel in a built library (tools only).
    python tools/spills.py LIB.so KERNEL_SUBSTRING SRC_BASENAME"""
import glob, os, re, subprocess, sys, tempfile, collections
lib, kname, srcname = os.path.abspath(sys.argv[1]), sys.argv[2], sys.argv[3]
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", lib], cwd=tmp, capture_output=True)
src = {}
for f in glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "paper_2304_09590_b200", "csrc", srcname)):
    src = dict(enumerate(open(f).read().split("\n"), 1))
for cub in glob.glob(os.path.join(tmp, "*.cubin")):
    dis = subprocess.run(["nvdisasm", "--print-line-info-inline", cub], capture_output=True, text=True).stdout
    fn, cur, cnt = None, None, collections.Counter()
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
        if re.search(r"\b(STL|LDL)\b", l):
            cnt[(cur, "STL" if "STL" in l else "LDL")] += 1
        if re.search(r"\bEXIT\b", l) and cnt:
            pass
    if cnt:
        print(fn[:90])
        for (ln, k), v in sorted(cnt.items(), key=lambda kv: (kv[0][0] or 0)):
            print(f"  {ln} {k} {v}  {src.get(ln, '').strip()[:80]}")
        break
