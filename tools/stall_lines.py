"""Per-source-line warp stall samples (ncu source page) joined with nvdisasm
line info, for a line range of one file.
usage: python tools/stall_lines.py REPORT OBJ KERNEL_SUBSTR FILE LO HI"""
import csv, collections, io, os, re, subprocess, sys, tempfile
rep, obj, sym, fname, lo, hi = sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4], int(sys.argv[5]), int(sys.argv[6])
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
cubin = [os.path.join(d, f) for f in os.listdir(d) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout.split("\n")
sec = None; cur = "?"; a2l = {}; nsec = 0
for l in dis:
    if l.strip().startswith(".section") and ".text." in l:
        sec = sym in l; nsec += sec; continue
    if not sec: continue
    if "//##" in l:
        m = re.search(r'File "([^"]+)", line (\d+)', l)
        if m: cur = (m.group(1).split("/")[-1], int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if m: a2l[int(m.group(1), 16)] = cur
if nsec != 1:      # offsets are per function: several matches would mix their line maps
    sys.exit(f"{nsec} functions match {sym!r}: pass a substring of one mangled name")
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hi_ = [i for i, r in enumerate(rows) if "Instructions Executed" in r][0]
hdr = rows[hi_]
cols = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
data = [r for r in rows[hi_ + 1:] if len(r) == len(hdr)]
base = int(data[0][0], 16)
per = collections.defaultdict(collections.Counter)
for r in data:
    ln = a2l.get(int(r[0], 16) - base, ("?", 0))
    for c in cols:
        v = r[hdr.index(c)]
        if v and v.replace(".", "").isdigit(): per[ln][c] += float(v)
tot = sum(sum(c.values()) for c in per.values())
src = open(os.path.join("paper_2201_05024_b200/csrc", fname)).read().split("\n") if os.path.exists(os.path.join("paper_2201_05024_b200/csrc", fname)) else []
for (f, l), c in sorted(per.items(), key=lambda t: t[0][1] if t[0][0] == fname else 0):
    if f != fname or not lo <= l <= hi: continue
    s = sum(c.values())
    top = ", ".join(f"{k[6:]}={v:.0f}" for k, v in c.most_common(3))
    print(f"{l:5d} {100*s/tot:5.1f}%  {top:50s} {src[l-1].strip()[:60] if src else ''}")
