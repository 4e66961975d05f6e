"""Per-source-line executed instructions of one kernel: ncu source page (SASS
addresses + 'Instructions Executed') joined with nvdisasm -g line info.
usage: python tools/sass_lines.py REPORT.ncu-rep OBJ.o KERNEL_SYMBOL_SUBSTR UNITS [top]"""
import csv, collections, io, re, subprocess, sys, tempfile, os
rep, obj, sym, units = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
cubin = [os.path.join(d, f) for f in os.listdir(d) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout.split("\n")
sec = None; cur = "?"; a2l = {}
for l in dis:
    if l.strip().startswith(".section") and ".text." in l:
        sec = sym in l
        continue
    if not sec:
        continue
    if "//##" in l:
        m = re.search(r'File "([^"]+)", line (\d+)', l)
        if m: cur = m.group(1).split("/")[-1] + ":" + m.group(2)
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if m: a2l[int(m.group(1), 16)] = cur
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hi = [i for i, r in enumerate(rows) if "Instructions Executed" in r][0]
hdr = rows[hi]; ie = hdr.index("Instructions Executed")
data = [(int(r[0], 16), int(r[ie] or 0)) for r in rows[hi + 1:] if len(r) == len(hdr) and r[ie].isdigit()]
base = data[0][0]
per = collections.Counter()
for a, n in data: per[a2l.get(a - base, "?")] += n
tot = sum(per.values())
print(f"{tot / units:.1f} instructions per unit")
srcs = {}
for k, v in per.most_common(top):
    f, _, ln = k.partition(":")
    txt = ""
    for root in ("paper_2201_05024_b200/csrc",):
        pth = os.path.join(root, f)
        if os.path.exists(pth):
            srcs.setdefault(pth, open(pth).read().split("\n"))
            txt = srcs[pth][int(ln) - 1].strip()[:80]
    print(f"{v / units:7.1f}  {k:24s} {txt}")
