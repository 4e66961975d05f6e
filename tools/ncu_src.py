"""Dump an ncu source page (SASS) as rows: address, exec count, stall samples, top stall reasons, source."""
import csv, io, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
hdr = rows[0]; rows = rows[1:]
st = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
iex = hdr.index("Instructions Executed"); ia = hdr.index("Address"); isrc = hdr.index("Source")
iss = hdr.index("Warp Stall Sampling (All Samples)")
lo = int(sys.argv[2], 16) if len(sys.argv) > 2 else 0
hi = int(sys.argv[3], 16) if len(sys.argv) > 3 else 1 << 40
for r in rows:
    a = int(r[ia], 16) & 0xfffff
    if lo <= a <= hi:
        reasons = sorted(((int(r[i] or 0), hdr[i][6:]) for i in st), reverse=True)[:2]
        rs = " ".join(f"{n}:{v}" for v, n in reasons if v)
        print(f"{a:05x} {int(r[iex] or 0):7d} {int(r[iss] or 0):5d}  {r[isrc].strip()[:70]:70s} {rs}")
