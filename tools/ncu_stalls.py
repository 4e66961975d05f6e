"""Per-region stall breakdown from an ncu source page: groups SASS instructions by
their execution count bucket (e.g. the per-step critical path has count == steps*CTAs)."""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
hdr = rows[0]; rows = rows[1:]
st = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
iex = hdr.index("Instructions Executed"); ia = hdr.index("Address"); isrc = hdr.index("Source")
lo = int(sys.argv[2], 16) if len(sys.argv) > 2 else 0
hi = int(sys.argv[3], 16) if len(sys.argv) > 3 else 1 << 40
agg = collections.Counter(); n = 0; ex = 0
for r in rows:
    a = int(r[ia], 16) & 0xfffff
    if lo <= a <= hi:
        n += 1; ex += int(r[iex] or 0)
        for i in st:
            agg[hdr[i]] += int(r[i] or 0)
print(f"range {lo:x}-{hi:x}: {n} instrs, executed {ex}")
for k, v in agg.most_common(12):
    print(f"  {k:28s} {v}")
