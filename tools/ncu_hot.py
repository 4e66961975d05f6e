"""Summarise an ncu source page (SASS): hottest instructions by stall samples."""
import csv, io, subprocess, sys
rep = sys.argv[1]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.reader(io.StringIO("\n".join(lines[start:]))))
hdr = rows[0]; rows = rows[1:]
ia, isrc, iss, iex = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
tot = sum(int(r[iss] or 0) for r in rows)
print("total samples", tot, "instructions", len(rows))
mode = sys.argv[3] if len(sys.argv) > 3 else "hot"
if mode == "hot":
    for r in sorted(rows, key=lambda r: -int(r[iss] or 0))[:n]:
        print(f"{int(r[iss] or 0):7d} {int(r[iex] or 0):9d}  {r[ia][-5:]}  {r[isrc].strip()[:90]}")
else:
    lo, hi = int(sys.argv[4], 16), int(sys.argv[5], 16)
    for r in rows:
        a = int(r[ia], 16) & 0xfffff
        if lo <= a <= hi:
            print(f"{int(r[iss] or 0):7d} {int(r[iex] or 0):9d}  {r[ia][-5:]}  {r[isrc].strip()[:100]}")
