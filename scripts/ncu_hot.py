"""Top SASS instructions by warp-stall samples from an ncu report (source page)."""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = next(i for i, r in enumerate(rows) if "Source" in r and "# Samples" in r)
hdr = rows[h]
si, src, ie = hdr.index("# Samples"), hdr.index("Source"), hdr.index("Instructions Executed")
body = [r for r in rows[h + 1:] if len(r) > si]
tot = sum(int(r[si] or 0) for r in body)
print("total samples", tot, "instructions", sum(int(r[ie] or 0) for r in body))
for k, r in sorted(enumerate(body), key=lambda kr: -int(kr[1][si] or 0))[:top]:
    print(f"{k:5d} {int(r[si] or 0):7d} {int(r[ie] or 0):11d}  {r[src].strip()[:90]}")
