"""Per-source-line warp-stall samples and executed instructions from an ncu report."""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, res, hdr = None, [], None
for r in rows:
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0]:
        try:
            res.append((int(r[6] or 0), int(r[7] or 0), float(r[10] or 0), f"{fname}:{r[0]}", r[1].strip()[:80]))
        except (ValueError, IndexError):
            pass
tot = sum(x[0] for x in res)
print("total samples", tot)
for s, ie, thr, loc, src in sorted(res, reverse=True)[:top]:
    print(f"{s:8d} {100.0 * s / max(tot, 1):5.1f}% {ie:11d} thr{thr:5.1f}  {loc:22s} {src}")
