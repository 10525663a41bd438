"""Attribute the SASS of one kernel (ncu source page, cuda+sass) to line ranges of its .cu file:
ncu_phases.py REP KERNEL FILE name:first-last ...  (warp instructions, thread instructions, samples)."""
import csv
import io
import subprocess
import sys

rep, kern, fname = sys.argv[1], sys.argv[2], sys.argv[3]
ranges = []
for spec in sys.argv[4:]:
    name, _, r = spec.partition(":")
    a, b = r.split("-")
    ranges.append((name, int(a), int(b)))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur_file, cur_line, hdr = None, None, None
acc = {}
for r in rows:
    if len(r) == 2 and r[0] in ("File Name", "File Path"):
        cur_file = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) < 9:
        continue
    if r[0]:
        cur_line = int(r[0])
        continue
    if not r[2].startswith("0x"):
        continue
    # columns: line, source, address, sass, stall (all), stall (not issued), samples, inst, thread inst
    sm, ie, ti = (int(r[i] or 0) for i in (6, 7, 8))
    key = "other:" + (cur_file or "?")
    if cur_file == fname:
        key = next((n for n, a, b in ranges if a <= cur_line <= b), f"{fname}:other")
    t = acc.setdefault(key, [0, 0, 0])
    t[0] += ie
    t[1] += ti
    t[2] += sm
tot = [sum(v[i] for v in acc.values()) for i in range(3)]
print(f"{'range':24s} {'warp inst':>14s} {'%':>6s} {'thr/inst':>8s} {'samples %':>9s}")
for k, v in sorted(acc.items(), key=lambda kv: -kv[1][2]):
    print(f"{k:24s} {v[0]:14d} {100 * v[0] / tot[0]:6.1f} {v[1] / max(v[0], 1):8.1f} {100 * v[2] / tot[2]:9.1f}")
