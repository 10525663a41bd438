"""Summarise gpurun_out/<tag>_ab.log: per variant, per config, kernel times (ms)."""
import json
import sys

lib = None
for line in open(sys.argv[1]):
    if line.startswith("== "):
        lib = line[3:].strip().split("libmt_")[-1].replace(".so", "")
        continue
    try:
        d = json.loads(line)
    except ValueError:
        print(lib, line.strip()[:200])
        continue
    t = dict(d["times_ms"])
    tot = sum(t.values())
    print(f"{lib:>10} {d['cfg']} pairs={d['pairs']} total={tot:8.2f} " +
          " ".join(f"{k}={v:.2f}" for k, v in t.items() if v > 0.05))
