import json
import sys

for line in open(sys.argv[1]):
    try:
        d = json.loads(line)
    except Exception:
        print(line[:300])
        continue
    print(d["cfg"], [(k, round(v, 3)) for k, v in d["times_ms"]])
    print("    ", {k: round(v, 3) for k, v in d["per_vertex"].items()})
