"""Reader for tests/golden/*.txt fixtures (hand-derived, each with its citation)."""
import glob
import os

import numpy as np

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _ints(s):
    return [tuple(int(x) for x in part.split()) for part in s.split(";") if part.strip()]


def load(path):
    d = {}
    with open(path) as fh:
        for line in fh:
            line = line.rstrip("\n")
            if not line or line.startswith("#"):
                continue
            k, _, v = line.partition(":")
            d[k.strip()] = v.strip()
    dims = tuple(int(x) for x in d["dims"].split())
    f = np.array([float(x) for x in d["f"].split()], dtype=np.float32)
    return dict(
        name=os.path.basename(path),
        dims=dims,
        conn=int(d["conn"]),
        split=bool(int(d["split"])),
        f=f,
        triplets=_ints(d["triplets"]),
        pairs=_ints(d.get("pairs", "")),
        essential=[int(x) for x in d.get("essential", "").split()],
    )


def all_cases():
    return [load(p) for p in sorted(glob.glob(os.path.join(GOLDEN_DIR, "*.txt")))]
