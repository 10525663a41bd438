"""Build variant libraries for A/B timing: ab_build.py NAME:DEF1,DEF2 ...  ->  ab/libmt_NAME.so
(run them with MT_LIBRARY=ab/libmt_NAME.so python scripts/stats.py c5)."""
import os
import sys
from concurrent.futures import ThreadPoolExecutor

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2301_10838_b200 import build as B

root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.makedirs(os.path.join(root, "ab"), exist_ok=True)


def one(spec):
    name, _, defs = spec.partition(":")
    out = os.path.join(root, "ab", f"libmt_{name}.so")
    return B.build(defines=[d for d in defs.split(",") if d], out=out)


with ThreadPoolExecutor(4) as ex:
    for p in ex.map(one, sys.argv[1:]):
        print(p)
