"""Interleaved A/B of library builds in ONE process: ab_interleave.py CFG lib1.so lib2.so ...
Each round runs every library once (mt_compute + mt_diagram, per-kernel CUDA-event times via
mt_set_profiling); reports the median per kernel over the rounds, so clock drift and box
differences hit every variant alike.  Each .so is dlopen'ed privately (RTLD_LOCAL)."""
import ctypes
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2301_10838_b200 import fields

cfg, paths = sys.argv[1], sys.argv[2:]
rounds = int(os.environ.get("ROUNDS", "7"))
f, dims, conn = fields.make(cfg, device="cuda" if cfg == "c5" else "cpu")
fd = torch.from_numpy(f).cuda()
n = fd.numel()
T = torch.empty(n, dtype=torch.int64, device="cuda")
dimsc = (ctypes.c_uint32 * 3)(*dims)
vp = ctypes.c_void_p
runs = []
shared = {"ws": None}   # one workspace for all contexts: they run one after the other on one stream
for p in paths:
    L = ctypes.CDLL(os.path.abspath(p))
    L.mt_workspace_bytes.restype = ctypes.c_size_t
    L.mt_workspace_bytes.argtypes = [vp, ctypes.c_int]
    L.mt_create.argtypes = [ctypes.POINTER(vp), vp, ctypes.c_int, ctypes.c_int, vp, ctypes.c_size_t]
    L.mt_compute.argtypes = [vp, vp, vp, ctypes.c_uint32, vp]
    L.mt_diagram.argtypes = [vp, vp, ctypes.c_uint64, ctypes.POINTER(ctypes.c_uint64), ctypes.POINTER(ctypes.c_uint64), vp]
    L.mt_set_profiling.argtypes = [vp, ctypes.c_int]
    L.mt_kernel_times.argtypes = [vp, ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(ctypes.c_float), ctypes.c_int]
    nb = L.mt_workspace_bytes(dimsc, conn)
    if shared["ws"] is None:
        shared["ws"] = torch.empty(int(nb * 1.3) + 256, dtype=torch.uint8, device="cuda")
    ws = shared["ws"]
    assert ws.numel() >= nb + 256, "variants' workspaces differ too much"
    h = vp()
    assert L.mt_create(ctypes.byref(h), dimsc, conn, 0, vp((ws.data_ptr() + 255) // 256 * 256), nb) == 0
    L.mt_set_profiling(h, 1)
    runs.append({"name": os.path.basename(p), "L": L, "h": h, "ws": ws, "t": {}})
stream = vp(torch.cuda.current_stream().cuda_stream)
a, b = ctypes.c_uint64(0), ctypes.c_uint64(0)
for r in range(rounds + 1):
    for run in runs:
        L, h = run["L"], run["h"]
        assert L.mt_compute(h, vp(fd.data_ptr()), vp(T.data_ptr()), 0, stream) == 0
        L.mt_diagram(h, None, 0, ctypes.byref(a), ctypes.byref(b), stream)   # (timing-only builds may report errors)
        names = (ctypes.c_char_p * 16)()
        ms = (ctypes.c_float * 16)()
        k = L.mt_kernel_times(h, names, ms, 16)
        if r == 0:
            continue   # warm-up round
        tot = 0.0
        for i in range(k):
            run["t"].setdefault(names[i].decode(), []).append(ms[i])
            tot += ms[i]
        run["t"].setdefault("TOTAL", []).append(tot)
for run in runs:
    med = {k: round(statistics.median(v), 3) for k, v in run["t"].items()}
    print(json.dumps({"cfg": cfg, "lib": run["name"], "median_ms": med, "pairs": a.value}), flush=True)
