#!/usr/bin/env python
"""bench.py -- merge tree + 0-dim persistence diagram throughput on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl mt|reference]

A step is one pass of the whole hot path (keys, steepest-descent
init, CAS edge merge, repair, diagram) over one synthetic field: mt_compute +
mt_diagram through the C ABI, inputs resident in HBM.  ``value`` is
Mvertices/s over all ranks; ``e2e`` repeats the step through the public API
with pinned HOST buffers (H2D of f, D2H of the triplet store and the diagram
inside the timed region).  ``roofline`` reports the dominant kernel's
algorithmic bytes per CUDA-event-timed
launch against the measured HBM copy bandwidth.  ``cpu_baseline`` times the
oracle O1 (serial C, 1 core) on a bounded sub-block of the same field.

--impl reference times the oracle itself (the only "reference" this paper-only
build has) on bounded samples of the same workload.
Under torchrun (N > 1) the grid is split into z-slabs, one per rank
(paper_2301_10838_b200/dist.py): local merge tree, NCCL all-gather of the
boundary forests, global merge + repair; the same total grid on every N
(strong scaling), time = max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "merge tree + 0-dim diagram Mvertices/s at 1/2/4/8 B200; % of HBM roofline"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", default="c5", choices=["c1", "c2", "c3", "c4", "c5"])
    p.add_argument("--scale", type=int, default=None, help="override the grid edge (debug)")
    p.add_argument("--impl", default="mt", choices=["mt", "reference"])
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--split", action="store_true", help="split tree (MT_FLAG_SPLIT_TREE)")
    return p.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index: int):
        self.dev = device_index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.dev), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax = float(parts[2])
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def field_for(cfg, scale, device):
    from paper_2301_10838_b200 import fields
    return fields.make(cfg, scale=scale, device=device)


def oracle_rate(f, dims, conn, planes, split=False):
    """O1 on the first `planes` z-planes (2D: rows) of the field; returns (Mv/s, n, seconds)."""
    import oracle
    nx, ny, nz = dims
    if nz > 1:
        sub_dims = (nx, ny, min(planes, nz))
    else:
        sub_dims = (nx, min(max(1, planes * 64), ny), 1)
    n = sub_dims[0] * sub_dims[1] * sub_dims[2]
    sub = np.ascontiguousarray(f[:n])
    conn = 4 if sub_dims[2] == 1 else conn
    t0 = time.perf_counter()
    oracle.merge_tree(sub, sub_dims, conn=conn, split=split)
    dt = time.perf_counter() - t0
    return n / dt / 1e6, n, dt, sub_dims


def paper_cpu_rate(f, dims, conn, planes, split=False):
    """The paper's Alg. 1-5 with CAS on all host cores (OpenMP; baseline/paper_cpu) on the first
    `planes` z-planes; the second of two runs is timed.  Returns (Mv/s, n, seconds, dims, threads)."""
    from baseline import paper_cpu
    nx, ny, nz = dims
    sub_dims = (nx, ny, min(planes, nz)) if nz > 1 else (nx, min(max(1, planes * 64), ny), 1)
    n = sub_dims[0] * sub_dims[1] * sub_dims[2]
    sub = np.ascontiguousarray(f[:n])
    conn = 4 if sub_dims[2] == 1 else conn
    dt = 0.0
    for _ in range(2):
        t0 = time.perf_counter()
        paper_cpu.merge_tree(sub, sub_dims, conn=conn, split=split)
        dt = time.perf_counter() - t0
    return n / dt / 1e6, n, dt, sub_dims, paper_cpu.max_threads()


def cpu_sample_planes(cfg, target_s, rate=1.3e6):
    # oracle throughput is ~1-2 Mv/s on one core; pick the number of planes that
    # gives about target_s seconds of work
    from paper_2301_10838_b200.fields import CONFIGS
    nx, ny, nz = CONFIGS[cfg]["dims"]
    per_plane = nx * ny if nz > 1 else nx * 64
    return max(1, int(target_s * rate / per_plane))


def run_reference(args, rank, world):
    """--impl reference: the oracle O1 timed on bounded samples of the workload."""
    if rank != 0:
        return
    import oracle  # noqa: F401  (test infrastructure; the one place bench executes it besides cpu_baseline)
    f, dims, conn = field_for(args.config, args.scale, "cuda" if args.config == "c5" and _has_cuda() else "cpu")
    planes = cpu_sample_planes(args.config, 3.0)
    for _ in range(args.warmup):
        oracle_rate(f, dims, conn, planes, args.split)
    times, nv = [], 0
    for _ in range(args.steps):
        r, n, dt, sub = oracle_rate(f, dims, conn, planes, args.split)
        times.append(dt)
        nv = n
    total = sum(times)
    value = nv * args.steps / total / 1e6
    cores = 1
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "Mvertices/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": _config(args, dims, conn),
        "cpu_baseline": {"value": value, "unit": "Mvertices/s", "cores": cores, "kind": "oracle",
                         "sample": f"O1 (serial C union-find) on the first {sub} sub-grid of the "
                                   f"{args.config} field per step"},
        "e2e": {"value": value, "unit": "Mvertices/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def _device_index():
    # MT_FORCE_DEVICE puts every rank on one GPU (with MT_DIST_BACKEND=gloo) to test the
    # multi-rank path on a single-GPU box; normally LOCAL_RANK picks the GPU
    return int(os.environ.get("MT_FORCE_DEVICE", os.environ.get("LOCAL_RANK", 0)))


def _has_cuda():
    import torch
    return torch.cuda.is_available()


def _config(args, dims, conn, world=1):
    from paper_2301_10838_b200.fields import CONFIGS
    return {"workload": f"{args.config}: {CONFIGS[args.config]['name']}" + (" (split tree)" if args.split else ""),
            "dims": list(dims), "connectivity": conn, "vertices": int(np.prod(dims)),
            "l2_policy": "inputs larger than L2 + 512 MiB L2 flush before every timed step",
            "parallelism": f"zslab{world} (NCCL all-gather of boundary forests)" if world > 1 else "single"}


# algorithmic bytes of each kernel: n vertices, rec diagram
# records, ecross tile-crossing edges; the store is counted at the paper's 8 B per vertex
def _ecross(dims):
    nx, ny, nz = dims
    ty, tz = (128, 1) if nz == 1 else (16, 8)
    kx, ky, kz = -(-nx // 32) - 1, -(-ny // ty) - 1, -(-nz // tz) - 1
    return kx * ny * nz + ky * nx * nz + kz * nx * ny


ALG_BYTES = {
    "tile_tmt": lambda n, rec, ec: 12 * n,                 # read f (4) + write the tile store (8)
    "dedupe_cross": lambda n, rec, ec: 16 * ec,            # the tile store (order key, R) of both ends
    "merge_queue": lambda n, rec, ec: 2 * 8 * ec,          # (lower bound) both end cells of every crossing edge
    "repair": lambda n, rec, ec: 16 * n,                   # read the tile store (8), write T (8)
    "diagram": lambda n, rec, ec: 4 * n + 16 * rec,        # one 4-B word per vertex to find the minima + records
    "finish_diagram": lambda n, rec, ec: 0,
}


class SingleRunner:
    """One GPU, the whole grid: mt_compute + mt_diagram through the C ABI."""

    def __init__(self, dims, conn, f, dev, flags):
        from paper_2301_10838_b200 import _lib
        self.lib = _lib
        self.mt = _lib.MergeTree(dims, conn, device=dev.index)
        self.ctx = self.mt.ctx
        self.n = int(np.prod(dims))
        self.f = f
        self.T = torch_empty(self.n, dev)
        self.flags = flags

    def step(self, f=None, rec_dev=None):
        lib = self.lib
        lib.mt_compute(self.ctx, (self.f if f is None else f).data_ptr(), self.T.data_ptr(), self.flags)
        st, npairs, ness = lib.mt_diagram(self.ctx, rec_dev.data_ptr() if rec_dev is not None else 0,
                                          rec_dev.shape[0] if rec_dev is not None else 0)
        if st != lib.MT_OK:
            raise lib.MTError(st, "mt_diagram")
        return npairs, ness


class SlabRunner:
    """Rank r of a z-slab decomposition (paper_2301_10838_b200.dist): local merge tree, NCCL all-gather
    of the boundary forests, global merge + repair of the slab."""

    def __init__(self, dims, f_slab, dev, flags):
        from paper_2301_10838_b200 import _lib
        from paper_2301_10838_b200.dist import DistMergeTree
        self.lib = _lib
        import torch.distributed as dist
        # the library's own NCCL exchange (mt_create_dist) on NCCL groups; torch's collectives otherwise
        self.d = DistMergeTree(dims, device=dev, transport="nccl" if dist.get_backend() == "nccl" else "torch")
        self.ctx = self.d.slab.ctx
        self.n = self.d.slab.n
        self.f = f_slab
        self.T = torch_empty(self.n, dev)
        self.split = bool(flags)

    def step(self, f=None, rec_dev=None):
        lib = self.lib
        self.d.compute(self.f if f is None else f, self.split, self.T)
        st, npairs, ness = lib.mt_diagram(self.ctx, rec_dev.data_ptr() if rec_dev is not None else 0,
                                          rec_dev.shape[0] if rec_dev is not None else 0)
        if st != lib.MT_OK:
            raise lib.MTError(st, "mt_diagram")
        return npairs, ness


def torch_empty(n, dev):
    import torch
    return torch.empty(n, dtype=torch.int64, device=dev)


def run_mt(args, rank, world):
    import torch
    import torch.distributed as dist

    from paper_2301_10838_b200 import _lib

    dev = torch.device("cuda", _device_index())
    torch.cuda.set_device(dev)
    f_np, dims, conn = field_for(args.config, args.scale, dev if args.config == "c5" else "cpu")
    n_global = int(np.prod(dims))
    flags = _lib.MT_FLAG_SPLIT_TREE if args.split else 0
    if world > 1:
        from paper_2301_10838_b200.dist import slab_bounds
        if dims[2] < world or conn != 6:
            raise SystemExit("multi-GPU runs need a 3D grid with at least one plane per rank")
        zb = slab_bounds(dims[2], world)
        plane = dims[0] * dims[1]
        f_np = np.ascontiguousarray(f_np[zb[rank] * plane: zb[rank + 1] * plane])
        runner = SlabRunner(dims, torch.from_numpy(f_np).to(dev), dev, flags)
    else:
        runner = SingleRunner(dims, conn, torch.from_numpy(f_np).to(dev), dev, flags)
    n_local = runner.n
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    for _ in range(max(3, args.warmup)):
        runner.step()
    _lib.mt_set_profiling(runner.ctx, True)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    kt = {}
    launches = 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev.index) as clk:
        for i in range(args.steps):
            flush.fill_(i & 0xff)  # evict L2 between timed steps (outside the events)
            ev[i][0].record(stream)
            npairs, ness = runner.step()
            ev[i][1].record(stream)
            launches += _lib.mt_last_launch_count(runner.ctx)
            for name, ms in _lib.mt_kernel_times(runner.ctx, 16):
                kt.setdefault(name, []).append(ms)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    _lib.mt_set_profiling(runner.ctx, False)
    step_ms = [a.elapsed_time(b) for a, b in ev]
    my_ms = sum(step_ms)
    if world > 1:
        t = torch.tensor([my_ms, float(npairs), float(ness), float(launches)], dtype=torch.float64, device=dev)
        tm = t.clone()
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        max_ms = float(tm[0].item())
        npairs, ness, launches = int(t[1].item()), int(t[2].item()), int(t[3].item())
    else:
        max_ms = my_ms
    ms_per_step = max_ms / args.steps
    value = n_global / (ms_per_step * 1e-3) / 1e6

    # roofline of the dominant kernel (rank 0's kernels; per launch, its own slab)
    peak, peak_kind = peaks()
    recs = npairs + ness
    avg = {k: statistics.mean(v) for k, v in kt.items()}
    dom = max((k for k in avg if k in ALG_BYTES), key=lambda k: avg[k])
    local_dims = (dims[0], dims[1], n_local // (dims[0] * dims[1]))
    alg = ALG_BYTES[dom](n_local, recs * n_local // n_global, _ecross(local_dims))
    achieved = alg / (avg[dom] * 1e-3) / 1e9
    traffic, issue = None, None
    prof_path = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(prof_path):
        try:
            prof = json.load(open(prof_path))
            traffic = prof.get(args.config, {}).get(dom)
            issue = prof.get("issue", {}).get(args.config, {}).get(dom)
        except Exception:
            traffic, issue = None, None
    # secondary ceilings (SURVEY.md 8d, N11 microbenchmarks in profiles/): the global merge is
    # bound by 128-bit L2 CAS throughput, the repair by random 16-B cell gathers; per-launch event
    # counts from one ncu capture (profiles/traffic.json "secondary"), live kernel times here
    secondary = None
    if os.path.exists(prof_path):
        try:
            sec = json.load(open(prof_path)).get("secondary", {}).get(args.config, {})
            secondary = {}
            for k, d in sec.items():
                if k in avg and not k.startswith("_"):
                    rate = d["count_per_launch"] / (avg[k] * 1e-3)
                    secondary[k] = {"bound": d["bound"], "achieved": rate, "peak": d["peak"], "unit": d["unit"],
                                    "frac": rate / d["peak"], "count_per_launch": d["count_per_launch"],
                                    "source": d["source"]}
        except Exception:
            secondary = None
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                # what actually bounds the kernel (ncu, profiles/traffic.json): instruction issue
                "issue": issue,
                "alg_bytes_per_launch": alg, "kernel_ms": avg[dom],
                "kernel_share_of_step": avg[dom] / ms_per_step,
                "kernels_ms": avg,
                "step_alg_bytes_per_vertex": 12 + 16 * recs / n_global,
                "step_frac": (12 * n_global + 16 * recs) / (ms_per_step * 1e-3) / 1e9 / (peak * world)}

    # end to end through the public API with pinned host buffers: every step copies its field
    # from host memory and its triplets + diagram back (inside the timed region).  One GPU: the
    # library's HostPipeline overlaps H2D(i+1) / compute(i) / D2H(i-1) on three streams; slabs:
    # sequential copies around each distributed step.
    e2e = None
    if not args.no_e2e:
        e2e_steps = max(2, min(args.steps, 10))   # (a longer run amortises the pipeline fill: H2D(0) + compute(0))
        f_host = torch.from_numpy(f_np).pin_memory()
        cap = (n_local + 1) // 2 + 2
        if world == 1:
            from paper_2301_10838_b200.pipeline import HostPipeline
            del runner
            torch.cuda.empty_cache()
            pipe = HostPipeline(dims, conn, device=dev.index)
            T_hosts = [torch.empty(n_local, dtype=torch.int64).pin_memory() for _ in range(2)]
            nrec = npairs + ness  # known from the timed steps (the field does not change)
            rec_hosts = [torch.empty((nrec + 1, 4), dtype=torch.int32).pin_memory() for _ in range(2)]
            pipe.run([f_host], T_hosts[:1], rec_hosts[:1], args.split)      # warm-up
            torch.cuda.synchronize()
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record(stream)     # mt_compute_host starts after, and `stream` waits for, its pipeline
            counts = pipe.run([f_host] * e2e_steps, [T_hosts[i % 2] for i in range(e2e_steps)],
                              [rec_hosts[i % 2] for i in range(e2e_steps)], args.split, stream)
            t1.record(stream)
            torch.cuda.synchronize()
            e_ms = t0.elapsed_time(t1)
            a, b = counts[-1]
            h2d, d2h = 4 * n_local, 8 * n_local + 16 * (a + b)
        else:
            T_host = torch.empty(n_local, dtype=torch.int64).pin_memory()
            rec_dev = torch.empty((cap, 4), dtype=torch.int32, device=dev)
            rec_host = torch.empty(rec_dev.shape, dtype=torch.int32).pin_memory()
            f_dev = torch.empty(n_local, dtype=torch.float32, device=dev)
            h2d = d2h = 0
            dist.barrier()
            torch.cuda.synchronize()
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record(stream)
            for _ in range(e2e_steps):
                f_dev.copy_(f_host, non_blocking=True)
                a, b = runner.step(f_dev, rec_dev)
                T_host.copy_(runner.T, non_blocking=True)
                rec_host[: a + b].copy_(rec_dev[: a + b], non_blocking=True)
                h2d = 4 * n_local
                d2h = 8 * n_local + 16 * (a + b)
            t1.record(stream)
            torch.cuda.synchronize()
            e_ms = t0.elapsed_time(t1)
            t = torch.tensor([e_ms, float(h2d), float(d2h)], dtype=torch.float64, device=dev)
            tm = t.clone()
            dist.all_reduce(tm, op=dist.ReduceOp.MAX)
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
            e_ms, h2d, d2h = float(tm[0].item()), int(t[1].item()), int(t[2].item())
        e2e = {"value": n_global * e2e_steps / (e_ms * 1e-3) / 1e6, "unit": "Mvertices/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": e2e_steps,
               "overlap": "mt_compute_host (C ABI): H2D(i+1) | compute(i) | D2H(i-1) on the library's 3 streams"
               if world == 1 else "none"}

    cpu = cpu_paper = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        planes = cpu_sample_planes(args.config, 15.0)
        r, nv, dt, sub = oracle_rate(f_np, dims, conn, planes, args.split)
        cpu = {"value": r, "unit": "Mvertices/s", "cores": 1, "kind": "oracle",
               "sample": f"O1 (serial C union-find + elder rule) on the first {sub} sub-grid "
                         f"({nv} vertices, {dt:.1f} s) of the same field, 1 of {os.cpu_count()} host cores"}
        # the paper's own method on every host core (optional second CPU baseline,
        # the analogue of the paper's OpenMP column) -- a reported baseline, not the oracle
        try:
            pplanes = cpu_sample_planes(args.config, 2.0, rate=3e7)
            pr, pnv, pdt, psub, pthr = paper_cpu_rate(f_np, dims, conn, pplanes, args.split)
            cpu_paper = {"value": pr, "unit": "Mvertices/s", "cores": pthr, "kind": "paper Alg. 1-5, OpenMP + CAS",
                         "sample": f"baseline/paper_cpu on the first {psub} sub-grid ({pnv} vertices, {pdt:.2f} s, "
                                   f"second of two runs) of the same field, {pthr} of {os.cpu_count()} host threads"}
        except Exception as e:   # a missing OpenMP toolchain must not void the GPU measurement
            cpu_paper = {"unavailable": str(e)[:200]}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "Mvertices/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded generator, paper_2301_10838_b200/fields.py)",
            "config": _config(args, dims, conn, world),
            "pairs": npairs, "essential": ness,
            "step_ms": {"median": statistics.median(step_ms), "min": min(step_ms), "max": max(step_ms)},
            "roofline": roofline, "secondary_ceilings": secondary, "cpu_baseline": cpu,
            "cpu_paper_method": cpu_paper, "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        if world > 1:
            line["forest_records"] = runner.d.forest_records
        print(json.dumps(line), flush=True)


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(_device_index())
        backend = os.environ.get("MT_DIST_BACKEND", "nccl")  # gloo: multi-rank test on one GPU
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", _device_index()))
        else:
            dist.init_process_group(backend)
    try:
        run_mt(args, rank, world)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
