"""Host logic of the multi-GPU path on CPU: slab bounds, and the variable-size all-gather of
boundary-forest records over a world_size-2 gloo group."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2301_10838_b200.dist import allgather_varsize, slab_bounds


@pytest.mark.parametrize("nz,p", [(1024, 8), (1024, 2), (37, 3), (8, 8), (512, 3), (16, 5), (100, 7)])
def test_slab_bounds(nz, p):
    b = slab_bounds(nz, p)
    assert b[0] == 0 and b[-1] == nz and len(b) == p + 1
    assert all(b[i] < b[i + 1] for i in range(p))
    sizes = [b[i + 1] - b[i] for i in range(p)]
    if nz >= 8 * p:
        assert all(z % 8 == 0 for z in b[1:-1])   # tile-aligned cuts
        assert max(sizes) - min(sizes) <= 16
    else:
        assert max(sizes) - min(sizes) <= 2


def test_slab_bounds_rejects():
    with pytest.raises(ValueError):
        slab_bounds(3, 4)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # rank r contributes r*24+5 bytes of records (different sizes, one empty on rank 0 case)
        n = 0 if rank == 0 else rank * 24 + 5
        t = torch.arange(n, dtype=torch.int64).to(torch.uint8) + rank
        out = allgather_varsize(t)
        q.put((rank, out.tolist()))
    finally:
        dist.destroy_process_group()


def test_allgather_varsize_gloo_world2():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    expect = []
    for r in range(world):
        n = 0 if r == 0 else r * 24 + 5
        expect += [(i + r) & 0xff for i in range(n)]
    assert res[0] == expect and res[1] == expect
