"""Host-side logic of the x-slab decomposition, on CPU: slab bounds,
scatter / gather of the reference arrays, and the halo-plane schedule
(slabs.halo_plan, which capi.cu's NCCL exchange mirrors) run over real
torch.distributed gloo ranks (world sizes 2 and 3)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1504_02264_b200.slabs import gather, halo_plan, slab_bounds, slice_global


def test_slab_bounds_tile_the_axis():
    for im in (1, 7, 150, 151):
        for n in range(1, min(im, 9) + 1):
            b = [slab_bounds(im, n, s) for s in range(n)]
            assert b[0][0] == 1 and b[-1][1] == im
            assert all(b[s + 1][0] == b[s][1] + 1 for s in range(n - 1))
            sizes = [i1 - i0 + 1 for i0, i1 in b]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        slab_bounds(4, 5, 0)


def test_scatter_gather_roundtrip():
    rng = np.random.default_rng(0)
    for shape in ((12, 6, 5), (12, 6, 5, 3)):
        a = rng.standard_normal(shape).astype(np.float32)
        im = shape[0] - 2
        for n in (1, 2, 3, 5):
            b = [slab_bounds(im, n, s) for s in range(n)]
            parts = [slice_global(a, i0, i1) for i0, i1 in b]
            assert np.array_equal(gather(parts, b), a)


def test_halo_plan_shapes():
    assert halo_plan(5, False, False, 2) == []
    assert halo_plan(5, True, False, 2) == [("send", -1, 1, 2), ("recv", -1, 0, 1)]
    assert halo_plan(5, False, True, 1) == [("send", 1, 5, 1), ("recv", 1, 6, 1)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, im, depth, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(42)
        glob = rng.standard_normal((im + 4, 5, 4)).astype(np.float32)  # +2 planes for the depth-2 halo
        i0, i1 = slab_bounds(im, world, rank)
        n = i1 - i0 + 1
        # local buffer: planes 0 .. n+2 (depth-2 high halo), halos poisoned
        loc = np.full((n + 3, 5, 4), np.nan, np.float32)
        loc[1:n + 1] = glob[i0:i1 + 1]
        t = torch.from_numpy(loc)
        reqs = []
        for op, peer, first, cnt in halo_plan(n, rank > 0, rank < world - 1, depth):
            view = t[first:first + cnt].contiguous() if op == "send" else None
            if op == "send":
                reqs.append(dist.isend(view, rank + peer))
            else:
                buf = torch.empty((cnt, 5, 4))
                reqs.append((dist.irecv(buf, rank + peer), first, cnt, buf))
        for r in reqs:
            if isinstance(r, tuple):
                r[0].wait()
                t[r[1]:r[1] + r[2]] = r[3]
            else:
                r.wait()
        ok = True
        if rank > 0:
            ok &= np.array_equal(t[0].numpy(), glob[i0 - 1])
        if rank < world - 1:
            ok &= np.array_equal(t[n + 1:n + 1 + depth].numpy(), glob[i1 + 1:i1 + 1 + depth])
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,depth", [(2, 2), (3, 1), (3, 2)])
def test_halo_exchange_over_gloo(world, depth):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 11, depth, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    res = dict(q.get(timeout=5) for _ in range(world))
    assert all(res[r] for r in range(world)), res
