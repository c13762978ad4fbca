"""The one-process-per-GPU slab path on a single rank (the only NCCL
configuration one GPU allows): lesb_link_nccl, the face-buffer peer mapping
(NCCL all-gather + all-reduce of one rank), the step graph with its grouped
NCCL exchanges and the resident solver -- bitwise equal to the plain
single-domain step."""

import socket

import numpy as np
import pytest

import golden_inputs as gi

pytestmark = pytest.mark.gpu


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_single_rank_slab_domain_equals_domain():
    import torch.distributed as dist

    import paper_1504_02264_b200 as P
    from paper_1504_02264_b200.slabs import SlabDomain

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{free_port()}", rank=0, world_size=1)
    try:
        dims = (32, 24, 16)
        st = gi.random_state(*dims, seed=11, vel_scale=0.3)
        inflow = P.WindProfile(*gi.random_inflow(dims[2], seed=3))
        g = P.Grid(*dims, st["dx1"], st["dy1"], st["dzn"])
        fs = P.FlowState.create(g, dt=st["dt"], vn=st["vn"], cs=st["cs"])
        for n in ("u", "v", "w", "fgh", "fgh_old", "p", "mask"):
            getattr(fs, n)[...] = st[n]
        dom = SlabDomain(g, dt=st["dt"], vn=st["vn"], cs=st["cs"], device=0)
        try:
            dom.upload(st)
            for _ in range(4):
                P.les.step(fs, inflow, n_iter=20)
                dom.step(inflow, n_iter=20)
            for n in ("u", "v", "w", "fgh", "fgh_old", "p"):
                a = dom.slab.download(n, g.jm, g.km)
                b = np.array(getattr(fs, n))
                assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), n
        finally:
            dom.close()
    finally:
        dist.destroy_process_group()
