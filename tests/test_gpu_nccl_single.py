"""The one-process-per-GPU slab path on a single rank under a torch.distributed
NCCL process group (the bench's configuration; the only NCCL world one GPU
allows): lesb_link_nccl, the face-buffer peer mapping (NCCL all-gather +
all-reduce of one rank), the step graph with its grouped NCCL exchanges and
the library's own NCCL reductions -- the first failing stage (C5) and the
press residual history (C4) -- against the plain single-domain calls."""

import socket

import numpy as np
import pytest

import golden_inputs as gi

pytestmark = pytest.mark.gpu


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture()
def nccl_world():
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{free_port()}", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


def _state(dims, seed):
    import paper_1504_02264_b200 as P

    st = gi.random_state(*dims, seed=seed, vel_scale=0.3)
    g = P.Grid(*dims, st["dx1"], st["dy1"], st["dzn"])
    fs = P.FlowState.create(g, dt=st["dt"], vn=st["vn"], cs=st["cs"])
    for n in ("u", "v", "w", "fgh", "fgh_old", "p", "mask"):
        getattr(fs, n)[...] = st[n]
    return st, g, fs


def bits(a, b):
    return np.array_equal(np.ascontiguousarray(a).view(np.uint32), np.ascontiguousarray(b).view(np.uint32))


@pytest.mark.parametrize("dims", [(32, 24, 16), (300, 40, 12)])
def test_single_rank_slab_domain_equals_domain(nccl_world, dims):
    """Steps (with the residual history), press and a stored-halo solve on a
    one-rank NCCL slab domain equal the single-domain calls bitwise (the
    second grid does not fit the resident solver: streaming split passes)."""
    import paper_1504_02264_b200 as P
    from paper_1504_02264_b200.slabs import SlabDomain

    st, g, fs = _state(dims, seed=11)
    inflow = P.WindProfile(*gi.random_inflow(dims[2], seed=3))
    dom = SlabDomain(g, dt=st["dt"], vn=st["vn"], cs=st["cs"], device=0)
    try:
        dom.upload(st)
        for s in range(4):
            P.les.step(fs, inflow, n_iter=20)
            res = dom.step(inflow, n_iter=20, residuals=s == 3)
        for n in ("u", "v", "w", "fgh", "fgh_old", "p"):
            assert bits(dom.slab.download(n, g.jm, g.km), getattr(fs, n)), n
        assert res is not None and res.shape == (20,) and np.all(np.isfinite(res))
        r_dom = dom.press(n_iter=9)
        r_ref = P.les.press(fs, n_iter=9)
        assert bits(dom.slab.download("p", g.jm, g.km), fs.p)
        np.testing.assert_allclose(r_dom, r_ref, rtol=1e-12, atol=0)
        p0, rhs = gi.sor_problem(*dims, seed=5)
        p_dom, r_dom = dom.solve(p0, rhs, 1.7, 7, P.Scheme.REDBLACK, halo_policy=0)
        c = P.sor.build_uniform_coeffs(P.Grid.uniform(*dims, 2.0))
        p_ref, r_ref = P.sor.solve_pressure(p0, rhs, c, 1.7, 7, P.Scheme.REDBLACK)
        assert bits(p_dom, p_ref)
        np.testing.assert_allclose(r_dom, r_ref, rtol=1e-12, atol=0)
        g0 = dom.gather("u")
        assert bits(g0, fs.u)
    finally:
        dom.close()


def test_single_rank_slab_blowup_stage(nccl_world):
    """A non-finite value is reported with the reference's stage name after
    the library's NCCL stage reduction (velnw, test_les.py:307-312)."""
    import paper_1504_02264_b200 as P
    from paper_1504_02264_b200.slabs import SlabDomain

    dims = (8, 8, 8)
    st = gi.zero_state(*dims, h=1.0)
    st["u"][1, 1, 1] = np.inf
    g = P.Grid.uniform(*dims, 1.0)
    dom = SlabDomain(g, dt=0.5, device=0)
    try:
        dom.upload(st)
        z = np.zeros(8, np.float32)
        with pytest.raises(P.NumericsError) as err:
            dom.step(P.WindProfile(z, z, z), n_iter=2)
        assert err.value.stage == "velnw"
    finally:
        dom.close()


def test_single_rank_slab_async_copies(nccl_world):
    """SlabDomain.stage / commit_staged / download_async (bench.py's N-GPU
    e2e windows) on a one-rank NCCL slab: the staged state steps like the
    uploaded one, and a snapshot taken after step 1 is the step-1 state
    however many steps follow before the wait."""
    import paper_1504_02264_b200 as P
    from paper_1504_02264_b200.slabs import SlabDomain

    dims = (32, 24, 16)
    st, g, fs = _state(dims, seed=13)
    inflow = P.WindProfile(*gi.random_inflow(dims[2], seed=4))
    dom = SlabDomain(g, dt=st["dt"], vn=st["vn"], cs=st["cs"], device=0)
    names = ("u", "v", "w", "fgh", "fgh_old", "p")
    try:
        dom.upload(gi.zero_state(*dims))
        dom.stage(st)
        dom.commit_staged()
        P.les.step(fs, inflow, n_iter=20)
        dom.step(inflow, n_iter=20)
        after1 = {n: getattr(fs, n).copy() for n in names}
        pend = dom.download_async({n: np.empty(dom.slab_shape(n), np.float32) for n in names})
        for _ in range(3):
            P.les.step(fs, inflow, n_iter=20)
            dom.step(inflow, n_iter=20)
        for n in names:
            assert bits(dom.slab.download(n, g.jm, g.km), getattr(fs, n)), n
        got = pend.wait()
        for n in names:
            assert bits(got[n], after1[n]), ("snapshot", n)
        with pytest.raises(ValueError):
            dom.download_async({"u": np.empty((3, 3, 3), np.float32)})
    finally:
        dom.close()
