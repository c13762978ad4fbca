"""x-slab decomposition on one B200: n slabs stepped in one process with
halo-plane copies (lesb_group_step) must reproduce the single-domain step
bitwise for every field (halos included), report the same blow-up step and
stage, and give the same residuals to summation-order tolerance."""

import os
import subprocess
import sys

import numpy as np
import pytest

import golden_inputs as gi

pytestmark = pytest.mark.gpu

FIELDS = ("u", "v", "w", "fgh", "fgh_old", "p")


def bits_equal(a, b):
    return a.shape == b.shape and np.array_equal(np.ascontiguousarray(a).view(np.uint32),
                                                 np.ascontiguousarray(b).view(np.uint32))


def single(P, st, inflow, n_steps, n_iter, scheme):
    g = P.Grid(st["im"], st["jm"], st["km"], st["dx1"], st["dy1"], st["dzn"])
    fs = P.FlowState.create(g, dt=st["dt"], vn=st["vn"], cs=st["cs"])
    for n in FIELDS + ("mask",):
        getattr(fs, n)[...] = st[n]
    out = []
    for _ in range(n_steps):
        P.les.step(fs, P.WindProfile(*inflow), n_iter=n_iter, scheme=scheme)
        out.append({n: getattr(fs, n).copy() for n in FIELDS})
    return out


@pytest.mark.parametrize("solver", ["resident", "separate", "passes", "passes-copies", "passes-serial"])
@pytest.mark.parametrize("dims,nslabs,scheme", [
    ((24, 10, 8), 2, "redblack"),
    ((24, 10, 8), 3, "redblack"),
    ((9, 7, 5), 3, "redblack"),      # odd jm, equal slabs of 3 planes
    ((10, 7, 5), 3, "redblack"),     # uneven slabs: streaming passes
    ((16, 12, 10), 4, "twinned"),
    ((32, 32, 16), 4, "redblack"),
    ((48, 40, 20), 2, "redblack"),   # several resident tiles per slab in x and y
])
def test_slabs_equal_single_domain(dims, nslabs, scheme, solver, monkeypatch):
    """Red-black slabs of one shape run the resident solver as one group
    launch (tile faces cross slab boundaries through ghost slots, the
    in-process form of the NVLink peer path); LESB_GROUP_SEPARATE launches
    every slab on its own stream with its own epoch (what each rank does on
    its own GPU); LESB_GROUP_PASSES forces the streaming colour passes with
    plane copies -- by default with the exchange fused into the pass kernel
    (edge-plane values written straight into the neighbour's ghost planes,
    tag-checked) and every slab's passes on its own stream ordered only by
    the ghost tags (the multi-GPU protocol); "-serial" with the slabs'
    passes on one stream, "-copies" with a plane copy after every pass."""
    import paper_1504_02264_b200 as P
    from paper_1504_02264_b200.slabs import SlabGroup

    monkeypatch.delenv("LESB_GROUP_PASSES", raising=False)
    monkeypatch.delenv("LESB_GROUP_SEPARATE", raising=False)
    monkeypatch.delenv("LESB_GHOST", raising=False)
    monkeypatch.delenv("LESB_GROUP_STREAMS", raising=False)
    if solver.startswith("passes"):
        monkeypatch.setenv("LESB_GROUP_PASSES", "1")
        if solver == "passes-copies":
            monkeypatch.setenv("LESB_GHOST", "0")
        elif solver == "passes-serial":
            monkeypatch.setenv("LESB_GROUP_STREAMS", "0")
    elif solver == "separate":  # one launch per slab, own stream and epoch: the per-GPU form
        monkeypatch.setenv("LESB_GROUP_SEPARATE", "1")
    P.runtime.set_sor_path(0)
    st = gi.random_state(*dims, seed=sum(dims) * 7 + nslabs, vel_scale=0.3)
    inflow = gi.random_inflow(dims[2], seed=5)
    sch = P.Scheme(scheme)
    ref = single(P, st, inflow, 3, 12, sch)
    g = P.Grid(*dims, st["dx1"], st["dy1"], st["dzn"])
    grp = SlabGroup(g, nslabs, dt=st["dt"], vn=st["vn"], cs=st["cs"])
    try:
        grp.upload(st)
        for s in range(3):
            grp.step(P.WindProfile(*inflow), n_iter=12, scheme=sch)
            for n in FIELDS:
                got = grp.gather(n)
                assert bits_equal(got, ref[s][n]), (dims, nslabs, s, n)
    finally:
        grp.close()


def test_slabs_config1_blowup():
    """Config 1 (32x32x16, one building straddling slabs): same hashes at
    step 10 and the same blow-up step and stage (17, velfg) as one domain."""
    import paper_1504_02264_b200 as P
    from paper_1504_02264_b200.slabs import SlabGroup

    st = gi.config1_state()
    g = P.Grid(32, 32, 16, st["dx1"], st["dy1"], st["dzn"])
    grp = SlabGroup(g, 3, dt=st["dt"], vn=st["vn"], cs=st["cs"])
    try:
        grp.upload(st)
        inflow = P.WindProfile(*gi.default_inflow(16))
        step = 0
        with pytest.raises(P.NumericsError) as err:
            while step < 40:
                grp.step(inflow)
                step += 1
        assert step + 1 == 17
        assert err.value.stage == "velfg"
    finally:
        grp.close()


def test_slabs_runtime_specialised():
    """The slab group tests with every kernel compiled for its geometry at run
    time (LESB_JIT_MIN_CELLS=0, fresh process): the slabs of a group share
    one specialised resident kernel (same shape and tile plan), and slabs
    launched one by one must not wait on a neighbour whose kernel is still
    being compiled (measured: slab positions as compile-time constants gave
    each slab its own kernel and the "separate" launches timed out)."""
    env = dict(os.environ, LESB_JIT_MIN_CELLS="0")
    r = subprocess.run([sys.executable, "-m", "pytest", os.path.abspath(__file__), "-q", "-x", "-p", "no:cacheprovider",
                        "-k", "equal_single_domain and (resident or separate or serial)"],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
