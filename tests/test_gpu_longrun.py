"""Long-run flow statistics (probes P3, P10, P11): the building-free
reference-stable configurations run for hundreds of steps on the device reach
the statistics the reference itself reported -- 32x32x16 x 1000 steps, and
64x64x32 / 128x128x32 x 400 steps -- and x-slab decompositions of them stay
bitwise equal to the single domain for the whole run (1 vs N "GPUs", here
slabs on one device)."""

import numpy as np
import pytest

import golden_inputs as gi

pytestmark = pytest.mark.gpu

# (grid, steps): reference values as printed by the probes,
# compared at the precision they were printed with
PROBES = [
    ((32, 32, 16), 1000, {"mean_u": (0.59973, 5e-6), "rms_w": (0.007295, 5e-7), "max_div": (0.0015, 5e-5)}),
    ((64, 64, 32), 400, {"mean_u": (0.631, 5e-4), "rms_w": (0.037, 5e-4), "max_div": (0.0028, 5e-5)}),
    ((128, 128, 32), 400, {"mean_u": (0.373, 5e-4), "rms_w": (0.094, 5e-4), "max_div": (0.0049, 5e-5),
                           "max_u": (0.7882, 5e-5)}),
]


def flow_stats(fs, g):
    u, v, w = (np.array(getattr(fs, n)) for n in ("u", "v", "w"))
    im, jm, km = g.im, g.jm, g.km
    ui, wi = u[1:-1, 1:-1, 1:-1], w[1:-1, 1:-1, 1:-1]
    div = (((u[1:-1, 1:-1, 1:-1] - u[:-2, 1:-1, 1:-1]) / g.dx1[1:im + 1, None, None]
            + (v[1:-1, 1:-1, 1:-1] - v[1:-1, :-2, 1:-1]) / g.dy1[None, 1:jm + 1, None])
           + (w[1:-1, 1:-1, 1:-1] - w[1:-1, 1:-1, :-2]) / g.dzn[None, None, 1:km + 1])
    return {"mean_u": float(ui.astype(np.float64).mean()),
            "rms_w": float(np.sqrt((wi.astype(np.float64) ** 2).mean())),
            "max_u": float(np.abs(u).max()),          # includes the inflow face
            "max_div": float(np.abs(div).max())}


def make(P, dims):
    st = gi.zero_state(*dims)
    g = P.Grid(*dims, st["dx1"], st["dy1"], st["dzn"])
    return st, g


@pytest.mark.parametrize("dims,n_steps,want", PROBES)
def test_long_run_statistics_match_reference(dims, n_steps, want):
    import paper_1504_02264_b200 as P

    st, g = make(P, dims)
    fs = P.FlowState.create(g, dt=0.5, vn=0.8, cs=0.14)
    inflow = P.WindProfile(*gi.default_inflow(dims[2]))
    assert P.les.run_steps(fs, inflow, n_steps) == n_steps
    got = flow_stats(fs, g)
    for k, (ref, tol) in want.items():
        assert abs(got[k] - ref) <= tol, (dims, k, got[k], ref)


@pytest.mark.parametrize("nslabs,mode", [(2, "resident"), (4, "resident"), (2, "separate"), (4, "passes")])
def test_long_run_slabs_bitwise(nslabs, mode, monkeypatch):
    """64x64x32 x 400 steps: slabs equal one domain bitwise at the end."""
    import paper_1504_02264_b200 as P
    from paper_1504_02264_b200.slabs import SlabGroup

    monkeypatch.delenv("LESB_GROUP_PASSES", raising=False)
    monkeypatch.delenv("LESB_GROUP_SEPARATE", raising=False)
    if mode == "passes":
        monkeypatch.setenv("LESB_GROUP_PASSES", "1")
    elif mode == "separate":
        monkeypatch.setenv("LESB_GROUP_SEPARATE", "1")
    dims, n_steps = (64, 64, 32), 400
    st, g = make(P, dims)
    fs = P.FlowState.create(g, dt=0.5, vn=0.8, cs=0.14)
    inflow = P.WindProfile(*gi.default_inflow(dims[2]))
    P.les.run_steps(fs, inflow, n_steps)
    grp = SlabGroup(g, nslabs, dt=0.5, vn=0.8, cs=0.14)
    try:
        grp.upload(st)
        for _ in range(n_steps):
            grp.step(inflow)
        for n in ("u", "v", "w", "p", "fgh", "fgh_old"):
            a, b = grp.gather(n), np.array(getattr(fs, n))
            assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), (nslabs, mode, n)
    finally:
        grp.close()


def run_to_blowup(stepper, limit):
    """Steps until NumericsError; returns (failing step, 1-based; stage)."""
    import paper_1504_02264_b200 as P

    done = 0
    with pytest.raises(P.NumericsError) as err:
        while done < limit:
            stepper()
            done += 1
    return done + 1, err.value.stage


@pytest.mark.parametrize("dims,nslabs,want", [((150, 150, 90), 2, (54, "velfg")),
                                              ((600, 600, 90), 4, None)])
def test_km90_blowup_step_and_stage(dims, nslabs, want):
    """the building-free km=90 flow is not finite in the
    reference dynamics (probe P10: 150x150x90 fails in velfg at step 54).  One
    domain reaches the reference's failing step and stage, and an x-slab
    decomposition fails at the same step and stage (600x600x90: the strong-
    scaling grid, whose failing step the reference did not record)."""
    import paper_1504_02264_b200 as P
    from paper_1504_02264_b200.slabs import SlabGroup

    st, g = make(P, dims)
    inflow = P.WindProfile(*gi.default_inflow(dims[2]))
    fs = P.FlowState.create(g, dt=0.5, vn=0.8, cs=0.14)
    one = run_to_blowup(lambda: P.les.step(fs, inflow), 200)
    if want is not None:
        assert one == want
    grp = SlabGroup(g, nslabs, dt=0.5, vn=0.8, cs=0.14)
    try:
        grp.upload(st)
        assert run_to_blowup(lambda: grp.step(inflow), 200) == one
    finally:
        grp.close()


def test_weak_scaling_long_run_slabs_bitwise():
    """Config 5(c): 300x300x32 per GPU x 1000 steps, here two slabs (global
    600x300x32) on one device against the single domain, bitwise."""
    import paper_1504_02264_b200 as P
    from paper_1504_02264_b200.slabs import SlabGroup

    dims, n_steps = (600, 300, 32), 1000
    st, g = make(P, dims)
    inflow = P.WindProfile(*gi.default_inflow(dims[2]))
    fs = P.FlowState.create(g, dt=0.5, vn=0.8, cs=0.14)
    assert P.les.run_steps(fs, inflow, n_steps) == n_steps
    grp = SlabGroup(g, 2, dt=0.5, vn=0.8, cs=0.14)
    try:
        grp.upload(st)
        for _ in range(n_steps):
            grp.step(inflow)
        for n in ("u", "v", "w", "p", "fgh", "fgh_old"):
            a, b = grp.gather(n), np.array(getattr(fs, n))
            assert np.array_equal(a.view(np.uint32), b.view(np.uint32)), n
        assert np.isfinite(np.array(fs.u)).all()
    finally:
        grp.close()
