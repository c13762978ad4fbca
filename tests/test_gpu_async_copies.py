"""Asynchronous state copies (FlowState.stage / commit_staged /
download_async over lesb_stage_upload / lesb_stage_commit /
lesb_download_async / lesb_copies_wait): a staged state steps bitwise like an
assigned one (against the reference's golden step vectors), a snapshot taken
mid-run is the state at that point however many steps follow before the
wait, and the pipelined restart/dump pattern bench.py's e2e uses gives the
same fields as the synchronous one."""

from __future__ import annotations

import os

import numpy as np
import pytest

import golden_inputs as gi

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = np.load(os.path.join(HERE, "golden", "small.npz"))
FIELDS = ("u", "v", "w", "fgh", "fgh_old", "p")
ALL = FIELDS + ("mask",)


def bits_equal(a, b):
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.uint32), b.view(np.uint32))


def grid_of(P, st):
    return P.Grid(st["im"], st["jm"], st["km"], st["dx1"], st["dy1"], st["dzn"])


def pinned_like(a):
    import torch

    return torch.empty(a.shape, dtype=torch.float32, pin_memory=True).numpy()


@pytest.mark.parametrize("tag,dims,n_steps", gi.STEP_CASES)
def test_staged_state_steps_bitwise(tag, dims, n_steps):
    import paper_1504_02264_b200 as P

    st = gi.step_state(tag, *dims)
    inflow = P.WindProfile(*gi.step_inflow(tag, dims[2]))
    scheme = P.Scheme(gi.STEP_SCHEME[tag])
    fs = P.FlowState.create(grid_of(P, st), dt=st["dt"], vn=st["vn"], cs=st["cs"])
    P.les.step(fs, P.WindProfile(*gi.step_inflow(tag, dims[2])), n_iter=3, scheme=scheme)  # some other state first
    fs.stage(**{n: st[n].copy() for n in ALL})
    assert not bits_equal(fs.u, st["u"]), "staging does not change the state"
    fs.commit_staged()
    snaps = {}
    for s in range(1, n_steps + 1):
        P.les.step(fs, inflow, n_iter=gi.STEP_NITER[tag], scheme=scheme)
        if s == 1:
            snaps = fs.download_async({n: np.empty_like(st[n]) for n in FIELDS})
    for n in FIELDS:
        assert bits_equal(getattr(fs, n), GOLD[f"{tag}/step{n_steps}/{n}"]), (tag, n)
    out = snaps.wait()
    for n in FIELDS:
        assert bits_equal(out[n], GOLD[f"{tag}/step1/{n}"]), ("snapshot after step 1", tag, n)


def test_stage_argument_errors():
    import paper_1504_02264_b200 as P

    st = gi.step_state("st975", 9, 7, 5)
    fs = P.FlowState.create(grid_of(P, st), dt=st["dt"])
    with pytest.raises(ValueError):
        fs.stage(q=st["u"])
    with pytest.raises(ValueError):
        fs.stage(u=st["u"][:-1])
    with pytest.raises(ValueError):
        fs.download_async({"u": np.empty(st["u"].shape, np.float64)})
    with pytest.raises(ValueError):
        fs.download_async({"fgh": np.empty_like(st["u"])})
    fs.commit_staged()  # nothing staged: no-op


@pytest.mark.parametrize("chunk_mb", [None, "0.03", "0"])
def test_pipelined_windows_match_synchronous(monkeypatch, chunk_mb):
    """bench.py's e2e pattern at 64x48x32 with buildings: the next window's
    initial state staged during the current window, each window's fields
    downloaded asynchronously while the next runs -- against the same
    windows run with assignment and synchronous reads.  Copies in the
    default chunks (one per field here), in 30 KB chunks (many per field,
    pumped one per step, the rest flushed by commit / wait) and unchunked."""
    import paper_1504_02264_b200 as P

    if chunk_mb is not None:
        monkeypatch.setenv("LESB_COPY_CHUNK_MB", chunk_mb)

    st = gi.config2_state(64, 48, 32)
    rng = np.random.default_rng(5)
    inits = []
    for k in range(3):  # three different initial states, one per window
        d = {n: st[n].copy() for n in ALL}
        for n in ("u", "v", "w"):
            d[n][1:-1, 1:-1, 1:-1] = (0.01 * (k + 1) * rng.standard_normal(d[n][1:-1, 1:-1, 1:-1].shape)).astype(
                np.float32)
        inits.append(d)
    inflow = P.WindProfile(*gi.default_inflow(32))
    steps = 6
    grid = grid_of(P, st)

    ref = []
    fs = P.FlowState.create(grid, dt=0.5, vn=0.8, cs=0.14)
    for d in inits:
        for n in ALL:
            setattr(fs, n, d[n].copy())
        for _ in range(steps):
            P.les.step(fs, inflow)
        ref.append({n: getattr(fs, n).copy() for n in FIELDS})

    fs = P.FlowState.create(grid, dt=0.5, vn=0.8, cs=0.14)
    ins = [{n: pinned_like(d[n]) for n in ALL} for d in inits]
    for a, d in zip(ins, inits):
        for n in ALL:
            a[n][...] = d[n]
    outs = [{n: pinned_like(st[n]) for n in FIELDS} for _ in inits]
    pend = []
    fs.stage(**ins[0])
    for w in range(len(inits)):
        fs.commit_staged()
        P.les.step(fs, inflow)
        if w + 1 < len(inits):
            fs.stage(**ins[w + 1])
        for _ in range(steps - 1):
            P.les.step(fs, inflow)
        pend.append(fs.download_async(outs[w]))
    for w, p in enumerate(pend):
        got = p.wait()
        for n in FIELDS:
            assert bits_equal(got[n], ref[w][n]), (w, n)
    for n in ALL:  # the staged inputs were not written to
        for a, d in zip(ins, inits):
            assert bits_equal(a[n], d[n])
