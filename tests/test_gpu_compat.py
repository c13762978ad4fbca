"""The real drop-in path: the reference's callers hand the rebound functions
the reference's OWN numpy FlowState (cli.run_les_standalone -> les.step,
cli.py:208; the reference tests; les_main).  That state is a non-frozen
@dataclass (les.py:36-71: unhashable, plain numpy arrays), so these tests
drive a look-alike dataclass -- and gmcf_mini's own FlowState when the
reference is importable (baseline/_ref on the GPU box) -- through step,
press, every stage, solve_pressure, redblack_iteration and twinned_sweep,
i.e. through the compat path (les._resolve / les._writeback: upload, run,
copy the written fields back into the caller's arrays).  Bitwise against
the reference's golden vectors, as test_gpu_parity does for the device
FlowState.
"""

from __future__ import annotations

import hashlib
import json
import os
from dataclasses import dataclass, field

import numpy as np
import pytest

import golden_inputs as gi

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = np.load(os.path.join(HERE, "golden", "small.npz"))
META = json.load(open(os.path.join(HERE, "golden", "golden_meta.json")))
FIELDS = ("u", "v", "w", "fgh", "fgh_old", "p")
RTOL_RES = 1e-12


@dataclass
class RefShapedState:
    """Same fields, defaults and methods as gmcf_mini.les.FlowState
    (les.py:36-71); like it, unhashable (``@dataclass`` sets __hash__ = None)."""

    u: np.ndarray
    v: np.ndarray
    w: np.ndarray
    fgh: np.ndarray
    fgh_old: np.ndarray
    p: np.ndarray
    mask: np.ndarray
    grid: object
    dt: float
    vn: float = 1e-5
    cs: float = 0.14
    _coeffs: object = field(default=None, repr=False)

    @classmethod
    def create(cls, grid, dt, vn=1e-5, cs=0.14):
        shape = (grid.im + 2, grid.jm + 2, grid.km + 2)
        z = lambda: np.zeros(shape, np.float32)  # noqa: E731
        return cls(z(), z(), z(), np.zeros(shape + (3,), np.float32), np.zeros(shape + (3,), np.float32), z(),
                   z(), grid, dt, vn, cs)

    def coeffs(self):
        if self._coeffs is None:
            import paper_1504_02264_b200 as P

            self._coeffs = P.sor.build_uniform_coeffs(self.grid)
        return self._coeffs

    def velocities(self):
        return self.u, self.v, self.w


def _state_classes():
    out = [RefShapedState]
    try:
        from gmcf_mini.les import FlowState as RefFS  # baseline/_ref on the box

        out.append(RefFS)
    except ImportError:
        pass
    return out


@pytest.fixture(params=_state_classes(), ids=lambda c: c.__module__ + "." + c.__name__)
def SC(request):
    return request.param


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def bits_equal(a, b):
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.uint32), b.view(np.uint32))


def hstate(SC, st):
    import paper_1504_02264_b200 as P

    g = P.Grid(st["im"], st["jm"], st["km"], st["dx1"], st["dy1"], st["dzn"])
    fs = SC.create(g, dt=st["dt"], vn=st["vn"], cs=st["cs"])
    for n in FIELDS + ("mask",):
        getattr(fs, n)[...] = st[n]
    return fs


def test_unhashable(SC):
    g = gi.random_state(3, 2, 1, seed=1)
    fs = hstate(SC, g)
    with pytest.raises(TypeError):
        hash(fs)


@pytest.mark.parametrize("tag,dims,uniform", gi.STAGE_CASES)
def test_stages_compat_bitwise(SC, tag, dims, uniform):
    import paper_1504_02264_b200 as P

    st = gi.random_state(*dims, seed=gi.seed_of(tag), uniform=uniform)
    inflow = P.WindProfile(*gi.random_inflow(dims[2], seed=gi.seed_of(tag) + 1))
    calls = {
        "velnw": P.les.velnw,
        "bondv1": lambda fs: P.les.bondv1(fs, inflow),
        "velfg": P.les.velfg_merged,
        "feedbf": P.les.feedbf,
        "les": P.les.les_viscosity,
        "adam": P.les.adam,
    }
    if uniform:
        calls["press"] = lambda fs: P.les.press(fs, n_iter=7)
        calls["press_tw"] = lambda fs: P.les.press(fs, n_iter=7, scheme=P.Scheme.TWINNED)
    for name, fn in calls.items():
        fs = hstate(SC, st)
        ids = {n: id(getattr(fs, n)) for n in FIELDS}
        res = fn(fs)
        for n in FIELDS:
            assert id(getattr(fs, n)) == ids[n], "stages mutate the caller's arrays in place"
            assert bits_equal(getattr(fs, n), GOLD[f"{tag}/{name}/{n}"]), (tag, name, n)
        if name.startswith("press"):
            np.testing.assert_allclose(res, GOLD[f"{tag}/{name}/res"], rtol=RTOL_RES, atol=0)
    fs = hstate(SC, st)
    assert bits_equal(P.les.divergence(fs), GOLD[f"{tag}/divergence"])
    assert bits_equal(P.les.strain_magnitude(fs), GOLD[f"{tag}/strain"])


@pytest.mark.parametrize("tag,dims,n_steps", gi.STEP_CASES)
def test_step_compat_bitwise(SC, tag, dims, n_steps):
    import paper_1504_02264_b200 as P

    fs = hstate(SC, gi.step_state(tag, *dims))
    inflow = P.WindProfile(*gi.step_inflow(tag, dims[2]))
    scheme = P.Scheme(gi.STEP_SCHEME[tag])
    for s in range(1, n_steps + 1):
        assert P.les.step(fs, inflow, n_iter=gi.STEP_NITER[tag], scheme=scheme) is fs
        if s in (1, n_steps):
            for n in FIELDS:
                assert bits_equal(getattr(fs, n), GOLD[f"{tag}/step{s}/{n}"]), (tag, s, n)


def test_config1_compat_anchors_and_blowup(SC):
    """Config 1 through the compat path: the reference's hashes at steps 1
    and 10 and NumericsError('velfg') at step 17 -- with the host arrays
    modified between steps (the compat path re-uploads every call)."""
    import paper_1504_02264_b200 as P

    meta = META["config1"]
    fs = hstate(SC, gi.config1_state())
    inflow = P.WindProfile(*gi.default_inflow(16))
    step = 0
    with pytest.raises(P.NumericsError) as err:
        while step < 40:
            P.les.step(fs, inflow)
            step += 1
            if step in (1, 10):
                for n in FIELDS:
                    assert sha(getattr(fs, n)) == meta[f"step{step}"][n], (step, n)
    assert step + 1 == meta["blowup"]["step"]
    assert err.value.stage == meta["blowup"]["stage"]


def test_host_edit_between_steps_is_seen(SC):
    """A caller that edits its arrays between steps (as the reference's tests
    do) gets the same result as a fresh state carrying the edit."""
    import paper_1504_02264_b200 as P

    inflow = P.WindProfile(*gi.default_inflow(16))
    a = hstate(SC, gi.config1_state())
    P.les.step(a, inflow)
    a.u[5, 5, 5] += 0.25
    a.p[...] = 0.0
    snap = {n: getattr(a, n).copy() for n in FIELDS + ("mask",)}
    P.les.step(a, inflow)
    b = P.FlowState.create(a.grid, dt=a.dt, vn=a.vn, cs=a.cs)
    for n, v in snap.items():
        getattr(b, n)[...] = v
    P.les.step(b, inflow)
    for n in FIELDS:
        assert bits_equal(getattr(a, n), getattr(b, n)), n


@pytest.mark.parametrize("tag,dims,h", gi.SOR_CASES)
def test_sor_entry_points_numpy(tag, dims, h):
    """solve_pressure / redblack_iteration / twinned_sweep take plain numpy
    arrays (sor.py:162-309): p0 untouched, p and tp mutated in place."""
    import paper_1504_02264_b200 as P

    p0, rhs = gi.sor_problem(*dims, seed=gi.seed_of(tag))
    grid = P.Grid.uniform(*dims, h)
    c = P.sor.build_uniform_coeffs(grid)
    halo = P.les._pressure_halo(grid)
    p0c = p0.copy()
    p, res = P.sor.solve_pressure(p0c, rhs, c, 1.7, 9, P.Scheme.REDBLACK, 1, halo_fn=halo)
    assert bits_equal(p0c, p0)
    assert bits_equal(p, GOLD[f"{tag}/redblack/press/p"])
    p = p0.copy()
    pid = id(p)
    r = P.sor.redblack_iteration(p, rhs, c, 1.7, halo)
    assert id(p) == pid and bits_equal(p, GOLD[f"{tag}/rbiter/p"])
    np.testing.assert_allclose(r, GOLD[f"{tag}/rbiter/res"][0], rtol=RTOL_RES)
    tp = GOLD[f"{tag}/twsweep/in"].copy()
    r = P.sor.twinned_sweep(tp, rhs, c, 1.0, 1)
    assert bits_equal(tp, GOLD[f"{tag}/twsweep/out"])
    np.testing.assert_allclose(r, GOLD[f"{tag}/twsweep/res"][0], rtol=RTOL_RES)


def test_installed_reference_step(SC):
    """With install(), the reference module's own ``les.step`` is the device
    step and works on the caller's state (cli.py:208's call)."""
    gl = pytest.importorskip("gmcf_mini.les")
    import paper_1504_02264_b200 as P

    P.install()
    try:
        assert gl.step is P.les.step
        fs = hstate(SC, gi.config1_state())
        inflow = P.WindProfile(*gi.default_inflow(16))
        gl.step(fs, inflow)
        for n in FIELDS:
            assert sha(getattr(fs, n)) == META["config1"]["step1"][n], n
    finally:
        P.uninstall()
