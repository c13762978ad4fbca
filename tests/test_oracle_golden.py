"""Pin the CPU oracle (oracle/les_oracle.py) against golden vectors produced
by the unmodified reference (tests/golden/make_golden.py).  CPU only."""

import hashlib
import json
import os

import numpy as np
import pytest

import golden_inputs as gi
from oracle import les_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = np.load(os.path.join(HERE, "golden", "small.npz"))
META = json.load(open(os.path.join(HERE, "golden", "golden_meta.json")))
FIELDS = O.FIELDS


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def ostate(st):
    o = O.OState.zeros(st["im"], st["jm"], st["km"], dt=st["dt"], vn=st["vn"], cs=st["cs"])
    for n in FIELDS + ("mask", "dx1", "dy1", "dzn"):
        getattr(o, n)[...] = st[n]
    return o


def assert_state(o, prefix):
    for n in FIELDS:
        exp = GOLD[prefix + n]
        got = getattr(o, n)
        assert np.array_equal(got.view(np.uint32), exp.view(np.uint32)), f"{prefix}{n}"


@pytest.mark.parametrize("tag,dims,uniform", gi.STAGE_CASES)
def test_oracle_stages_bitwise(tag, dims, uniform):
    st = gi.random_state(*dims, seed=gi.seed_of(tag), uniform=uniform)
    inflow = gi.random_inflow(dims[2], seed=gi.seed_of(tag) + 1)
    calls = {
        "velnw": O.velnw,
        "bondv1": lambda o: O.bondv1(o, *inflow),
        "velfg": O.velfg,
        "feedbf": O.feedbf,
        "les": O.les_viscosity,
        "adam": O.adam,
    }
    if uniform:
        calls["press"] = lambda o: O.press(o, n_iter=7)
        calls["press_tw"] = lambda o: O.press(o, n_iter=7, scheme="twinned")
    for name, fn in calls.items():
        o = ostate(st)
        res = fn(o)
        assert_state(o, f"{tag}/{name}/")
        if name.startswith("press"):
            np.testing.assert_allclose(res, GOLD[f"{tag}/{name}/res"], rtol=1e-12, atol=0)
    o = ostate(st)
    assert np.array_equal(O.divergence(o), GOLD[f"{tag}/divergence"])
    assert np.array_equal(O.strain_magnitude(o), GOLD[f"{tag}/strain"])


@pytest.mark.parametrize("tag,dims,h", gi.SOR_CASES)
def test_oracle_sor_bitwise(tag, dims, h):
    p0, rhs = gi.sor_problem(*dims, seed=gi.seed_of(tag))
    c = O.uniform_coeffs(*dims, h)
    for scheme, om in (("redblack", 1.7), ("twinned", 1.0)):
        for pol in ("stored", "press"):
            p, res = O.solve_pressure(p0, rhs, c, om, 9, scheme, None if pol == "stored" else "press")
            assert np.array_equal(p, GOLD[f"{tag}/{scheme}/{pol}/p"]), (scheme, pol)
            np.testing.assert_allclose(res, GOLD[f"{tag}/{scheme}/{pol}/res"], rtol=1e-12, atol=0)
    p = p0.copy()
    r = O.rb_iteration(p, rhs, c, 1.7, "press")
    assert np.array_equal(p, GOLD[f"{tag}/rbiter/p"])
    np.testing.assert_allclose(r, GOLD[f"{tag}/rbiter/res"][0], rtol=1e-12)
    tp = GOLD[f"{tag}/twsweep/in"].copy()
    src = np.ascontiguousarray(tp[..., 1])
    dst = np.ascontiguousarray(tp[..., 0])
    r = O.tw_sweep(src, dst, rhs, c, 1.0)
    assert np.array_equal(dst, GOLD[f"{tag}/twsweep/out"][..., 0])
    np.testing.assert_allclose(r, GOLD[f"{tag}/twsweep/res"][0], rtol=1e-12)


@pytest.mark.parametrize("tag,dims,n_steps", gi.STEP_CASES)
def test_oracle_step_bitwise(tag, dims, n_steps):
    o = ostate(gi.step_state(tag, *dims))
    inflow = gi.step_inflow(tag, dims[2])
    assert np.array_equal(np.stack(inflow), GOLD[f"{tag}/inflow"])
    for s in range(1, n_steps + 1):
        O.step(o, *inflow, n_iter=gi.STEP_NITER[tag], scheme=gi.STEP_SCHEME[tag])
        if s in (1, n_steps):
            assert_state(o, f"{tag}/step{s}/")


def test_oracle_config1_anchors_and_blowup():
    """32x32x16 with one building: hashes at steps 1 and 10 and the blow-up
    at step 17 in velfg (probe P4/P7)."""
    meta = META["config1"]
    o = ostate(gi.config1_state())
    inflow = gi.default_inflow(16)
    assert sha(np.stack(inflow)) == META["default_inflow16_sha"]
    step = 0
    with pytest.raises(O.OracleNumericsError) as err:
        while step < 40:
            O.step(o, *inflow)
            step += 1
            if step in (1, 10):
                for n in FIELDS:
                    assert sha(getattr(o, n)) == meta[f"step{step}"][n], (step, n)
    assert step + 1 == meta["blowup"]["step"]
    assert err.value.stage == meta["blowup"]["stage"] == "velfg"


def test_oracle_press_halo_idempotent():
    rng = np.random.default_rng(3)
    p = rng.uniform(-1, 1, size=(11, 9, 7)).astype(np.float32)
    O.press_halo(p)
    q = p.copy()
    O.press_halo(q)
    assert np.array_equal(p, q)


def test_oracle_hand_cases():
    """1x1x1 hand case (test_sor.py:137-146): p=1, residual 1, both schemes."""
    c = O.uniform_coeffs(1, 1, 1, 1.0)
    p0 = np.zeros((3, 3, 3), np.float32)
    rhs = np.zeros_like(p0)
    rhs[1, 1, 1] = -6.0
    for scheme in ("redblack", "twinned"):
        p, res = O.solve_pressure(p0, rhs, c, 1.0, 1, scheme, None)
        assert p[1, 1, 1] == np.float32(1.0)
        assert res[0] == 1.0 if scheme == "redblack" else res[0] >= 1.0
