"""Generate golden vectors from the UNMODIFIED reference (gmcf_mini).

Run in the build container, where the reference is importable:

    python tests/golden/make_golden.py            # small fixtures (seconds)
    python tests/golden/make_golden.py --large    # 150x150x90 anchors (minutes)

The reference is imported from /root/reference/pkg/src (or baseline/_ref);
nothing here travels to the GPU box except the .npz/.json outputs, which the
tests read.  Inputs are regenerated in the tests from the same seeds and
also stored, so a test can check that it rebuilt the same inputs.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
for cand in ("/root/reference/pkg/src", os.path.join(HERE, "..", "..", "baseline", "_ref")):
    if os.path.isdir(cand):
        sys.path.insert(0, cand)
        break

from gmcf_mini import les, sor  # noqa: E402
from gmcf_mini.coupling import WindProfile  # noqa: E402
from gmcf_mini.driver import DriverConfig, generate_profile  # noqa: E402
from gmcf_mini.errors import NumericsError  # noqa: E402
from gmcf_mini.les import FlowState  # noqa: E402
from gmcf_mini.sor import Grid, Scheme  # noqa: E402

sys.path.insert(0, os.path.join(HERE, ".."))
import golden_inputs as gi  # noqa: E402

FIELDS = ("u", "v", "w", "fgh", "fgh_old", "p")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]


def to_flow(st: dict) -> FlowState:
    g = Grid(st["im"], st["jm"], st["km"], st["dx1"], st["dy1"], st["dzn"])
    fs = FlowState.create(g, dt=st["dt"], vn=st["vn"], cs=st["cs"])
    for n in FIELDS + ("mask",):
        getattr(fs, n)[...] = st[n]
    return fs


def dump_state(fs: FlowState, prefix: str, out: dict):
    for n in FIELDS:
        out[f"{prefix}{n}"] = getattr(fs, n).copy()


def stage_cases(out: dict):
    """Each stage alone on random states with random halos."""
    for tag, (im, jm, km), uniform in gi.STAGE_CASES:
        st = gi.random_state(im, jm, km, seed=gi.seed_of(tag), uniform=uniform)
        inflow = gi.random_inflow(km, seed=gi.seed_of(tag) + 1)
        calls = {
            "velnw": lambda fs: les.velnw(fs),
            "bondv1": lambda fs: les.bondv1(fs, WindProfile(*inflow)),
            "velfg": lambda fs: les.velfg_merged(fs),
            "feedbf": lambda fs: les.feedbf(fs),
            "les": lambda fs: les.les_viscosity(fs),
            "adam": lambda fs: les.adam(fs),
        }
        if uniform:
            calls["press"] = lambda fs: out.__setitem__(f"{tag}/press/res", les.press(fs, n_iter=7))
            calls["press_tw"] = lambda fs: out.__setitem__(
                f"{tag}/press_tw/res", les.press(fs, n_iter=7, scheme=Scheme.TWINNED))
        for name, fn in calls.items():
            fs = to_flow(st)
            fn(fs)
            dump_state(fs, f"{tag}/{name}/", out)
        fs = to_flow(st)
        out[f"{tag}/divergence"] = les.divergence(fs)
        out[f"{tag}/strain"] = les.strain_magnitude(fs)


def sor_cases(out: dict):
    """solve_pressure over schemes x halo policies."""
    for tag, (im, jm, km), h in gi.SOR_CASES:
        p0, rhs = gi.sor_problem(im, jm, km, seed=gi.seed_of(tag))
        c = sor.build_uniform_coeffs(Grid.uniform(im, jm, km, h))
        halo = les._pressure_halo(Grid.uniform(im, jm, km, h))
        for scheme, om in ((Scheme.REDBLACK, 1.7), (Scheme.TWINNED, 1.0)):
            for pol, fn in (("stored", None), ("press", halo)):
                p, res = sor.solve_pressure(p0, rhs, c, om, 9, scheme, 1, halo_fn=fn)
                out[f"{tag}/{scheme.value}/{pol}/p"] = p
                out[f"{tag}/{scheme.value}/{pol}/res"] = res
        # single iteration / sweep entry points
        p = p0.copy()
        out[f"{tag}/rbiter/res"] = np.array([sor.redblack_iteration(p, rhs, c, 1.7, halo)])
        out[f"{tag}/rbiter/p"] = p
        tp = sor.make_twinned(p0)
        tp[..., 1] = gi.sor_problem(im, jm, km, seed=gi.seed_of(tag) + 7)[0]
        out[f"{tag}/twsweep/in"] = tp.copy()
        out[f"{tag}/twsweep/res"] = np.array([sor.twinned_sweep(tp, rhs, c, 1.0, 1)])
        out[f"{tag}/twsweep/out"] = tp


def step_cases(out: dict, meta: dict):
    """Whole-step parity on small grids: full arrays."""
    for tag, (im, jm, km), n_steps in gi.STEP_CASES:
        st = gi.step_state(tag, im, jm, km)
        fs = to_flow(st)
        inflow = WindProfile(*gi.step_inflow(tag, km))
        meta[tag] = {"steps": n_steps}
        for s in range(1, n_steps + 1):
            try:
                les.step(fs, inflow, n_iter=gi.STEP_NITER[tag], scheme=Scheme(gi.STEP_SCHEME[tag]))
            except NumericsError as e:
                meta[tag]["blowup"] = {"step": s, "stage": e.stage}
                break
            if s in (1, n_steps):
                dump_state(fs, f"{tag}/step{s}/", out)
        out[f"{tag}/inflow"] = np.stack([inflow.u, inflow.v, inflow.w])


def config1(meta: dict):
    """Config 1 anchors: 32x32x16, one building, 50 RB iterations."""
    st = gi.config1_state()
    fs = to_flow(st)
    prof = generate_profile(DriverConfig(16, 0.05, 0.1, 0.1 + 2.0 * np.arange(1, 17), 0.2, 600.0), 0.0)
    meta["default_inflow16_sha"] = sha(np.stack([prof.u, prof.v, prof.w]))
    inflow = WindProfile(*gi.default_inflow(16))
    rec = {}
    step = 0
    try:
        while step < 40:
            les.step(fs, inflow)
            step += 1
            if step in (1, 10):
                rec[f"step{step}"] = {n: sha(getattr(fs, n)) for n in FIELDS}
                rec[f"step{step}"]["max_abs_u"] = float(np.abs(fs.u).max())
                rec[f"step{step}"]["sum_u"] = float(fs.u.astype(np.float64).sum())
    except NumericsError as e:
        rec["blowup"] = {"step": step + 1, "stage": e.stage}
    meta["config1"] = rec


def large(meta: dict):
    t0 = time.time()
    # press-only 150x150x90 anchors, h = 1
    im, jm, km = 150, 150, 90
    rng = np.random.default_rng(0)
    rhs = sor.make_field(im, jm, km)
    rhs[1:-1, 1:-1, 1:-1] = rng.uniform(-1, 1, size=(im, jm, km)).astype(np.float32)
    p0 = sor.make_field(im, jm, km)
    c = sor.build_uniform_coeffs(Grid.uniform(im, jm, km, 1.0))
    halo = les._pressure_halo(Grid.uniform(im, jm, km, 1.0))
    rec = {}
    for name, scheme, om, fn in (("rb_zero", Scheme.REDBLACK, 1.7, None),
                                 ("rb_press", Scheme.REDBLACK, 1.7, halo),
                                 ("tw_zero", Scheme.TWINNED, 1.0, None)):
        p, res = sor.solve_pressure(p0, rhs, c, om, 50, scheme, 1, halo_fn=fn)
        rec[name] = {"sha_p": sha(p), "res": [float(x) for x in res]}
        print(name, rec[name]["sha_p"], res[0], res[-1], f"{time.time()-t0:.0f}s", flush=True)
    meta["press150"] = rec
    # config 2: 150x150x90 with the 3x3 building array, 10 steps
    st = gi.config2_state()
    fs = to_flow(st)
    inflow = WindProfile(*gi.default_inflow(90))
    rec = {}
    for s in range(1, 11):
        les.step(fs, inflow)
        if s in (1, 10):
            rec[f"step{s}"] = {n: sha(getattr(fs, n)) for n in FIELDS}
        print("config2 step", s, f"{time.time()-t0:.0f}s", flush=True)
    meta["config2"] = rec


def blowups(meta: dict):
    """Blow-up step and stage at full size (probes P4/P10):
    config 2 with buildings and the building-free 150x150x90 flow."""
    t0 = time.time()
    for name, st in (("config2", gi.config2_state()), ("free150", gi.zero_state(150, 150, 90))):
        fs = to_flow(st)
        inflow = WindProfile(*gi.default_inflow(90))
        rec = {}
        for s in range(1, 80):
            try:
                les.step(fs, inflow)
            except NumericsError as e:
                rec = {"step": s, "stage": e.stage}
                break
        meta[f"blowup_{name}"] = rec
        print(name, rec, f"{time.time()-t0:.0f}s", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--large", action="store_true")
    ap.add_argument("--blowup", action="store_true")
    args = ap.parse_args()
    meta_path = os.path.join(HERE, "golden_meta.json")
    meta = json.load(open(meta_path)) if os.path.exists(meta_path) else {}
    if args.blowup:
        blowups(meta)
    elif args.large:
        large(meta)
    else:
        out: dict = {}
        stage_cases(out)
        sor_cases(out)
        step_cases(out, meta)
        config1(meta)
        np.savez_compressed(os.path.join(HERE, "small.npz"), **out)
        print("wrote", len(out), "arrays")
    with open(meta_path, "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
