"""SURVEY 8(f) rows 2 and 3 on the GPU: the sor-bench and les-standalone CLI
modes (cli.py:202-283) with the device runners installed, against the
unmodified reference CLI run on the host (baseline/_ref; skipped when the
reference is not importable), and GMCF dumps of a device FlowState against
the reference's writer (dump.py:16-27).

* les-standalone: the four field dumps are byte-identical to the
  reference's (the device steps are bitwise equal to les.step);
* sor-bench: residual CSVs equal the reference's rows to rtol 1e-12 (the
  float64 sums differ only in summation order), the reference's files and
  summary keys are all there, ``residuals_worker_invariant`` holds, and the
  device x-slab table's GPU-count invariance check passes (p bitwise equal
  for 1/2/4/8 slabs, residuals within rtol 1e-12).
"""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

import golden_inputs as gi

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

SOR_BENCH = """\
[runtime]
mode = sor-bench
seed = 3

[les]
im = {im}
jm = {jm}
km = {km}

[sor]
scheme = twinned
n_iter = {n_iter}
workers = 4
"""

STANDALONE = """\
[runtime]
mode = les-standalone
models = les:0.5
n_steps = {steps}

[les]
im = {im}
jm = {jm}
km = {km}

[sor]
n_iter = 20
"""


def _run(args, cwd, device: bool):
    """One CLI run in a fresh interpreter: the device runners
    (python -m paper_1504_02264_b200) or the unmodified reference."""
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([ROOT, REF, env.get("PYTHONPATH", "")])
    if device:
        cmd = [sys.executable, "-m", "paper_1504_02264_b200", *args]
    else:
        cmd = [sys.executable, "-c", "import sys; from gmcf_mini.cli import main; sys.exit(main(sys.argv[1:]))", *args]
    return subprocess.run(cmd, cwd=cwd, env=env, capture_output=True, text=True, timeout=900)


@pytest.fixture(scope="module")
def have_ref():
    if not os.path.isdir(os.path.join(REF, "gmcf_mini")):
        pytest.skip("reference not installed (scripts/install_reference.sh)")


def _csv(path):
    rows = open(path).read().strip().splitlines()
    return rows[0], np.array([float(r.split(",")[1]) for r in rows[1:]])


@pytest.mark.parametrize("dims,n_iter", [((24, 12, 8), 15), ((40, 33, 17), 9)])
def test_sor_bench_matches_reference(have_ref, tmp_path, dims, n_iter):
    cfg = tmp_path / "run.ini"
    cfg.write_text(SOR_BENCH.format(im=dims[0], jm=dims[1], km=dims[2], n_iter=n_iter))
    outs = {}
    for dev in (True, False):
        out = tmp_path / ("dev" if dev else "ref")
        r = _run(["sor-bench", "--config", str(cfg), "--out", str(out)], tmp_path, dev)
        assert r.returncode == 0, r.stdout + r.stderr
        outs[dev] = out
    for name in ("redblack_residuals.csv", "twinned_residuals.csv"):
        hd, vd = _csv(outs[True] / name)
        hr, vr = _csv(outs[False] / name)
        assert hd == hr and vd.shape == vr.shape == (n_iter,)
        np.testing.assert_allclose(vd, vr, rtol=1e-12, atol=0)
    assert (outs[True] / "sor_bench_times.csv").read_text().splitlines()[0] == "scheme,workers,seconds"
    sd = json.loads((outs[True] / "summary.json").read_text())
    sr = json.loads((outs[False] / "summary.json").read_text())
    assert set(sr) <= set(sd)
    for k in ("mode", "domain", "n_iter", "worker_counts"):
        assert sd[k] == sr[k], k
    assert sd["residuals_worker_invariant"] is True
    inv = sd["device"]["gpu_count_invariance"]
    assert sd["device"]["slab_counts"] == [1, 2, 4, 8]
    for scheme in ("redblack", "twinned"):
        assert inv[scheme]["p_bitwise"], scheme
        assert inv[scheme]["residuals_within_rtol_1e-12"], inv[scheme]


def test_les_standalone_dumps_bytewise(have_ref, tmp_path):
    cfg = tmp_path / "run.ini"
    cfg.write_text(STANDALONE.format(steps=6, im=20, jm=12, km=10))
    outs = {}
    for dev in (True, False):
        out = tmp_path / ("dev" if dev else "ref")
        r = _run(["les-standalone", "--config", str(cfg), "--out", str(out)], tmp_path, dev)
        assert r.returncode == 0, r.stdout + r.stderr
        outs[dev] = out
    for n in ("u", "v", "w", "p"):
        a = (outs[True] / f"{n}.gmcf").read_bytes()
        b = (outs[False] / f"{n}.gmcf").read_bytes()
        assert a == b, n
    sd = json.loads((outs[True] / "summary.json").read_text())
    sr = json.loads((outs[False] / "summary.json").read_text())
    assert sd["steps"] == sr["steps"] and sd["max_abs_u"] == sr["max_abs_u"]


def test_les_standalone_blowup_exit_code(have_ref, tmp_path):
    """A numerical blow-up exits 4 with the reference's message prefix
    (cli.py:379-381): config 1's buildings are absent here, so force it
    with a huge dt."""
    cfg = tmp_path / "run.ini"
    cfg.write_text(STANDALONE.format(steps=40, im=8, jm=8, km=8).replace("les:0.5", "les:1e30"))
    r = _run(["les-standalone", "--config", str(cfg), "--out", str(tmp_path / "o")], tmp_path, True)
    ref = _run(["les-standalone", "--config", str(cfg), "--out", str(tmp_path / "r")], tmp_path, False)
    assert r.returncode == ref.returncode
    if ref.returncode == 4:
        assert "numerical error" in r.stderr


def test_write_state_device_bytes_equal_reference_writer(tmp_path):
    """dump.write_state of a device FlowState (pitched D2H of the
    Python-visible arrays) writes the reference writer's exact bytes for the
    reference's arrays: checked against the config-1 step-10 golden hashes'
    state recomputed by the oracle and written with the format rules."""
    import paper_1504_02264_b200 as P
    from oracle import les_oracle as O

    st = gi.config1_state()
    g = P.Grid(32, 32, 16, st["dx1"], st["dy1"], st["dzn"])
    fs = P.FlowState.create(g, dt=st["dt"], vn=st["vn"], cs=st["cs"])
    o = O.OState.zeros(32, 32, 16)
    for n in ("u", "v", "w", "fgh", "fgh_old", "p", "mask"):
        getattr(fs, n)[...] = st[n]
        getattr(o, n)[...] = st[n]
    for n in ("dx1", "dy1", "dzn"):
        getattr(o, n)[...] = st[n]
    inflow = gi.default_inflow(16)
    P.les.run_steps(fs, P.WindProfile(*inflow), 3)
    for _ in range(3):
        O.step(o, *inflow)
    paths = P.dump.write_state(fs, tmp_path)
    try:
        sys.path.append(REF)
        from gmcf_mini import dump as rdump
    except ImportError:
        rdump = None
    for path in paths:
        n = path.stem
        exp = b"GMCF" + np.asarray(getattr(o, n).shape, "<u4").tobytes() + np.ascontiguousarray(
            getattr(o, n), "<f4").tobytes()
        assert path.read_bytes() == exp, n
        if rdump is not None:
            rp = tmp_path / f"ref_{n}.gmcf"
            rdump.write_field(rp, getattr(o, n))
            assert rp.read_bytes() == path.read_bytes(), n


def test_checkpoint_resume_bitwise(tmp_path):
    """Checkpoint / resume of a device FlowState: 3 steps, write_checkpoint,
    a fresh FlowState restored with read_checkpoint, 3 more steps -- bitwise
    equal to 6 uninterrupted steps (the reference has final dumps only; this
    is the resume half SURVEY 5 lists)."""
    import paper_1504_02264_b200 as P

    st = gi.config1_state()
    g = P.Grid(32, 32, 16, st["dx1"], st["dy1"], st["dzn"])
    inflow = P.WindProfile(*gi.default_inflow(16))

    def fresh():
        fs = P.FlowState.create(g, dt=st["dt"], vn=st["vn"], cs=st["cs"])
        for n in ("u", "v", "w", "fgh", "fgh_old", "p", "mask"):
            getattr(fs, n)[...] = st[n]
        return fs

    straight = fresh()
    P.les.run_steps(straight, inflow, 6)
    first = fresh()
    P.les.run_steps(first, inflow, 3)
    P.dump.write_checkpoint(first, tmp_path / "ck")
    resumed = P.FlowState.create(g, dt=st["dt"], vn=st["vn"], cs=st["cs"])
    P.dump.read_checkpoint(resumed, tmp_path / "ck")
    P.les.run_steps(resumed, inflow, 3)
    for n in ("u", "v", "w", "fgh", "fgh_old", "p"):
        a, b = getattr(straight, n), getattr(resumed, n)
        assert np.array_equal(np.ascontiguousarray(a).view(np.uint32), np.ascontiguousarray(b).view(np.uint32)), n
