"""Boundary-range launch geometry (reference sor.py:312-349, cli.py:286-320;
SURVEY 8(f) row 4).

CPU: the host functions follow the reference (against gmcf_mini itself when
it is importable, and against an independent enumeration of the three face
families otherwise) including the error contract.
GPU: the device decode equals map_boundary_gid gid for gid over the padded
range, the device audit reports full coverage / a tight padding guard, the
boundary-audit runner prints and writes what the reference does, and the
face refresh launched over the geometry equals the reference pressure halo
(les.py:341-355) on every face-interior halo cell while leaving edges alone.
"""

import json
import types

import numpy as np
import pytest

from paper_1504_02264_b200 import sor as S
from paper_1504_02264_b200.reftypes import PADDING, Face

DOMAINS = [(1, 1, 1), (3, 4, 5), (7, 2, 9), (16, 16, 8), (150, 150, 90)]


def families(ip, jp, kp):
    """The boundary points in gid order, enumerated independently."""
    pts = [(Face.YZ, (j, k)) for k in range(kp) for j in range(jp)]
    pts += [(Face.ZX, (k, i)) for k in range(kp) for i in range(ip)]
    pts += [(Face.XY, (j, i)) for j in range(jp) for i in range(ip)]
    return pts


@pytest.mark.parametrize("dom", DOMAINS[:4])
def test_host_decode_matches_face_families(dom):
    ip, jp, kp = dom
    br = S.boundary_range(ip, jp, kp)
    pts = families(ip, jp, kp)
    assert br == len(pts) == jp * kp + kp * ip + jp * ip
    for gid, (f, c) in enumerate(pts):
        bp = S.map_boundary_gid(gid, ip, jp, kp)
        assert bp.face == f and bp.coords == c
    for gid in range(br, S.padded_range(br, 32, 3)):
        assert S.map_boundary_gid(gid, ip, jp, kp) is PADDING


def test_host_padding_and_errors():
    assert S.padded_range(0, 4, 2) == 0
    assert S.padded_range(8, 4, 2) == 8
    assert S.padded_range(9, 4, 2) == 16
    with pytest.raises(ValueError, match="ip, jp, kp must be >= 1"):
        S.boundary_range(0, 1, 1)
    with pytest.raises(ValueError, match="gid must be >= 0"):
        S.map_boundary_gid(-1, 1, 1, 1)
    with pytest.raises(ValueError, match="range must be >= 0"):
        S.padded_range(-1, 1, 1)
    with pytest.raises(ValueError, match="nthreads and nunits must be >= 1"):
        S.padded_range(1, 0, 1)


def test_host_functions_match_reference():
    import os
    import sys

    src = "/root/reference/pkg/src"  # CPU test only (the reference is not on the GPU box)
    if os.path.isdir(src) and src not in sys.path:
        sys.path.append(src)
    ref = pytest.importorskip("gmcf_mini.sor")
    for ip, jp, kp in DOMAINS[:4]:
        assert S.boundary_range(ip, jp, kp) == ref.boundary_range(ip, jp, kp)
        for nt, nu in ((1, 1), (32, 2), (128, 4)):
            br = ref.boundary_range(ip, jp, kp)
            assert S.padded_range(br, nt, nu) == ref.padded_range(br, nt, nu)
        for gid in range(S.padded_range(S.boundary_range(ip, jp, kp), 16, 1)):
            a = S.map_boundary_gid(gid, ip, jp, kp)
            b = ref.map_boundary_gid(gid, ip, jp, kp)
            if b is ref.PADDING:
                assert a is PADDING
            else:
                assert (a.face.value, a.coords) == (b.face.value, b.coords)


@pytest.mark.gpu
@pytest.mark.parametrize("dom", DOMAINS)
def test_device_decode_matches_host(dom):
    ip, jp, kp = dom
    br = S.boundary_range(ip, jp, kp)
    pr = S.padded_range(br, 256, 1)
    face, c0, c1 = S.boundary_decode(ip, jp, kp, 0, pr)
    pts = families(ip, jp, kp)
    codes = {Face.YZ: 0, Face.ZX: 1, Face.XY: 2}
    want_f = np.array([codes[f] for f, _ in pts] + [-1] * (pr - br), np.int32)
    want_c = np.array([c for _, c in pts] + [(-1, -1)] * (pr - br), np.int32).reshape(-1, 2)
    np.testing.assert_array_equal(face, want_f)
    np.testing.assert_array_equal(c0, want_c[:, 0])
    np.testing.assert_array_equal(c1, want_c[:, 1])
    # spot-check the object view against map_boundary_gid
    objs = S.boundary_points(face[:50], c0[:50], c1[:50])
    for gid, o in enumerate(objs):
        assert o == S.map_boundary_gid(gid, ip, jp, kp)


@pytest.mark.gpu
@pytest.mark.parametrize("dom", DOMAINS)
@pytest.mark.parametrize("nt,nu", [(1, 1), (32, 3), (128, 4), (1024, 2)])
def test_device_audit(dom, nt, nu):
    ip, jp, kp = dom
    st = S.boundary_audit(ip, jp, kp, nt, nu)
    br = S.boundary_range(ip, jp, kp)
    assert st["boundary_range"] == br
    assert st["padded_range"] == S.padded_range(br, nt, nu)
    assert st["covered_once"] == br
    assert st["covered_more"] == st["not_covered"] == 0
    assert st["range_gids_in_padding"] == st["padding_escapes"] == 0
    assert st["first_violation"] == -1


@pytest.mark.gpu
def test_audit_runner_matches_reference_output(tmp_path, capsys):
    from paper_1504_02264_b200 import les

    cfg = types.SimpleNamespace(im=20, jm=12, km=9, nthreads=64, nunits=3)
    summary = les.run_boundary_audit(cfg, tmp_path)
    br = 12 * 9 + 9 * 20 + 12 * 20
    pr = S.padded_range(br, 64, 3)
    want = {"mode": "boundary-audit", "domain": [20, 12, 9], "boundary_range": br, "padded_range": pr,
            "padding_gids": pr - br}
    assert summary == want
    assert json.loads((tmp_path / "summary.json").read_text()) == want
    assert (tmp_path / "summary.json").read_text() == json.dumps(want, indent=2) + "\n"
    out = capsys.readouterr().out
    assert f"boundary audit ok: domain=(20,12,9) m=192 covered={br} padding={pr - br}" in out


@pytest.mark.gpu
@pytest.mark.parametrize("dom", [(6, 5, 4), (17, 9, 11), (150, 150, 90)])
def test_face_refresh_matches_pressure_halo(dom):
    import oracle.les_oracle as O
    from paper_1504_02264_b200 import les
    from paper_1504_02264_b200.reftypes import Grid

    im, jm, km = dom
    g = Grid.uniform(im, jm, km, 1.0)
    fs = les.FlowState.create(g, dt=0.5)
    rng = np.random.default_rng(7)
    p0 = rng.standard_normal((im + 2, jm + 2, km + 2)).astype(np.float32)
    fs.p[...] = p0
    les.refresh_pressure_faces(fs)
    got = np.array(fs.p)
    ref = p0.copy()
    O.press_halo(ref)
    face = np.zeros(p0.shape, bool)
    face[[0, -1], 1:-1, 1:-1] = True
    face[1:-1, [0, -1], 1:-1] = True
    face[1:-1, 1:-1, [0, -1]] = True
    np.testing.assert_array_equal(got[face].view(np.uint32), ref[face].view(np.uint32))
    interior = np.zeros(p0.shape, bool)
    interior[1:-1, 1:-1, 1:-1] = True
    rest = ~(face | interior)  # edges and corners: untouched
    np.testing.assert_array_equal(got[rest | interior].view(np.uint32), p0[rest | interior].view(np.uint32))
