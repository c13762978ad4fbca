"""GMCF dump format (CPU): round trip, header bytes, atomic write, and byte
identity with the reference writer where the reference is importable."""

import os
import sys

import numpy as np
import pytest

from paper_1504_02264_b200 import dump


def test_roundtrip_and_header(tmp_path):
    a = np.random.default_rng(1).standard_normal((4, 5, 6)).astype(np.float32)
    p = tmp_path / "u.gmcf"
    dump.write_field(p, a)
    raw = p.read_bytes()
    assert raw[:4] == b"GMCF"
    assert list(np.frombuffer(raw[4:16], "<u4")) == [4, 5, 6]
    assert len(raw) == 16 + a.size * 4
    assert np.array_equal(dump.read_field(p), a)
    assert not (tmp_path / "u.gmcf.tmp").exists()


def test_rejects_bad_input(tmp_path):
    with pytest.raises(ValueError):
        dump.write_field(tmp_path / "x.gmcf", np.zeros((2, 2), np.float32))
    (tmp_path / "bad.gmcf").write_bytes(b"NOPE" + bytes(12))
    with pytest.raises(ValueError):
        dump.read_field(tmp_path / "bad.gmcf")


def test_byte_identical_to_reference(tmp_path):
    ref = "/root/reference/pkg/src"
    if os.path.isdir(ref) and ref not in sys.path:
        sys.path.append(ref)
    rdump = pytest.importorskip("gmcf_mini.dump")
    a = np.random.default_rng(2).standard_normal((3, 7, 5)).astype(np.float32)
    dump.write_field(tmp_path / "ours.gmcf", a)
    rdump.write_field(tmp_path / "ref.gmcf", a)
    assert (tmp_path / "ours.gmcf").read_bytes() == (tmp_path / "ref.gmcf").read_bytes()
    assert np.array_equal(rdump.read_field(tmp_path / "ours.gmcf"), a)


def test_checkpoint_roundtrip_host(tmp_path):
    """write_checkpoint / read_checkpoint on a host state object: every field a
    step reads comes back bit for bit (fgh / fgh_old per component), with a
    sidecar; a checkpoint of another grid is refused."""
    from types import SimpleNamespace

    rng = np.random.default_rng(5)
    im, jm, km = 5, 4, 3
    sh = (im + 2, jm + 2, km + 2)
    grid = SimpleNamespace(im=im, jm=jm, km=km)
    src = SimpleNamespace(grid=grid)
    for n in ("u", "v", "w", "p", "mask"):
        setattr(src, n, rng.standard_normal(sh).astype(np.float32))
    for n in ("fgh", "fgh_old"):
        setattr(src, n, rng.standard_normal(sh + (3,)).astype(np.float32))
    paths = dump.write_checkpoint(src, tmp_path / "ck")
    assert len(paths) == 11 and (tmp_path / "ck" / "checkpoint.txt").exists()
    dst = SimpleNamespace(grid=grid)
    dump.read_checkpoint(dst, tmp_path / "ck")
    for n in dump.CHECKPOINT_FIELDS:
        a, b = getattr(src, n), getattr(dst, n)
        assert a.shape == b.shape and np.array_equal(a.view(np.uint32), b.view(np.uint32)), n
    other = SimpleNamespace(grid=SimpleNamespace(im=4, jm=4, km=3))
    with pytest.raises(ValueError):
        dump.read_checkpoint(other, tmp_path / "ck")
