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
