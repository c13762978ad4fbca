"""CPU checks of the drop-in boundary: liblesb200.so loads without a GPU and
exports every entry point include/les_b200.h declares, with the ABI version
and enum values the Python binding assumes.  No compute calls (no device)."""

import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "les_b200.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][\w\s\*]*?\b(lesb_\w+)\s*\(", src, flags=re.M)
    return sorted(set(names))


def header_enum(name):
    src = open(HEADER).read()
    m = re.search(rf"\b{name}\s*=\s*(-?\d+)", src) or re.search(rf"#define\s+{name}\s+(-?\d+)", src)
    assert m, name
    return int(m.group(1))


@pytest.fixture(scope="module")
def lib():
    from paper_1504_02264_b200 import build, _native

    build.build()
    return _native.load()


def test_header_declares_the_reference_surface():
    names = declared_functions()
    # one entry point per reference function on the hot path
    for n in ("lesb_step", "lesb_velnw", "lesb_bondv1", "lesb_velfg", "lesb_feedbf", "lesb_les_viscosity",
              "lesb_adam", "lesb_divergence", "lesb_strain_magnitude", "lesb_press", "lesb_solve_pressure",
              "lesb_redblack_iteration", "lesb_twinned_sweep", "lesb_create", "lesb_destroy"):
        assert n in names, n


def test_library_exports_every_declared_symbol(lib):
    raw = ctypes.CDLL(os.path.join(ROOT, "paper_1504_02264_b200", "liblesb200.so"))
    missing = [n for n in declared_functions() if not hasattr(raw, n)]
    assert not missing, missing


def test_binding_covers_every_declared_symbol(lib):
    from paper_1504_02264_b200 import _native

    missing = [n for n in declared_functions() if n not in _native._SIGS]
    assert not missing, missing


def test_abi_version_and_enums(lib):
    from paper_1504_02264_b200 import _native as N

    assert lib.lesb_abi_version() == header_enum("LESB_ABI_VERSION")
    for name in ("LESB_U", "LESB_V", "LESB_W", "LESB_P", "LESB_MASK", "LESB_FGH", "LESB_FGH_OLD", "LESB_RHS",
                 "LESB_REDBLACK", "LESB_TWINNED", "LESB_HALO_STORED", "LESB_HALO_PRESS", "LESB_OK",
                 "LESB_NONFINITE"):
        assert getattr(N, name) == header_enum(name), name
    for i, s in enumerate(N.STAGE_NAMES):
        assert header_enum(f"LESB_STAGE_{s.upper()}") == i


def test_argument_errors_without_a_device(lib):
    """Argument validation happens before any CUDA call, so it works here."""
    from paper_1504_02264_b200 import _native as N

    assert lib.lesb_create(None, None) == header_enum("LESB_E_ARG")
    assert b"null" in lib.lesb_last_error()
    assert lib.lesb_step(None, None, None, None, 1, 0, 1.0, None, None) == header_enum("LESB_E_ARG")
    assert lib.lesb_solve_pressure(4, 4, 4, None, None, None, 1.0, 0, 0, 0, None, None, 0) == \
        header_enum("LESB_E_ARG")
    with pytest.raises(N.NativeError):
        N.check(lib.lesb_destroy(None) - 1, "x")
