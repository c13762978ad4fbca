"""Device selection for the LES library (one process per GPU)."""

from __future__ import annotations

import os

_device: int | None = None


def set_device(ordinal: int) -> None:
    global _device
    _device = int(ordinal)


def current_device() -> int:
    if _device is not None:
        return _device
    if "LESB_DEVICE" in os.environ:
        return int(os.environ["LESB_DEVICE"])
    return int(os.environ.get("LOCAL_RANK", "0")) if os.environ.get("LESB_USE_LOCAL_RANK") else 0


SOR_AUTO, SOR_PASSES, SOR_RESIDENT, SOR_FUSED = 0, 1, 2, 3


def set_sor_path(path: int) -> None:
    """Red-black solver implementation for new domains and the host-buffer
    solver: 0 auto, 1 streaming colour passes (colour-split layout), 2
    shared-memory resident, 3 streaming colour passes on the natural layout.  Results are bitwise identical; this only
    selects the kernels."""
    from . import _native as N

    N.check(N.load().lesb_set_default_sor_path(int(path)), "lesb_set_default_sor_path")
