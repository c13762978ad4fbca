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
