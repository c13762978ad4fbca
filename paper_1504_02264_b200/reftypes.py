"""Host-side types of the reference interface.

The drop-in must share the reference's own classes where they exist --
``Scheme`` is compared by identity (les.py:373, sor.py:268, 273) -- so when
``gmcf_mini`` is importable its ``Scheme``, ``Grid``, ``SorCoeffs``,
``WindProfile`` and ``NumericsError`` are re-exported.  Otherwise (e.g. on
the GPU box, where the reference is not installed) equivalent definitions
with the same fields, validation and messages are used.
"""

from __future__ import annotations

try:  # pragma: no cover - depends on the environment
    from gmcf_mini.coupling import WindProfile  # type: ignore
    from gmcf_mini.errors import GmcfError, NumericsError  # type: ignore
    from gmcf_mini.sor import PADDING, BoundaryPoint, Face, Grid, Scheme, SorCoeffs  # type: ignore

    HAVE_REFERENCE = True
except Exception:  # noqa: BLE001
    HAVE_REFERENCE = False

    import enum
    from dataclasses import dataclass

    import numpy as np

    class Scheme(enum.Enum):  # sor.py:29-31
        REDBLACK = "redblack"
        TWINNED = "twinned"

    class Face(enum.Enum):  # sor.py:34-37
        YZ = "yz"
        ZX = "zx"
        XY = "xy"

    class _Padding:  # sor.py:40-49
        """Sentinel for gids that fall in the padded tail of the boundary range."""

        __slots__ = ()

        def __repr__(self) -> str:
            return "PADDING"

    PADDING = _Padding()

    @dataclass(frozen=True)
    class BoundaryPoint:  # sor.py:52-61
        """One boundary-face point: (j, k) on YZ, (k, i) on ZX, (j, i) on XY."""

        face: Face
        coords: tuple

    class GmcfError(Exception):  # errors.py:8-9
        pass

    class NumericsError(GmcfError):  # errors.py:20-28
        """A numerical stage produced non-finite values."""

        def __init__(self, stage: str, detail: str = ""):
            self.stage = stage
            msg = f"non-finite values after stage '{stage}'"
            if detail:
                msg += f": {detail}"
            super().__init__(msg)

    @dataclass
    class Grid:  # sor.py:64-105
        im: int
        jm: int
        km: int
        dx1: np.ndarray
        dy1: np.ndarray
        dzn: np.ndarray

        def __post_init__(self):
            if min(self.im, self.jm, self.km) < 1:
                raise ValueError("grid dimensions must be >= 1")
            self.dx1 = np.asarray(self.dx1, dtype=np.float32)
            self.dy1 = np.asarray(self.dy1, dtype=np.float32)
            self.dzn = np.asarray(self.dzn, dtype=np.float32)
            for name, arr, n in (("dx1", self.dx1, self.im + 3), ("dy1", self.dy1, self.jm + 2),
                                 ("dzn", self.dzn, self.km + 2)):
                if arr.shape != (n,):
                    raise ValueError(f"{name} must have length {n}, got {arr.shape}")
                if not (arr > 0).all():
                    raise ValueError(f"{name} must be positive everywhere")

        @classmethod
        def uniform(cls, im: int, jm: int, km: int, h: float) -> "Grid":
            return cls(im, jm, km, np.full(im + 3, h, np.float32), np.full(jm + 2, h, np.float32),
                       np.full(km + 2, h, np.float32))

    @dataclass
    class SorCoeffs:  # sor.py:108-118
        cn1: np.ndarray
        cn2l: np.ndarray
        cn2s: np.ndarray
        cn3l: np.ndarray
        cn3s: np.ndarray
        cn4l: np.ndarray
        cn4s: np.ndarray

    class ConfigError(GmcfError):
        pass

    @dataclass
    class WindProfile:  # coupling.py:40-67
        u: np.ndarray
        v: np.ndarray
        w: np.ndarray
        t: int = 0

        def __post_init__(self):
            self.u = np.asarray(self.u, dtype=np.float32)
            self.v = np.asarray(self.v, dtype=np.float32)
            self.w = np.asarray(self.w, dtype=np.float32)
            if not (self.u.shape == self.v.shape == self.w.shape) or self.u.ndim != 1:
                raise ConfigError("wind profile components must be 1-D arrays of equal length")
            if self.u.shape[0] < 1:
                raise ConfigError("wind profile needs at least one level")

        @property
        def kp(self) -> int:
            return self.u.shape[0]

def _scheme_member(scheme, name: str) -> bool:
    """``scheme is Scheme.<name>`` for this module's Scheme and for the
    reference's own (gmcf_mini.sor.Scheme), whichever the caller holds: the
    reference compares by identity (sor.py:268, 273), and the drop-in must
    accept the reference's members even when this package was imported before
    gmcf_mini was importable."""
    if scheme is getattr(Scheme, name):
        return True
    return type(scheme).__name__ == "Scheme" and getattr(scheme, "name", None) == name


def is_redblack(scheme) -> bool:
    return _scheme_member(scheme, "REDBLACK")


def is_twinned(scheme) -> bool:
    return _scheme_member(scheme, "TWINNED")


__all__ = ["Scheme", "Grid", "SorCoeffs", "WindProfile", "NumericsError", "HAVE_REFERENCE", "is_redblack",
           "is_twinned"]
