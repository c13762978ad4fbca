"""Drop-in for ``gmcf_mini.sor`` (reference: /root/reference/pkg/src/gmcf_mini/sor.py).

Same function names, signatures, argument validation, error types and
return values; the iterations run on the GPU through liblesb200.so.

``halo_fn`` support: ``None`` (the halo keeps p0's stored values) and the
press boundary policy (``les._pressure_halo(grid)`` of this package or of
the reference).  Any other callable raises ``NotImplementedError`` -- there
is no CPU path.
"""

from __future__ import annotations

import numpy as np

from . import _native as N
from .reftypes import PADDING, BoundaryPoint, Face, Grid, Scheme, SorCoeffs, is_redblack

__all__ = [
    "Grid", "Scheme", "SorCoeffs", "build_uniform_coeffs", "make_field", "make_twinned",
    "redblack_iteration", "twinned_sweep", "solve_pressure", "PressureHalo", "halo_policy",
    "Face", "BoundaryPoint", "PADDING", "boundary_range", "map_boundary_gid", "padded_range",
    "boundary_decode", "boundary_audit",
]


def build_uniform_coeffs(grid: Grid) -> SorCoeffs:
    """Coefficients for a uniformly spaced grid (sor.py:121-137): all
    neighbour weights 1/h^2, cn1 = h^2/6 over the interior."""
    spacings = np.concatenate([grid.dx1, grid.dy1, grid.dzn])
    h = float(spacings[0])
    if not np.all(spacings == np.float32(h)):
        raise ValueError("build_uniform_coeffs requires uniform spacing on all axes")
    w = np.float32(1.0 / (h * h))
    cn1 = np.full((grid.im, grid.jm, grid.km), np.float32(h * h / 6.0), dtype=np.float32)
    ax = np.full(grid.im, w, dtype=np.float32)
    ay = np.full(grid.jm, w, dtype=np.float32)
    az = np.full(grid.km, w, dtype=np.float32)
    return SorCoeffs(cn1, ax, ax.copy(), ay, ay.copy(), az, az.copy())


def make_field(im: int, jm: int, km: int) -> np.ndarray:
    """Zero field with a one-cell halo (sor.py:140-142)."""
    return np.zeros((im + 2, jm + 2, km + 2), dtype=np.float32)


def make_twinned(p: np.ndarray) -> np.ndarray:
    """Pair-interleaved copy, both components equal to p (sor.py:145-150)."""
    tp = np.empty(p.shape + (2,), dtype=np.float32)
    tp[..., 0] = p
    tp[..., 1] = p
    return tp


class PressureHalo:
    """The press boundary policy (les.py:341-355) as a recognisable callable.

    Passed as ``halo_fn`` it selects the device's PRESS halo policy.  Called
    directly on a host array it applies the same boundary values to that
    array (a host utility, as in the reference; not used by the device path).
    """

    def __init__(self, grid: Grid):
        self.jm = grid.jm

    def __call__(self, p: np.ndarray) -> None:
        jm = self.jm
        p[0, :, :] = p[1, :, :]
        p[-1, :, :] = 0.0
        p[:, 0, :] = p[:, jm, :]
        p[:, -1, :] = p[:, 1, :]
        p[:, :, 0] = p[:, :, 1]
        p[:, :, -1] = 0.0


def halo_policy(halo_fn, p_shape) -> int:
    """Map a halo_fn onto a device policy (STORED / PRESS)."""
    if halo_fn is None:
        return N.LESB_HALO_STORED
    jm = p_shape[1] - 2
    if isinstance(halo_fn, PressureHalo):
        if halo_fn.jm != jm:
            raise ValueError(f"halo_fn was built for jm={halo_fn.jm}, field has jm={jm}")
        return N.LESB_HALO_PRESS
    # the reference's own closure: les._pressure_halo(grid).<locals>.refresh
    if (getattr(halo_fn, "__qualname__", "") == "_pressure_halo.<locals>.refresh"
            and getattr(halo_fn, "__module__", "").endswith("les")):
        names = halo_fn.__code__.co_freevars
        cells = halo_fn.__closure__ or ()
        env = {n: c.cell_contents for n, c in zip(names, cells)}
        if env.get("jm") == jm:
            return N.LESB_HALO_PRESS
    raise NotImplementedError(
        "only halo_fn=None and les._pressure_halo(grid) run on the device; "
        f"got {halo_fn!r}")


def _check_shapes(p: np.ndarray, rhs: np.ndarray, c: SorCoeffs) -> tuple[int, int, int]:
    """sor.py:153-159"""
    if p.shape != rhs.shape:
        raise ValueError(f"p shape {p.shape} != rhs shape {rhs.shape}")
    im, jm, km = (n - 2 for n in p.shape[:3])
    if c.cn1.shape != (im, jm, km):
        raise ValueError(f"cn1 shape {c.cn1.shape} does not match interior ({im},{jm},{km})")
    return im, jm, km


def _device() -> int:
    from . import runtime

    return runtime.current_device()


def solve_pressure(p0, rhs, c, omega, n_iter, scheme: Scheme, workers: int = 1, halo_fn=None):
    """``n_iter`` iterations of RED-BLACK SOR or TWINNED sweeps on the GPU
    (sor.py:255-309).  Returns ``(p, residuals)``; p0 and rhs are not
    modified.  ``workers`` is validated as in the reference and otherwise
    ignored: the device result is identical for every worker count."""
    if n_iter < 1:
        raise ValueError("n_iter must be >= 1")
    if workers < 1:
        raise ValueError("workers must be >= 1")
    if is_redblack(scheme) and workers > 1:
        raise ValueError("REDBLACK supports workers=1 only; use TWINNED for parallel runs")
    im, jm, km = _check_shapes(p0, rhs, c)
    policy = halo_policy(halo_fn, p0.shape)
    keep: list = []
    cf = N.make_coeffs(c, keep)
    p0c = N.f32c(p0)
    rhsc = N.f32c(rhs)
    p = np.empty_like(p0c)
    res = np.zeros(n_iter, dtype=np.float64)
    sch = N.LESB_REDBLACK if is_redblack(scheme) else N.LESB_TWINNED
    N.check(N.load().lesb_solve_pressure(im, jm, km, N.fptr(p0c), N.fptr(rhsc), cf, float(omega), int(n_iter),
                                         sch, policy, N.fptr(p), N.dptr(res), _device()),
            "solve_pressure")
    return p, res


def redblack_iteration(p, rhs, c, omega, halo_fn=None) -> float:
    """One red-black iteration in place (sor.py:181-203); returns the
    squared-correction sum of both colour passes."""
    im, jm, km = _check_shapes(p, rhs, c)
    policy = halo_policy(halo_fn, p.shape)
    keep: list = []
    cf = N.make_coeffs(c, keep)
    work = p if (p.dtype == np.float32 and p.flags.c_contiguous) else N.f32c(p)
    res = np.zeros(1, dtype=np.float64)
    N.check(N.load().lesb_redblack_iteration(im, jm, km, N.fptr(work), N.fptr(N.f32c(rhs)), cf, float(omega),
                                             policy, N.dptr(res), _device()),
            "redblack_iteration")
    if work is not p:
        p[...] = work
    return float(res[0])


def twinned_sweep(tp, rhs, c, omega, nrd: int) -> float:
    """One sweep reading component ``nrd`` and writing component 1-nrd
    (sor.py:232-246)."""
    if tp.ndim != 4 or tp.shape[3] != 2:
        raise ValueError(f"twinned array must have a trailing pair axis, got {tp.shape}")
    if nrd not in (0, 1):
        raise ValueError("nrd must be 0 or 1")
    im, jm, km = _check_shapes(tp[..., 0], rhs, c)
    keep: list = []
    cf = N.make_coeffs(c, keep)
    src = np.ascontiguousarray(tp[..., nrd])
    dst = np.ascontiguousarray(tp[..., 1 - nrd])
    res = np.zeros(1, dtype=np.float64)
    N.check(N.load().lesb_twinned_sweep(im, jm, km, N.fptr(src), N.fptr(dst), N.fptr(N.f32c(rhs)), cf,
                                        float(omega), N.dptr(res), _device()),
            "twinned_sweep")
    tp[..., 1 - nrd] = dst
    return float(res[0])


# ---------------------------------------------------------------------------
# Boundary-range launch geometry (sor.py:312-349; the paper's gid -> face map)
# ---------------------------------------------------------------------------
def boundary_range(ip: int, jp: int, kp: int) -> int:
    """Size of the 1-D index space enumerating the three boundary families
    (sor.py:312-316)."""
    if min(ip, jp, kp) < 1:
        raise ValueError("ip, jp, kp must be >= 1")
    return jp * kp + kp * ip + jp * ip


def map_boundary_gid(gid: int, ip: int, jp: int, kp: int):
    """Decode one global id into a boundary point, or PADDING past the range
    (sor.py:319-338; host index math, as in the reference).  The device does
    the same decode for whole launches: boundary_decode / boundary_audit."""
    if gid < 0:
        raise ValueError("gid must be >= 0")
    n_yz = jp * kp
    n_zx = kp * ip
    if gid < n_yz:
        return BoundaryPoint(Face.YZ, (gid % jp, gid // jp))
    if gid < n_yz + n_zx:
        r = gid - n_yz
        return BoundaryPoint(Face.ZX, (r // ip, r % ip))
    if gid < n_yz + n_zx + jp * ip:
        r = gid - n_yz - n_zx
        return BoundaryPoint(Face.XY, (r // ip, r % ip))
    return PADDING


def padded_range(range_: int, nthreads: int, nunits: int) -> int:
    """Pad a work range up to a multiple of nthreads * nunits (sor.py:341-349)."""
    if range_ < 0:
        raise ValueError("range must be >= 0")
    if nthreads < 1 or nunits < 1:
        raise ValueError("nthreads and nunits must be >= 1")
    m = nthreads * nunits
    rem = range_ % m
    return range_ if rem == 0 else range_ + (m - rem)


_FACES = (Face.YZ, Face.ZX, Face.XY)


def boundary_decode(ip: int, jp: int, kp: int, gid0: int = 0, n: int | None = None):
    """Decode gids [gid0, gid0 + n) on the GPU (default: the whole boundary
    range).  Returns (face, c0, c1) int32 arrays: face 0 YZ, 1 ZX, 2 XY, -1
    PADDING, (c0, c1) the BoundaryPoint coords (-1 for padding)."""
    boundary_range(ip, jp, kp)
    if gid0 < 0:
        raise ValueError("gid must be >= 0")
    if n is None:
        n = boundary_range(ip, jp, kp) - gid0
    n = max(int(n), 0)
    face = np.empty(n, np.int32)
    c0 = np.empty(n, np.int32)
    c1 = np.empty(n, np.int32)
    ip_ = lambda a: a.ctypes.data_as(N.IP)  # noqa: E731
    N.check(N.load().lesb_boundary_decode(ip, jp, kp, int(gid0), n, ip_(face), ip_(c0), ip_(c1)),
            "boundary_decode")
    return face, c0, c1


def boundary_points(face, c0, c1) -> list:
    """BoundaryPoint / PADDING objects of decoded arrays (for comparison with
    map_boundary_gid)."""
    return [PADDING if f < 0 else BoundaryPoint(_FACES[f], (int(a), int(b))) for f, a, b in zip(face, c0, c1)]


def boundary_audit(ip: int, jp: int, kp: int, nthreads: int, nunits: int) -> dict:
    """The boundary audit (cli.py:286-320) as one GPU launch: every gid of
    the padded range decoded by the thread that would own it (blocks of
    nthreads threads x nunits gids), per-point hit counts, padding guard."""
    boundary_range(ip, jp, kp)
    padded_range(0, nthreads, nunits)
    st = (N.C.c_longlong * 8)()
    N.check(N.load().lesb_boundary_audit(ip, jp, kp, nthreads, nunits, st), "boundary_audit")
    keys = ("boundary_range", "padded_range", "range_gids_in_padding", "padding_escapes", "covered_once",
            "covered_more", "not_covered", "first_violation")
    return dict(zip(keys, (int(x) for x in st)))

