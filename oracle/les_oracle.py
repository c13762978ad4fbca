"""CPU ORACLE for the DPRI-LES time step -- TEST INFRASTRUCTURE ONLY.

This module is the parity checker for the CUDA path in
``paper_1504_02264_b200``.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it;
the product package never does (it fails loudly without its CUDA library).

It is a point-wise restatement of the reference hot path
(``/root/reference/pkg/src/gmcf_mini/les.py`` and ``sor.py``), written as
whole-array float32 numpy expressions so that every operation rounds once,
in the reference's evaluation order.  Boundary handling is restated in the
closed forms of SURVEY.md Appendix B (halo cell -> interior source cell)
instead of the reference's sequential slice writes; the two are equal
value-for-value, which ``tests/test_oracle_golden.py`` pins against golden
vectors produced by the unmodified reference (``tests/golden/make_golden.py``).

Parity status: PINNED (bitwise for all fields, rtol 1e-12 for the float64
residual sums) against tests/golden/*.npz.

Array conventions (as the reference, les.py:56-63): C-order float32
``(im+2, jm+2, km+2)`` with a one-cell halo, k contiguous; ``fgh``/``fgh_old``
carry a trailing component axis of 3.  Spacings: ``dx1`` has im+3 entries,
``dy1`` jm+2, ``dzn`` km+2 (sor.py:64-94).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

F32 = np.float32
STAGES = ("velnw", "bondv1", "velfg", "feedbf", "les", "adam", "press")
FIELDS = ("u", "v", "w", "fgh", "fgh_old", "p")


class OracleNumericsError(Exception):
    """Raised when a stage leaves a non-finite value (les.py:384-390)."""

    def __init__(self, stage: str, name: str):
        super().__init__(f"non-finite values after stage '{stage}': field {name}")
        self.stage = stage
        self.field = name


@dataclass
class OState:
    """Plain container mirroring the reference FlowState fields (les.py:37-52)."""

    u: np.ndarray
    v: np.ndarray
    w: np.ndarray
    fgh: np.ndarray
    fgh_old: np.ndarray
    p: np.ndarray
    mask: np.ndarray
    dx1: np.ndarray
    dy1: np.ndarray
    dzn: np.ndarray
    dt: float
    vn: float = 1e-5
    cs: float = 0.14
    extra: dict = field(default_factory=dict)

    @property
    def dims(self):
        return tuple(n - 2 for n in self.u.shape)

    @classmethod
    def zeros(cls, im, jm, km, h=2.0, dt=0.5, vn=0.8, cs=0.14):
        sh = (im + 2, jm + 2, km + 2)
        z = lambda: np.zeros(sh, F32)  # noqa: E731
        return cls(z(), z(), z(), np.zeros(sh + (3,), F32), np.zeros(sh + (3,), F32), z(), z(),
                   np.full(im + 3, h, F32), np.full(jm + 2, h, F32), np.full(km + 2, h, F32),
                   dt, vn, cs)

    @classmethod
    def from_flowstate(cls, fs):
        """Copy a reference-shaped FlowState (any object with the same attributes)."""
        g = fs.grid
        return cls(fs.u.copy(), fs.v.copy(), fs.w.copy(), fs.fgh.copy(), fs.fgh_old.copy(),
                   fs.p.copy(), fs.mask.copy(), np.asarray(g.dx1, F32).copy(),
                   np.asarray(g.dy1, F32).copy(), np.asarray(g.dzn, F32).copy(),
                   fs.dt, fs.vn, fs.cs)

    def copy(self):
        return OState(*(getattr(self, n).copy() for n in
                        ("u", "v", "w", "fgh", "fgh_old", "p", "mask", "dx1", "dy1", "dzn")),
                      self.dt, self.vn, self.cs)


# ---------------------------------------------------------------------------
# index helpers
# ---------------------------------------------------------------------------

def _box(dims, axis=None, lo=None, hi=None):
    """Slices selecting the interior 1..N on every axis, except ``axis`` which
    runs over [lo, hi)."""
    out = [slice(1, n + 1) for n in dims]
    if axis is not None:
        out[axis] = slice(lo, hi)
    return tuple(out)


def _bcast(vec, axis):
    shape = [1, 1, 1]
    shape[axis] = -1
    return np.asarray(vec, F32).reshape(shape)


def _spac(st: OState, axis):
    return (st.dx1, st.dy1, st.dzn)[axis]


def _d_central(f, axis, lo, hi, dims, s):
    """(f[P+e] - f[P-e]) / (s[P] + s[P+1]) for axis coordinate P in [lo, hi)
    (les.py:100-110)."""
    up = _box(dims, axis, lo + 1, hi + 1)
    dn = _box(dims, axis, lo - 1, hi - 1)
    den = s[lo:hi] + s[lo + 1:hi + 1]
    return (f[up] - f[dn]) / _bcast(den, axis)


def _d_onesided_top(f, axis, dims, s):
    """(f[N+1] - f[N]) / s[N+1] on the single plane N+1 (les.py:111-117)."""
    n = dims[axis]
    return (f[_box(dims, axis, n + 1, n + 2)] - f[_box(dims, axis, n, n + 1)]) / F32(s[n + 1])


def _d_at_base(f, axis, dims, s):
    return _d_central(f, axis, 1, dims[axis] + 1, dims, s)


def _d_at_shift(f, axis, dims, s):
    """Derivative at P + e_axis for P interior: central for 2..N, one-sided at N+1."""
    n = dims[axis]
    parts = []
    if n >= 2:
        parts.append(_d_central(f, axis, 2, n + 1, dims, s))
    parts.append(_d_onesided_top(f, axis, dims, s))
    return np.concatenate(parts, axis=axis)


# ---------------------------------------------------------------------------
# stages
# ---------------------------------------------------------------------------

def velnw(st: OState) -> None:
    """u += dt*(fgh_0 - 2(p[i+1]-p[i])/(dx1[i]+dx1[i+1])) on faces 0..N per axis
    (les.py:218-241)."""
    im, jm, km = st.dims
    dt = F32(st.dt)
    two = F32(2.0)
    vel = (st.u, st.v, st.w)
    for a in range(3):
        n = st.dims[a]
        s = _spac(st, a)
        faces = _box(st.dims, a, 0, n + 1)
        nxt = _box(st.dims, a, 1, n + 2)
        grad = ((st.p[nxt] - st.p[faces]) * two) / _bcast(s[0:n + 1] + s[1:n + 2], a)
        comp = st.fgh[..., a][faces]
        vel[a][faces] = vel[a][faces] + dt * (comp - grad)


def _halo_source(n, idx):
    """Vector of source indices for a periodic axis: 0 -> n, n+1 -> 1."""
    src = idx.copy()
    src[idx == 0] = n
    src[idx == n + 1] = 1
    return src


def bondv1(st: OState, inflow_u, inflow_v, inflow_w) -> None:
    """Velocity halos in closed form (les.py:244-266):
    resolve k (w -> 0 at k in {0, km+1}; u,v clamp to 1..km), then j
    (periodic), then i (0 -> inflow at the resolved k, im+1 -> im)."""
    im, jm, km = st.dims
    if len(inflow_u) != km:
        raise ValueError(f"inflow has {len(inflow_u)} levels, grid has km={km}")
    I = np.arange(im + 2)[:, None, None]
    J = np.arange(jm + 2)[None, :, None]
    K = np.arange(km + 2)[None, None, :]
    kr = np.clip(K, 1, km)
    jr = _halo_source(jm, np.arange(jm + 2))[None, :, None]
    ir = np.where(I == im + 1, im, I)
    halo = (I == 0) | (I == im + 1) | (J == 0) | (J == jm + 1) | (K == 0) | (K == km + 1)
    halo = np.broadcast_to(halo, st.u.shape)
    for f, inflow, is_w in ((st.u, inflow_u, False), (st.v, inflow_v, False), (st.w, inflow_w, True)):
        inflow = np.asarray(inflow, F32)
        src = f[np.broadcast_to(np.where(I == 0, 1, ir), f.shape),
                np.broadcast_to(jr, f.shape), np.broadcast_to(kr, f.shape)]
        west = np.broadcast_to(inflow[kr - 1], f.shape)
        val = np.where(np.broadcast_to(I == 0, f.shape), west, src)
        if is_w:
            val = np.where(np.broadcast_to((K == 0) | (K == km + 1), f.shape), F32(0.0), val)
        f[halo] = val[halo]


def _velfg_component(st: OState, m: int) -> np.ndarray:
    """Force component m over the interior (les.py:121-192, combine at 128-175)."""
    dims = st.dims
    vel = (st.u, st.v, st.w)
    vm = vel[m]
    cov, cp, diu, dp = [], [], [], []
    for d in range(3):
        s = _spac(st, d)
        n = dims[d]
        d0 = _d_at_base(vm, d, dims, s)
        d1 = _d_at_shift(vm, d, dims, s)
        carrier0 = vel[d][_box(dims)]
        carrier1 = vel[d][_box(dims, d, 2, n + 2)]
        cov.append(carrier0 * d0)
        cp.append(carrier1 * d1)
        diu.append(d0)
        dp.append(d1)
    two = F32(2.0)
    lo = [_bcast(_spac(st, a)[1:dims[a] + 1], a) for a in range(3)]
    hi = [_bcast(_spac(st, a)[2:dims[a] + 2], a) for a in range(3)]
    avg = []
    for d in range(3):
        if d == m:  # staggered direction: spacing-weighted average
            avg.append((hi[d] * cov[d] + lo[d] * cp[d]) / (lo[d] + hi[d]))
        else:
            avg.append((cov[d] + cp[d]) / two)
    terms = []
    for d in range(3):
        diff = -diu[d] + dp[d]
        if d == m:
            terms.append(two * diff / (lo[d] + hi[d]))
        else:
            terms.append(diff / lo[d])
    df = terms[0] + terms[1] + terms[2]
    covc = avg[0] + avg[1] + avg[2]
    return -covc + F32(st.vn) * df


def velfg(st: OState) -> None:
    for m in range(3):
        st.fgh[_box(st.dims) + (m,)] = _velfg_component(st, m)


def feedbf(st: OState) -> None:
    """fgh_m -= (mask/dt) v_m; v_m *= 1 - mask on the interior (les.py:269-282)."""
    b = _box(st.dims)
    msk = st.mask[b]
    coef = msk / F32(st.dt)
    keep = F32(1.0) - msk
    for m, vel in enumerate((st.u, st.v, st.w)):
        st.fgh[b + (m,)] = st.fgh[b + (m,)] - coef * vel[b]
        vel[b] = vel[b] * keep


def csd2_field(st: OState) -> np.ndarray:
    """(cs * cbrt(dx*dy*dz))^2 over the interior (les.py:305-310)."""
    im, jm, km = st.dims
    prod = (_bcast(st.dx1[1:im + 1], 0) * _bcast(st.dy1[1:jm + 1], 1)) * _bcast(st.dzn[1:km + 1], 2)
    delta = np.cbrt(prod).astype(F32)
    cd = F32(st.cs) * delta
    return cd * cd


def strain_magnitude(st: OState) -> np.ndarray:
    """|S| = sqrt(sum_ij S_ij S_ij), central differences (les.py:285-296)."""
    dims = st.dims
    vel = (st.u, st.v, st.w)
    d = [[_d_at_base(vel[m], a, dims, _spac(st, a)) for a in range(3)] for m in range(3)]
    h = F32(0.5)
    s12 = h * (d[0][1] + d[1][0])
    s13 = h * (d[0][2] + d[2][0])
    s23 = h * (d[1][2] + d[2][1])
    diag = d[0][0] * d[0][0] + d[1][1] * d[1][1] + d[2][2] * d[2][2]
    off = s12 * s12 + s13 * s13 + s23 * s23
    return np.sqrt(diag + F32(2.0) * off)


def les_viscosity(st: OState) -> None:
    """fgh_m += nu_t * lap(v_m), nu_t = csd2 * |S| (les.py:299-320); no-op at cs == 0."""
    if st.cs == 0.0:
        return
    dims = st.dims
    nu = csd2_field(st) * strain_magnitude(st)
    b = _box(dims)
    for m, vel in enumerate((st.u, st.v, st.w)):
        lap = np.zeros(dims, F32)
        for a in range(3):
            h = _bcast(_spac(st, a)[1:dims[a] + 1], a)
            up = _box(dims, a, 2, dims[a] + 2)
            dn = _box(dims, a, 0, dims[a])
            lap = lap + ((vel[up] - F32(2.0) * vel[b]) + vel[dn]) / (h * h)
        st.fgh[b + (m,)] = st.fgh[b + (m,)] + nu * lap


def adam(st: OState) -> None:
    """fgh <- 1.5 fgh - 0.5 fgh_old; fgh_old <- previous fgh, whole arrays (les.py:323-327)."""
    prev = st.fgh.copy()
    st.fgh[...] = F32(1.5) * prev - F32(0.5) * st.fgh_old
    st.fgh_old[...] = prev


def divergence(st: OState) -> np.ndarray:
    """Staggered divergence over the interior (les.py:330-338)."""
    dims = st.dims
    b = _box(dims)
    vel = (st.u, st.v, st.w)
    out = None
    for a in range(3):
        lo = _box(dims, a, 0, dims[a])
        t = (vel[a][b] - vel[a][lo]) / _bcast(_spac(st, a)[1:dims[a] + 1], a)
        out = t if out is None else out + t
    return out


# ---------------------------------------------------------------------------
# pressure halo and SOR (sor.py:121-309, les.py:341-381)
# ---------------------------------------------------------------------------

def press_halo(p: np.ndarray) -> None:
    """Closed form of the press halo (les.py:341-355): resolve k
    (0 -> 1, km+1 -> 0), then j (periodic), then i (0 -> 1, im+1 -> 0)."""
    im, jm, km = (n - 2 for n in p.shape)
    I = np.arange(im + 2)[:, None, None]
    J = np.arange(jm + 2)[None, :, None]
    K = np.arange(km + 2)[None, None, :]
    ks = np.where(K == 0, 1, np.minimum(K, km))
    js = _halo_source(jm, np.arange(jm + 2))[None, :, None]
    is_ = np.where(I == 0, 1, np.minimum(I, im))
    shp = p.shape
    val = p[np.broadcast_to(is_, shp), np.broadcast_to(js, shp), np.broadcast_to(ks, shp)]
    zero = np.broadcast_to((K == km + 1) | (I == im + 1), shp)
    val = np.where(zero, F32(0.0), val)
    halo = np.broadcast_to((I == 0) | (I == im + 1) | (J == 0) | (J == jm + 1) | (K == 0) | (K == km + 1), shp)
    p[halo] = val[halo]


@dataclass
class Coeffs:
    cn1: np.ndarray
    cn2l: np.ndarray
    cn2s: np.ndarray
    cn3l: np.ndarray
    cn3s: np.ndarray
    cn4l: np.ndarray
    cn4s: np.ndarray


def uniform_coeffs(im, jm, km, h) -> Coeffs:
    """Uniform-spacing stencil weights (sor.py:121-137): 1/h^2 and cn1 = h^2/6."""
    h = float(F32(h))
    w = F32(1.0 / (h * h))
    return Coeffs(np.full((im, jm, km), F32(h * h / 6.0), F32),
                  np.full(im, w, F32), np.full(im, w, F32), np.full(jm, w, F32),
                  np.full(jm, w, F32), np.full(km, w, F32), np.full(km, w, F32))


def _nbsum(p, c: Coeffs):
    """Weighted six-neighbour sum in the reference order E, W, N, S, T, B (sor.py:162-171)."""
    e = p[2:, 1:-1, 1:-1]
    w_ = p[:-2, 1:-1, 1:-1]
    n = p[1:-1, 2:, 1:-1]
    s = p[1:-1, :-2, 1:-1]
    t = p[1:-1, 1:-1, 2:]
    b = p[1:-1, 1:-1, :-2]
    acc = _bcast(c.cn2l, 0) * e
    acc = acc + _bcast(c.cn2s, 0) * w_
    acc = acc + _bcast(c.cn3l, 1) * n
    acc = acc + _bcast(c.cn3s, 1) * s
    acc = acc + _bcast(c.cn4l, 2) * t
    acc = acc + _bcast(c.cn4s, 2) * b
    return acc


def colour(im, jm, km, nrd):
    """True where (i0 + j0 + k0 + nrd) is even, 0-based interior (sor.py:174-178)."""
    i, j, k = np.ogrid[0:im, 0:jm, 0:km]
    return ((i + j + k + nrd) & 1) == 0


def rb_iteration(p, rhs, c: Coeffs, omega, policy: str | None) -> float:
    """One red-black iteration in place (sor.py:181-203).  ``policy`` is None
    (stored halo) or "press" (les._pressure_halo)."""
    im, jm, km = (n - 2 for n in p.shape)
    om = F32(omega)
    total = 0.0
    interior = p[1:-1, 1:-1, 1:-1]
    for nrd in (0, 1):
        if policy == "press":
            press_halo(p)
        rel = om * (c.cn1 * (_nbsum(p, c) - rhs[1:-1, 1:-1, 1:-1]) - interior)
        sel = colour(im, jm, km, nrd)
        interior[sel] = interior[sel] + rel[sel]
        r = rel[sel].astype(np.float64)
        total += float(np.sum(r * r))
    if policy == "press":
        press_halo(p)
    return total


def tw_sweep(src, dst, rhs, c: Coeffs, omega) -> float:
    """Jacobi sweep reading ``src`` and writing ``dst`` interior (sor.py:206-246)."""
    om = F32(omega)
    centre = src[1:-1, 1:-1, 1:-1]
    rel = om * (c.cn1 * (_nbsum(src, c) - rhs[1:-1, 1:-1, 1:-1]) - centre)
    dst[1:-1, 1:-1, 1:-1] = centre + rel
    r = rel.astype(np.float64)
    return float(np.sum(r * r))


def solve_pressure(p0, rhs, c: Coeffs, omega, n_iter, scheme: str, policy: str | None):
    """Returns (p, residuals[n_iter]) (sor.py:255-309).  scheme is "redblack" or "twinned"."""
    res = np.zeros(n_iter, np.float64)
    if scheme == "redblack":
        p = p0.copy()
        for it in range(n_iter):
            res[it] = rb_iteration(p, rhs, c, omega, policy)
        return p, res
    a = p0.copy()
    b = p0.copy()
    if policy == "press":
        press_halo(a)
        press_halo(b)
    for it in range(n_iter):
        s = tw_sweep(a, b, rhs, c, omega)
        if policy == "press":
            press_halo(b)
        s += tw_sweep(b, a, rhs, c, omega)
        if policy == "press":
            press_halo(a)
        res[it] = s
    return a, res


def press(st: OState, n_iter=50, scheme="redblack", omega=None):
    """rhs = div/dt on the interior, solve with the press halo (les.py:358-381)."""
    if omega is None:
        omega = 1.7 if scheme == "redblack" else 1.0
    im, jm, km = st.dims
    spac = np.concatenate([st.dx1, st.dy1, st.dzn])
    if not np.all(spac == spac[0]):
        raise ValueError("build_uniform_coeffs requires uniform spacing on all axes")
    c = uniform_coeffs(im, jm, km, float(spac[0]))
    rhs = np.zeros_like(st.p)
    rhs[1:-1, 1:-1, 1:-1] = divergence(st) / F32(st.dt)
    p, res = solve_pressure(st.p, rhs, c, omega, n_iter, scheme, "press")
    st.p[...] = p
    return res


def check_finite(st: OState, stage: str) -> None:
    for name in FIELDS:
        if not np.isfinite(getattr(st, name)).all():
            raise OracleNumericsError(stage, name)


def step(st: OState, inflow_u, inflow_v, inflow_w, n_iter=50, scheme="redblack") -> OState:
    """The ordered seven stages with a finiteness check after each (les.py:393-416)."""
    runs = (
        ("velnw", lambda: velnw(st)),
        ("bondv1", lambda: bondv1(st, inflow_u, inflow_v, inflow_w)),
        ("velfg", lambda: velfg(st)),
        ("feedbf", lambda: feedbf(st)),
        ("les", lambda: les_viscosity(st)),
        ("adam", lambda: adam(st)),
        ("press", lambda: press(st, n_iter, scheme)),
    )
    with np.errstate(over="ignore", invalid="ignore", divide="ignore"):
        for name, fn in runs:
            fn()
            check_finite(st, name)
    return st


# ---------------------------------------------------------------------------
# synthetic workloads
# ---------------------------------------------------------------------------

def log_inflow(km: int, t_seconds: float = 0.0):
    """WRF-style log-law inflow as driver.generate_profile with the CLI
    defaults (driver.py:44-57; cli.py:38-47): u*=0.05, z0=0.1,
    z_k = 0.1 + 2k, gust 0.2 over 600 s.  f64 maths, f32 output."""
    import math

    z = 0.1 + 2.0 * np.arange(1, km + 1, dtype=np.float64)
    phase = 2.0 * math.pi * ((t_seconds % 600.0) / 600.0)
    gust = 1.0 + 0.2 * math.sin(phase)
    u = (0.05 / 0.41) * np.log(z / 0.1) * gust
    zeros = np.zeros(km, F32)
    return u.astype(F32), zeros, zeros.copy()


def building_mask_config1(im=32, jm=32, km=16):
    """Config 1: one block mask[12:20, 12:20, 1:9] = 1."""
    m = np.zeros((im + 2, jm + 2, km + 2), F32)
    m[12:20, 12:20, 1:9] = 1.0
    return m


def building_mask_3x3(im=150, jm=150, km=90):
    """Config 2: 3x3 building array, 16x16 footprints at i0 = 30+40bi,
    j0 = 30+40bj, heights 10+10((bi+bj) mod 3) from k=1."""
    m = np.zeros((im + 2, jm + 2, km + 2), F32)
    for bi in range(3):
        for bj in range(3):
            i0, j0 = 30 + 40 * bi, 30 + 40 * bj
            h = 10 + 10 * ((bi + bj) % 3)
            m[i0:i0 + 16, j0:j0 + 16, 1:1 + h] = 1.0
    return m
