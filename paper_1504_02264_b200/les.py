"""Drop-in for ``gmcf_mini.les`` (reference: /root/reference/pkg/src/gmcf_mini/les.py).

``FlowState`` keeps the prognostic fields resident on the GPU and exposes the
reference's attributes (u, v, w, fgh, fgh_old, p, mask as float32 numpy
arrays of the reference shapes, grid, dt, vn, cs, coeffs(), velocities()).

Host/device coherence: reading ``state.u`` returns a host array that is
brought up to date from the device first; any field handed out is assumed
modified and is uploaded before the next device operation.  Keep the rule
of the reference API -- always go through ``state.<field>`` -- and results
are identical; an array object held across a device operation is refreshed
only when ``state.<field>`` is read again.

The module functions also accept the reference's own (numpy) FlowState: the
state is uploaded, the operation runs on the GPU, and the fields the stage
writes are copied back into the caller's arrays.
"""

from __future__ import annotations

import weakref

import numpy as np

from . import _native as N
from . import runtime
from .reftypes import Grid, NumericsError, Scheme, SorCoeffs, is_redblack, is_twinned
from .sor import PressureHalo, build_uniform_coeffs

__all__ = [
    "FlowState", "PendingCopies", "step", "velnw", "bondv1", "velfg_merged", "velfg_twopass", "feedbf",
    "strain_magnitude", "les_viscosity", "adam", "divergence", "press", "_pressure_halo",
    "STAGES", "run_steps", "les_main", "refresh_pressure_faces", "run_boundary_audit",
]

STAGES = N.STAGE_NAMES
_FIELD_ID = {"u": N.LESB_U, "v": N.LESB_V, "w": N.LESB_W, "p": N.LESB_P, "mask": N.LESB_MASK,
             "fgh": N.LESB_FGH, "fgh_old": N.LESB_FGH_OLD}
_ALL = ("u", "v", "w", "fgh", "fgh_old", "p", "mask")
_STAGE_FIELDS = ("u", "v", "w", "fgh", "fgh_old", "p")  # les.py:384


def _csd2(grid: Grid, cs: float):
    """(cs*cbrt(dx*dy*dz))^2 exactly as les.py:305-310 evaluates it; a scalar
    on uniform grids, else a per-cell field."""
    dx = grid.dx1[1:grid.im + 1]
    dy = grid.dy1[1:grid.jm + 1]
    dz = grid.dzn[1:grid.km + 1]
    if np.all(dx == dx[0]) and np.all(dy == dy[0]) and np.all(dz == dz[0]):
        prod = (dx[:1].reshape(1, 1, 1) * dy[:1].reshape(1, 1, 1)) * dz[:1].reshape(1, 1, 1)
        delta = np.cbrt(prod).astype(np.float32)
        val = (np.float32(cs) * delta) ** 2
        return None, float(val.reshape(-1)[0])
    delta = np.cbrt(dx.reshape(-1, 1, 1) * dy.reshape(1, -1, 1) * dz.reshape(1, 1, -1)).astype(np.float32)
    return np.ascontiguousarray((np.float32(cs) * delta) ** 2, dtype=np.float32), 0.0


class _Handle:
    """Owns one lesb_handle (one domain on one device)."""

    def __init__(self, grid: Grid, dt, vn, cs, device: int):
        lib = N.load()
        self.lib = lib
        self.dims = (grid.im, grid.jm, grid.km)
        self._keep = [N.f32c(grid.dx1), N.f32c(grid.dy1), N.f32c(grid.dzn)]
        csd2, csd2s = _csd2(grid, cs)
        desc = N.lesb_desc(grid.im, grid.jm, grid.km, 0, 1, 1, *[N.fptr(a) for a in self._keep],
                           float(dt), float(vn), float(cs), N.fptr(csd2), csd2s, int(device))
        h = N.C.c_void_p()
        N.check(lib.lesb_create(N.C.byref(desc), N.C.byref(h)), "lesb_create")
        self.h = h
        self._fin = weakref.finalize(self, lib.lesb_destroy, h)

    def call(self, name, *args):
        return N.check(getattr(self.lib, name)(self.h, *args), name)


class FlowState:
    """Prognostic state (les.py:37-71), resident on the GPU."""

    def __init__(self, u, v, w, fgh, fgh_old, p, mask, grid: Grid, dt: float, vn: float = 1e-5,
                 cs: float = 0.14, _coeffs: SorCoeffs | None = None):
        self.__dict__["_host"] = {}
        self.__dict__["_dev_newer"] = set()
        self.__dict__["_lent"] = set(_ALL)
        self.__dict__["_h"] = None
        self.__dict__["_pushed_phys"] = None
        self.__dict__["_pushed_coeffs"] = None
        self.__dict__["_staged"] = {}
        for n, a in zip(_ALL, (u, v, w, fgh, fgh_old, p, mask)):
            self._host[n] = a
        self.grid = grid
        self.dt = dt
        self.vn = vn
        self.cs = cs
        self._coeffs = _coeffs

    @classmethod
    def create(cls, grid: Grid, dt: float, vn: float = 1e-5, cs: float = 0.14) -> "FlowState":
        """Zero-filled state (les.py:54-63)."""
        shape = (grid.im + 2, grid.jm + 2, grid.km + 2)
        z = lambda: np.zeros(shape, dtype=np.float32)  # noqa: E731
        st = cls(z(), z(), z(), np.zeros(shape + (3,), np.float32), np.zeros(shape + (3,), np.float32),
                 z(), z(), grid=grid, dt=dt, vn=vn, cs=cs)
        st._lent.clear()  # the device starts zero-filled as well
        return st

    # -- reference API -------------------------------------------------------
    def coeffs(self) -> SorCoeffs:
        if self._coeffs is None:
            self._coeffs = build_uniform_coeffs(self.grid)
        return self._coeffs

    def velocities(self):
        return self.u, self.v, self.w

    # -- coherence -----------------------------------------------------------
    def _pull(self, name):
        if name in self._dev_newer:
            arr = self._host[name]
            if not (isinstance(arr, np.ndarray) and arr.dtype == np.float32 and arr.flags.c_contiguous):
                arr = np.empty(self._shape(name), np.float32)
                self._host[name] = arr
            N.check(self._h.lib.lesb_download(self._h.h, _FIELD_ID[name], N.fptr(arr)), "lesb_download")
            self._dev_newer.discard(name)

    def _shape(self, name):
        g = self.grid
        s = (g.im + 2, g.jm + 2, g.km + 2)
        return s + (3,) if name in ("fgh", "fgh_old") else s

    def sync(self) -> "FlowState":
        """Bring every host array up to date with the device."""
        for n in _ALL:
            self._pull(n)
        return self

    # -- asynchronous copies (overlap with the steps) --------------------------
    def stage(self, **arrays) -> "FlowState":
        """Start copying ``arrays`` (field name -> array of that field's
        shape) to the device without changing the state; they become the state
        at ``commit_staged()``.  The copies overlap device work (fully when the
        arrays are pinned); the arrays must stay unchanged until the first
        device operation after the commit has returned."""
        h = self.handle()
        for n, a in arrays.items():
            if n not in _FIELD_ID:
                raise ValueError(f"unknown field {n!r}")
            a = N.f32c(np.asarray(a))
            if a.shape != self._shape(n):
                raise ValueError(f"field {n} has shape {a.shape}, expected {self._shape(n)}")
            h.call("lesb_stage_upload", _FIELD_ID[n], N.fptr(a))
            self._staged[n] = a
        return self

    def commit_staged(self) -> "FlowState":
        """The staged arrays become the state, in order with the device work
        (as if assigned: ``state.u = a``; a later read of ``state.u`` refreshes
        ``a`` in place)."""
        if not self._staged:
            return self
        self._lent.difference_update(self._staged)
        h = self.handle()
        h.call("lesb_stage_commit")
        for n, a in self._staged.items():
            self._host[n] = a
            self._dev_newer.discard(n)
        self._staged.clear()
        return self

    def download_async(self, out: dict) -> "PendingCopies":
        """Enqueue copies of the fields named by ``out`` (name -> float32
        C-contiguous array of the field's shape; pinned memory overlaps fully)
        as they stand after the device work enqueued so far, and return at
        once.  Later steps do not disturb the copies (the device snapshots
        the fields first).  The arrays are complete after ``wait()`` on the
        returned object."""
        h = self.handle()
        for n, a in out.items():
            if n not in _FIELD_ID:
                raise ValueError(f"unknown field {n!r}")
            if not (isinstance(a, np.ndarray) and a.dtype == np.float32 and a.flags.c_contiguous
                    and a.flags.writeable and a.shape == self._shape(n)):
                raise ValueError(f"out[{n!r}] must be a writeable C-contiguous float32 array of shape "
                                 f"{self._shape(n)}")
            h.call("lesb_download_async", _FIELD_ID[n], N.fptr(a))
        return PendingCopies(h, out)

    def handle(self) -> _Handle:
        """The device domain, with host-side changes uploaded."""
        if self._h is None:
            self.__dict__["_h"] = _Handle(self.grid, self.dt, self.vn, self.cs, runtime.current_device())
            self.__dict__["_pushed_phys"] = (self.dt, self.vn, self.cs)
        h = self._h
        phys = (self.dt, self.vn, self.cs)
        if phys != self._pushed_phys:
            csd2, csd2s = _csd2(self.grid, self.cs)
            N.check(h.lib.lesb_set_physics(h.h, float(self.dt), float(self.vn), float(self.cs), N.fptr(csd2),
                                           csd2s), "lesb_set_physics")
            self.__dict__["_pushed_phys"] = phys
        for n in list(self._lent):
            arr = np.asarray(self._host[n])
            if arr.shape != self._shape(n):
                raise ValueError(f"field {n} has shape {arr.shape}, expected {self._shape(n)}")
            arr = N.f32c(arr)
            N.check(h.lib.lesb_upload(h.h, _FIELD_ID[n], N.fptr(arr)), "lesb_upload")
        self._lent.clear()
        return h

    def _ensure_coeffs(self, h: _Handle):
        c = self.coeffs()
        if self._pushed_coeffs is not c:
            keep: list = []
            cf = N.make_coeffs(c, keep)
            N.check(h.lib.lesb_set_coeffs(h.h, N.C.byref(cf)), "lesb_set_coeffs")
            self.__dict__["_pushed_coeffs"] = c

    def _device_wrote(self, names):
        self._dev_newer.update(names)
        self._lent.difference_update(names)

    def __repr__(self):
        g = self.grid
        return f"FlowState(device, {g.im}x{g.jm}x{g.km}, dt={self.dt}, vn={self.vn}, cs={self.cs})"


class PendingCopies:
    """Asynchronous downloads in flight (FlowState.download_async)."""

    def __init__(self, h: _Handle, out: dict):
        self._h = h
        self.out = out

    def wait(self) -> dict:
        self._h.call("lesb_copies_wait")
        return self.out


def _field_property(name):
    def get(self):
        self._pull(name)
        self._lent.add(name)
        return self._host[name]

    def set_(self, value):
        self._host[name] = value
        self._dev_newer.discard(name)
        self._lent.add(name)

    return property(get, set_)


for _n in _ALL:
    setattr(FlowState, _n, _field_property(_n))


# ---------------------------------------------------------------------------
# reference FlowState objects: upload, run, copy the written fields back
# ---------------------------------------------------------------------------
# The reference FlowState is a non-frozen @dataclass: __hash__ is None, so it
# cannot key a WeakKeyDictionary.  The device twin is cached by id() and the
# entry is evicted by a finalizer when the caller's object dies (the weak
# reference also guards against a recycled id).
_compat: dict = {}


def _compat_lookup(state):
    ent = _compat.get(id(state))
    if ent is not None and ent[0]() is state:
        return ent[1]
    return None


def _compat_store(state, ds):
    key = id(state)
    try:
        ref = weakref.ref(state)
    except TypeError:  # no weak references (e.g. __slots__): do not cache
        return
    _compat[key] = (ref, ds)
    weakref.finalize(state, _compat.pop, key, None)


def _resolve(state):
    """(device state, write-back target or None)."""
    if isinstance(state, FlowState):
        return state, None
    ds = _compat_lookup(state)
    g = state.grid
    if ds is None or ds.grid is not g:
        ds = FlowState(state.u, state.v, state.w, state.fgh, state.fgh_old, state.p, state.mask, g,
                       state.dt, state.vn, state.cs)
        _compat_store(state, ds)
    for n in _ALL:
        ds._host[n] = getattr(state, n)
    ds._dev_newer.clear()
    ds._lent.update(_ALL)
    ds.dt, ds.vn, ds.cs = state.dt, state.vn, state.cs
    if getattr(state, "_coeffs", None) is not None:
        ds._coeffs = state._coeffs
    return ds, state


def _writeback(ds: FlowState, target, names):
    if target is None:
        return
    for n in names:
        if n in ds._dev_newer:
            arr = getattr(target, n)
            if isinstance(arr, np.ndarray) and arr.dtype == np.float32 and arr.flags.c_contiguous:
                N.check(ds._h.lib.lesb_download(ds._h.h, _FIELD_ID[n], N.fptr(arr)), "lesb_download")
            else:
                out = np.empty(ds._shape(n), np.float32)
                N.check(ds._h.lib.lesb_download(ds._h.h, _FIELD_ID[n], N.fptr(out)), "lesb_download")
                arr[...] = out
            ds._dev_newer.discard(n)


def _stage(state, fn_name, writes, *args):
    ds, target = _resolve(state)
    h = ds.handle()
    h.call(fn_name, *args)
    ds._device_wrote(writes)
    _writeback(ds, target, writes)


# ---------------------------------------------------------------------------
# stages
# ---------------------------------------------------------------------------
def velnw(state) -> None:
    """u += dt*(fgh - grad p), staggered, faces 0..N (les.py:218-241)."""
    _stage(state, "lesb_velnw", ("u", "v", "w"))


def refresh_pressure_faces(state) -> None:
    """The pressure halo refresh (les.py:341-355) on the face-interior halo
    cells -- the cells the SOR stencil reads -- launched over the paper's
    boundary-range geometry (sor.py:312-349): one GPU launch of
    padded_range(boundary_range(im, jm, km), 256, 1) threads, each decoding
    its gid to a face point.  Edges and corners are left unchanged."""
    _stage(state, "lesb_boundp_faces", ("p",))


def _inflow_arrays(inflow, km):
    kp = inflow.kp if hasattr(inflow, "kp") else len(inflow.u)
    if kp != km:
        raise ValueError(f"inflow has {kp} levels, grid has km={km}")
    return [N.f32c(getattr(inflow, c)) for c in ("u", "v", "w")]


def bondv1(state, inflow) -> None:
    """Velocity halos: inflow W, zero-gradient E, periodic y, free-slip z (les.py:244-266)."""
    arrs = _inflow_arrays(inflow, state.grid.km)
    _stage(state, "lesb_bondv1", ("u", "v", "w"), *[N.fptr(a) for a in arrs])


def velfg_merged(state) -> None:
    """Advection + diffusion force into fgh's interior (les.py:178-192)."""
    _stage(state, "lesb_velfg", ("fgh",))


def velfg_twopass(state) -> None:
    """Bitwise equal to velfg_merged by contract (les.py:195-215); same kernel."""
    _stage(state, "lesb_velfg", ("fgh",))


def feedbf(state) -> None:
    """Building feedback force and velocity masking (les.py:269-282)."""
    _stage(state, "lesb_feedbf", ("fgh", "u", "v", "w"))


def les_viscosity(state) -> None:
    """Smagorinsky eddy viscosity added to fgh; no-op at cs == 0 (les.py:299-320)."""
    if state.cs == 0.0:
        return
    _stage(state, "lesb_les_viscosity", ("fgh",))


def adam(state) -> None:
    """fgh <- 1.5 fgh - 0.5 fgh_old; fgh_old <- previous fgh (les.py:323-327)."""
    _stage(state, "lesb_adam", ("fgh", "fgh_old"))


def _interior_out(state, fn_name):
    ds, _ = _resolve(state)
    g = ds.grid
    out = np.empty((g.im, g.jm, g.km), np.float32)
    ds.handle().call(fn_name, N.fptr(out))
    return out


def strain_magnitude(state) -> np.ndarray:
    """|S| over the interior (les.py:285-296)."""
    return _interior_out(state, "lesb_strain_magnitude")


def divergence(state) -> np.ndarray:
    """Staggered divergence over the interior (les.py:330-338)."""
    return _interior_out(state, "lesb_divergence")


def _pressure_halo(grid: Grid):
    """The press boundary policy (les.py:341-355); as ``halo_fn`` it selects
    the device's PRESS policy."""
    return PressureHalo(grid)


def _scheme_code(scheme):
    if is_redblack(scheme):
        return N.LESB_REDBLACK
    if is_twinned(scheme):
        return N.LESB_TWINNED
    raise ValueError(f"unknown scheme {scheme!r}")


def _check_solver_args(n_iter, scheme, workers):
    """solve_pressure's validation (sor.py:264-269)."""
    if n_iter < 1:
        raise ValueError("n_iter must be >= 1")
    if workers < 1:
        raise ValueError("workers must be >= 1")
    if is_redblack(scheme) and workers > 1:
        raise ValueError("REDBLACK supports workers=1 only; use TWINNED for parallel runs")


def press(state, n_iter: int = 50, scheme: Scheme = Scheme.REDBLACK, omega: float | None = None,
          workers: int = 1) -> np.ndarray:
    """rhs = div(u)/dt; SOR with the press halo; p replaced in place.
    Returns the float64 residual history (les.py:358-381)."""
    if omega is None:
        omega = 1.7 if is_redblack(scheme) else 1.0
    sch = _scheme_code(scheme)
    _check_solver_args(n_iter, scheme, workers)
    ds, target = _resolve(state)
    h = ds.handle()
    ds._ensure_coeffs(h)
    res = np.zeros(n_iter, np.float64)
    h.call("lesb_press", int(n_iter), sch, float(omega), N.dptr(res))
    ds._device_wrote(("p",))
    _writeback(ds, target, ("p",))
    return res


def _check_finite(ds: FlowState, stage: str):
    ok = N.C.c_int(0)
    ds.handle().call("lesb_check_finite", N.C.byref(ok))
    if not ok.value:
        raise NumericsError(stage, "device finiteness check")


def _step_staged(state, inflow, n_iter, scheme, workers):
    """Stage-by-stage step with a full finiteness scan after each stage: the
    exact reference control flow (les.py:393-416), used when an argument
    error must surface mid-step as it does in the reference."""
    ds, target = _resolve(state)
    runs = (
        ("velnw", lambda: velnw(ds)),
        ("bondv1", lambda: bondv1(ds, inflow)),
        ("velfg", lambda: velfg_merged(ds)),
        ("feedbf", lambda: feedbf(ds)),
        ("les", lambda: les_viscosity(ds)),
        ("adam", lambda: adam(ds)),
        ("press", lambda: press(ds, n_iter, scheme, workers=workers)),
    )
    try:
        for name, run in runs:
            run()
            _check_finite(ds, name)
    finally:
        _writeback(ds, target, _STAGE_FIELDS)
    return state


def step(state, inflow, n_iter: int = 50, scheme: Scheme = Scheme.REDBLACK, workers: int = 1):
    """Advance one time step through the seven stages (les.py:393-416) as one
    CUDA-graph replay.  Raises NumericsError(stage) after the first stage
    that leaves a non-finite value."""
    g = state.grid
    kp = inflow.kp if hasattr(inflow, "kp") else len(inflow.u)
    bad_args = kp != g.km or n_iter < 1 or workers < 1 or (is_redblack(scheme) and workers > 1)
    if bad_args or not (is_redblack(scheme) or is_twinned(scheme)):
        return _step_staged(state, inflow, n_iter, scheme, workers)
    arrs = _inflow_arrays(inflow, g.km)
    ds, target = _resolve(state)
    h = ds.handle()
    ds._ensure_coeffs(h)
    omega = 1.7 if is_redblack(scheme) else 1.0
    stage = N.C.c_int(-1)
    rc = h.call("lesb_step", *[N.fptr(a) for a in arrs], int(n_iter), _scheme_code(scheme), float(omega), None,
                N.C.byref(stage))
    ds._device_wrote(_STAGE_FIELDS)
    _writeback(ds, target, _STAGE_FIELDS)
    if rc == N.LESB_NONFINITE:
        raise NumericsError(STAGES[stage.value], "device stage check")
    return state


def run_steps(state, inflow, n_steps: int, n_iter: int = 50, scheme: Scheme = Scheme.REDBLACK) -> int:
    """``n_steps`` calls of ``step`` with one host synchronisation at the
    end.  ``inflow`` is one WindProfile or a sequence (one per step).  Returns
    the number of steps completed; raises NumericsError (with ``.step`` set
    to the 0-based failing step and the reference's stage name) like the
    step-by-step loop would.  The steps are enqueued before a failure is
    known: after the error the fields hold the end of the last enqueued step,
    not the reference's state after the failing stage (use ``step`` for
    that)."""
    g = state.grid
    profs = list(inflow) if isinstance(inflow, (list, tuple)) else [inflow]
    block = np.stack([np.concatenate(_inflow_arrays(pr, g.km)) for pr in profs]).astype(np.float32)
    ds, target = _resolve(state)
    h = ds.handle()
    ds._ensure_coeffs(h)
    omega = 1.7 if is_redblack(scheme) else 1.0
    done = N.C.c_int(0)
    stage = N.C.c_int(-1)
    rc = h.call("lesb_run_steps", int(n_steps), N.fptr(np.ascontiguousarray(block)), len(profs), int(n_iter),
                _scheme_code(scheme), float(omega), N.C.byref(done), N.C.byref(stage))
    ds._device_wrote(_STAGE_FIELDS)
    _writeback(ds, target, _STAGE_FIELDS)
    if rc == N.LESB_NONFINITE:
        err = NumericsError(STAGES[stage.value], f"device stage check at step {done.value}")
        err.step = done.value
        raise err
    return done.value


def les_main(tile, model_id: int, flow, peers, n_steps: int, interval_microsteps: int, dt_microsteps: int = 1,
             data_id=None, sor_iters: int = 50, scheme: Scheme = Scheme.REDBLACK, record: dict | None = None,
             coupling_module=None):
    """The coupled LES loop (les.py:419-470) with the flow resident on the GPU.

    Same protocol as the reference -- sync every step, request a profile at
    coupled boundaries, interpolate at (t - interval) once two profiles exist
    (coupling.py:168-270, 366-388) -- but the state is uploaded once, every
    step is one CUDA-graph replay with the step's inflow (km x 3 floats) as
    its only host input, and the fields are copied back into ``flow`` when the
    loop ends (also when a stage fails: ``flow`` then holds the end of the
    failing step, the error names the reference stage).  ``coupling_module``
    defaults to ``gmcf_mini.coupling``.
    """
    if coupling_module is None:
        import importlib

        coupling_module = importlib.import_module("gmcf_mini.coupling")
    cp = coupling_module
    if data_id is None:
        data_id = cp.WIND_PROFILE_DATA_ID
    finished_status = cp.SyncStatus.PEER_FINISHED
    dev, target = _resolve(flow)
    state = cp.init(tile, model_id, peers, dt_microsteps, interval_microsteps)
    steps_done = 0
    interval_idx = 0
    first_interp = None
    boundaries: list = []
    try:
        for _ in range(n_steps):
            if cp.sync(state) is finished_status:
                break
            t = state.current_time
            if t % interval_microsteps == 0:
                got = cp.pre_exchange(state, data_id)
                if got is finished_status:
                    break
                interval_idx += 1
                boundaries.append({"interval": interval_idx, "time": t, "steps_before": steps_done})
            if state.series.can_interpolate:
                inflow = cp.interpolate_profile(state.series, t - interval_microsteps)
                if first_interp is None:
                    first_interp = interval_idx
            else:
                inflow = state.series.next
            step(dev, inflow, n_iter=sor_iters, scheme=scheme)
            steps_done += 1
            cp.advance_step(state)
    finally:
        if target is not None:
            for n in _STAGE_FIELDS:
                dev._dev_newer.add(n)
            _writeback(dev, target, _STAGE_FIELDS)
    cp.finished(state)
    cp.await_peer_fins(state)
    if record is not None:
        record["steps"] = steps_done
        record["first_interpolation_interval"] = first_interp
        record["boundaries"] = boundaries
        record["profiles_received"] = state.series.count_received
    return state


def run_boundary_audit(cfg, out_dir):
    """``boundary-audit`` mode (cli.py:286-320) with the decode on the GPU.

    The reference walks every gid of the padded range through
    map_boundary_gid in Python; here one launch of blocks of cfg.nthreads
    threads x cfg.nunits gids decodes them all (sor.boundary_audit) and the
    checks are the reference's: every boundary point covered exactly once,
    no in-range gid in the padding branch, no padding gid escaping the guard.
    Prints the reference's line and writes the same summary.json."""
    from pathlib import Path

    from . import dump as _dump
    from . import sor as _sor
    from .reftypes import GmcfError

    ip, jp, kp = cfg.im, cfg.jm, cfg.km
    st = _sor.boundary_audit(ip, jp, kp, cfg.nthreads, cfg.nunits)
    br, pr = st["boundary_range"], st["padded_range"]
    if st["range_gids_in_padding"]:
        raise GmcfError(f"coverage violation: gid {st['first_violation']} mapped to padding inside the range")
    if st["covered_more"]:
        raise GmcfError(f"coverage violation: {st['covered_more']} boundary points hit more than once")
    expected = jp * kp + kp * ip + jp * ip
    if st["covered_once"] != expected:
        raise GmcfError(f"coverage violation: {st['covered_once']} points covered, expected {expected}")
    if st["padding_escapes"]:
        raise GmcfError(f"padding violation: gid {st['first_violation']} escaped the guard")
    print(
        f"boundary audit ok: domain=({ip},{jp},{kp}) m={cfg.nthreads * cfg.nunits} "
        f"covered={br} padding={pr - br}",
        flush=True,
    )
    summary = {
        "mode": "boundary-audit",
        "domain": [ip, jp, kp],
        "boundary_range": br,
        "padded_range": pr,
        "padding_gids": pr - br,
    }
    _dump.write_json(Path(out_dir) / "summary.json", summary)
    return summary

