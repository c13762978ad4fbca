"""x-slab decomposition of the LES step over several GPUs.

The grid is cut along x (the slowest axis) into slabs of whole (j, k) planes,
so every halo exchange moves contiguous (jm+2)(km+2) planes; y stays local,
so the periodic wrap stays a local remap.  The kernels see a slab through its
geometry (``i_offset`` for the global red-black colour, ``west/east_boundary``
for which x faces are physical) and keep a depth-2 high-x velocity halo for
velfg's shifted derivative (les.py:100-110).  The exchange schedule is the
one SURVEY 8(e) verified by CPU emulation: velocities after velnw + bondv1
(depth 1 low, 2 high), pressure after every colour pass / sweep and after the
final halo, residuals summed once per press, stage flags OR-ed once per step.

Two drivers over the same C ABI:
  * ``SlabGroup``: n slabs in one process on one device, stepped together
    with plane copies (lesb_group_step) -- the single-GPU bitwise check of
    the decomposition;
  * ``SlabDomain``: one slab per process / GPU, NCCL send/recv of the halo
    planes inside the step's CUDA graph (lesb_link_nccl); the unique id and
    the stage-flag / residual reductions go through torch.distributed.
"""

from __future__ import annotations

import numpy as np

from . import _native as N
from .les import _FIELD_ID, _check_solver_args, _csd2, _inflow_arrays, _scheme_code
from .reftypes import Grid, NumericsError, Scheme, is_redblack
from .sor import build_uniform_coeffs

FIELDS = ("u", "v", "w", "fgh", "fgh_old", "p", "mask")
STATE = ("u", "v", "w", "fgh", "fgh_old", "p")


def slab_bounds(im: int, nslabs: int, s: int) -> tuple[int, int]:
    """Global interior planes [i0, i1] (1-based, inclusive) of slab s: the
    first im % nslabs slabs get one plane more."""
    if not 1 <= nslabs <= im:
        raise ValueError(f"cannot cut {im} planes into {nslabs} slabs")
    base, extra = divmod(im, nslabs)
    i0 = 1 + s * base + min(s, extra)
    return i0, i0 + base + (1 if s < extra else 0) - 1


def halo_plan(im_local: int, west: bool, east: bool, depth: int):
    """The plane exchange one slab performs (mirrors capi.cu nccl_exchange):
    a list of (op, peer, first local plane, number of planes) with peer -1 =
    west, +1 = east.  Used by the CPU tests to check the schedule."""
    plan = []
    if west:
        plan += [("send", -1, 1, depth), ("recv", -1, 0, 1)]
    if east:
        plan += [("send", +1, im_local, 1), ("recv", +1, im_local + 1, depth)]
    return plan


def slice_global(arr: np.ndarray, i0: int, i1: int) -> np.ndarray:
    """The slab's Python-visible array: global planes i0-1 .. i1+1."""
    return np.ascontiguousarray(arr[i0 - 1:i1 + 2])


def gather(parts: list[np.ndarray], bounds: list[tuple[int, int]]) -> np.ndarray:
    """Global array from slab arrays: interior planes from their owners, the
    west halo plane from the first slab, the east one from the last."""
    first = parts[0]
    im = bounds[-1][1]
    out = np.empty((im + 2,) + first.shape[1:], first.dtype)
    out[0] = parts[0][0]
    for part, (i0, i1) in zip(parts, bounds):
        out[i0:i1 + 1] = part[1:i1 - i0 + 2]
    out[im + 1] = parts[-1][-1]
    return out


class _Slab:
    """One slab domain (lesb_handle) with its geometry."""

    def __init__(self, grid: Grid, dt, vn, cs, i0: int, i1: int, device: int):
        lib = N.load()
        self.lib = lib
        self.i0, self.i1 = i0, i1
        im = i1 - i0 + 1
        self.im = im
        g = grid
        # spacings: global dx1[i0-1 .. i1+2] (im+3 entries)
        dx = np.asarray(g.dx1, np.float32)
        self._keep = [np.ascontiguousarray(dx[i0 - 1:i1 + 3]), N.f32c(g.dy1), N.f32c(g.dzn)]
        csd2, csd2s = _csd2(g, cs)
        if csd2 is not None:
            csd2 = np.ascontiguousarray(csd2[i0 - 1:i1])
            self._keep.append(csd2)
        desc = N.lesb_desc(im, g.jm, g.km, i0 - 1, int(i0 == 1), int(i1 == g.im),
                           *[N.fptr(a) for a in self._keep[:3]], float(dt), float(vn), float(cs),
                           N.fptr(csd2), csd2s, int(device))
        h = N.C.c_void_p()
        N.check(lib.lesb_create(N.C.byref(desc), N.C.byref(h)), "lesb_create")
        self.h = h
        self._staged: list = []
        self._committed: list = []
        c = build_uniform_coeffs(g)
        keep: list = []
        cf = N.make_coeffs(c, keep)
        # coefficient vectors restricted to the slab (cn2l/cn2s are per x plane)
        if cf.cn1:
            raise NotImplementedError("slabs need a scalar cn1 (uniform grids)")
        ax = [np.ascontiguousarray(np.asarray(getattr(c, n), np.float32)[i0 - 1:i1]) for n in ("cn2l", "cn2s")]
        keep.extend(ax)
        cf.cn2l, cf.cn2s = N.fptr(ax[0]), N.fptr(ax[1])
        N.check(lib.lesb_set_coeffs(h, N.C.byref(cf)), "lesb_set_coeffs")

    def upload(self, name, global_arr):
        part = slice_global(np.asarray(global_arr, np.float32), self.i0, self.i1)
        fid = N.LESB_RHS if name == "rhs" else _FIELD_ID[name]
        N.check(self.lib.lesb_upload(self.h, fid, N.fptr(part)), "lesb_upload")

    # asynchronous copies (les.FlowState.stage / commit_staged / download_async)
    def stage(self, name, global_arr):
        part = slice_global(np.asarray(global_arr, np.float32), self.i0, self.i1)  # (a view when contiguous)
        self._staged.append(part)  # alive until the copy has run
        N.check(self.lib.lesb_stage_upload(self.h, _FIELD_ID[name], N.fptr(part)), "lesb_stage_upload")

    def commit_staged(self):
        N.check(self.lib.lesb_stage_commit(self.h), "lesb_stage_commit")
        self._committed, self._staged = self._staged, []  # (dropped at the next commit: the steps between synchronise)

    def download_async(self, name, out):
        N.check(self.lib.lesb_download_async(self.h, _FIELD_ID[name], N.fptr(out)), "lesb_download_async")

    def copies_wait(self):
        N.check(self.lib.lesb_copies_wait(self.h), "lesb_copies_wait")

    def download(self, name, jm, km):
        shape = (self.im + 2, jm + 2, km + 2) + ((3,) if name in ("fgh", "fgh_old") else ())
        out = np.empty(shape, np.float32)
        N.check(self.lib.lesb_download(self.h, _FIELD_ID[name], N.fptr(out)), "lesb_download")
        return out

    def close(self):
        if self.h is not None:
            self.lib.lesb_destroy(self.h)
            self.h = None


class SlabGroup:
    """``nslabs`` x-slabs of one grid in this process, on one device."""

    def __init__(self, grid: Grid, nslabs: int, dt: float, vn: float = 1e-5, cs: float = 0.14, device: int = 0):
        self.grid = grid
        self.bounds = [slab_bounds(grid.im, nslabs, s) for s in range(nslabs)]
        self.slabs = [_Slab(grid, dt, vn, cs, i0, i1, device) for i0, i1 in self.bounds]
        arr = (N.C.c_void_p * nslabs)(*[s.h for s in self.slabs])
        self._arr = arr
        N.check(N.load().lesb_link_local(arr, nslabs), "lesb_link_local")

    def upload(self, state: dict):
        for name in FIELDS:
            for s in self.slabs:
                s.upload(name, state[name])

    def step(self, inflow, n_iter: int = 50, scheme: Scheme = Scheme.REDBLACK):
        g = self.grid
        arrs = _inflow_arrays(inflow, g.km)
        res = np.zeros(n_iter, np.float64)
        stage = N.C.c_int(-1)
        omega = 1.7 if is_redblack(scheme) else 1.0
        rc = N.check(N.load().lesb_group_step(self._arr, len(self.slabs), *[N.fptr(a) for a in arrs], int(n_iter),
                                              _scheme_code(scheme), float(omega), N.dptr(res), N.C.byref(stage)),
                     "lesb_group_step")
        if rc == N.LESB_NONFINITE:
            raise NumericsError(N.STAGE_NAMES[stage.value], "device stage check (slabs)")
        return res

    def solve(self, p0: np.ndarray, rhs: np.ndarray, omega: float, n_iter: int, scheme: Scheme = Scheme.REDBLACK,
              halo_policy: int = 0):
        """solve_pressure (sor.py:255-309) on the slabs: the global p0 and rhs
        are cut into the slabs, solved together (lesb_group_sor_solve) and p
        gathered back.  Returns (p, residuals): p bitwise equal to the
        single-domain solve; residuals summed over the slabs in order."""
        _check_solver_args(n_iter, scheme, 1)
        for s in self.slabs:
            s.upload("p", p0)
            s.upload("rhs", rhs)
        res = np.zeros(n_iter, np.float64)
        N.check(N.load().lesb_group_sor_solve(self._arr, len(self.slabs), int(n_iter), _scheme_code(scheme),
                                              float(omega), int(halo_policy), N.dptr(res)), "lesb_group_sor_solve")
        return self.gather("p"), res

    def gather(self, name: str) -> np.ndarray:
        g = self.grid
        return gather([s.download(name, g.jm, g.km) for s in self.slabs], self.bounds)

    def close(self):
        for s in self.slabs:
            s.close()


class _SlabPending:
    def __init__(self, slab, out):
        self._slab = slab
        self.out = out

    def wait(self) -> dict:
        self._slab.copies_wait()
        return self.out


class SlabDomain:
    """This rank's x-slab in a one-process-per-GPU run (torch.distributed
    initialised; NCCL for the device exchanges)."""

    def __init__(self, grid: Grid, dt: float, vn: float = 1e-5, cs: float = 0.14, device: int = 0):
        import torch.distributed as dist

        self.dist = dist
        self.rank, self.nranks = dist.get_rank(), dist.get_world_size()
        self.grid = grid
        self.bounds = [slab_bounds(grid.im, self.nranks, s) for s in range(self.nranks)]
        i0, i1 = self.bounds[self.rank]
        self.slab = _Slab(grid, dt, vn, cs, i0, i1, device)
        uid = N.C.create_string_buffer(128)
        if self.rank == 0:
            N.check(N.load().lesb_nccl_unique_id(uid, 128), "lesb_nccl_unique_id")
        box = [uid.raw if self.rank == 0 else None]
        dist.broadcast_object_list(box, src=0)
        uid = N.C.create_string_buffer(box[0], 128)
        N.check(N.load().lesb_link_nccl(self.slab.h, uid, self.nranks, self.rank), "lesb_link_nccl")

    def upload(self, state: dict):
        for name in FIELDS:
            self.slab.upload(name, state[name])

    def stage(self, state: dict):
        """Start copying this rank's part of the global fields in ``state``
        (pinned arrays overlap fully) to the device; they become the slab's
        state at ``commit_staged()`` (les.FlowState.stage)."""
        for name in FIELDS:
            if name in state:
                self.slab.stage(name, state[name])

    def commit_staged(self):
        self.slab.commit_staged()

    def download_async(self, out: dict):
        """Enqueue copies of this rank's slab fields into ``out`` (name ->
        float32 C-contiguous array of the slab's shape, ``slab_shape(name)``)
        as they stand after the work enqueued so far; ``wait()`` on the
        returned object completes them (les.FlowState.download_async)."""
        for n, a in out.items():
            if not (isinstance(a, np.ndarray) and a.dtype == np.float32 and a.flags.c_contiguous
                    and a.shape == self.slab_shape(n)):
                raise ValueError(f"out[{n!r}] must be a C-contiguous float32 array of shape {self.slab_shape(n)}")
            self.slab.download_async(n, a)
        return _SlabPending(self.slab, out)

    def slab_shape(self, name):
        g = self.grid
        return (self.slab.im + 2, g.jm + 2, g.km + 2) + ((3,) if name in ("fgh", "fgh_old") else ())

    def step(self, inflow, n_iter: int = 50, scheme: Scheme = Scheme.REDBLACK, residuals: bool = False):
        """One step (les.py:393-416) on every rank.  The library reduces the
        first failing stage over the ranks with NCCL, so
        every rank raises the same NumericsError; with ``residuals`` the
        press residual history is the NCCL sum over the slabs (C4)."""
        g = self.grid
        arrs = _inflow_arrays(inflow, g.km)
        stage = N.C.c_int(-1)
        omega = 1.7 if is_redblack(scheme) else 1.0
        res = np.zeros(n_iter, np.float64) if residuals else None
        rc = N.check(self.slab.lib.lesb_step(self.slab.h, *[N.fptr(a) for a in arrs], int(n_iter),
                                             _scheme_code(scheme), float(omega), N.dptr(res), N.C.byref(stage)),
                     "lesb_step")
        if rc == N.LESB_NONFINITE:
            raise NumericsError(N.STAGE_NAMES[stage.value], "device stage check (slabs)")
        return res

    def press(self, n_iter: int = 50, scheme: Scheme = Scheme.REDBLACK, omega: float | None = None) -> np.ndarray:
        """press (les.py:358-381) on the slabs: rhs from the slab's
        velocities, SOR with the press halo and the per-pass plane exchange;
        returns the global residual history (NCCL sum, C4) on every rank."""
        if omega is None:
            omega = 1.7 if is_redblack(scheme) else 1.0
        res = np.zeros(n_iter, np.float64)
        N.check(self.slab.lib.lesb_press(self.slab.h, int(n_iter), _scheme_code(scheme), float(omega), N.dptr(res)),
                "lesb_press")
        return res

    def solve(self, p0: np.ndarray, rhs: np.ndarray, omega: float, n_iter: int, scheme: Scheme = Scheme.REDBLACK,
              halo_policy: int = 0):
        """solve_pressure (sor.py:255-309) decomposed over the ranks: every
        rank passes the GLOBAL p0 and rhs (as sor-bench builds them), solves
        its slab, and gets its slab of p (global planes i0-1 .. i1+1) and the
        global residual history (NCCL sum over the slabs)."""
        _check_solver_args(n_iter, scheme, 1)
        self.slab.upload("p", p0)
        self.slab.upload("rhs", rhs)
        res = np.zeros(n_iter, np.float64)
        N.check(self.slab.lib.lesb_sor_solve(self.slab.h, int(n_iter), _scheme_code(scheme), float(omega),
                                             int(halo_policy), N.dptr(res)), "lesb_sor_solve")
        return self.slab.download("p", self.grid.jm, self.grid.km), res

    def gather(self, name: str):
        """The global array of a field on rank 0 (None elsewhere): every
        rank's slab travels to rank 0 (for dumps)."""
        part = self.slab.download(name, self.grid.jm, self.grid.km)
        parts = [None] * self.nranks if self.rank == 0 else None
        self.dist.gather_object(part, parts, dst=0)
        if self.rank != 0:
            return None
        return gather(parts, self.bounds)

    def close(self):
        self.slab.close()
