"""Press-only SOR benchmark (BASELINE.json configs[2]).

rhs[int] = default_rng(0).uniform(-1, 1) float32, p0 = 0, h = 1, red-black
with omega = 1.7, n_iter iterations, halo_fn=None (sor-bench semantics,
cli.py:222-283) or the press halo.  Inputs are device resident (uploaded once);
each timed solve restores p0 with a device copy first (untimed) and is
bracketed by CUDA events on the domain stream, with L2 flushed before it.

  python scripts/bench_press.py [im jm km] [--path 0|1|2|3] [--n-iter 50] [--reps 5] [--halo stored|press]

Prints one JSON line: M cell-iterations/s, us per iteration (median over
--reps timed solves), and the HBM roofline fraction against the algorithmic
bytes of SURVEY 8(d) with cn1 a scalar: red-black 12 B per cell and
iteration (p read + write, rhs read), twinned 24 B (two Jacobi sweeps, each
src read + rhs read + dst write).  --cpu adds the reference's CPU time
(cpu_baseline): the unmodified gmcf_mini.sor.solve_pressure from
baseline/_ref on a bounded number of iterations, extrapolated per
iteration (red-black: 1 thread; twinned: workers = os.cpu_count(), the
reference's only multi-core path, sor.py:292-307).
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT]

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1504_02264_b200 as P  # noqa: E402
from paper_1504_02264_b200 import _native as N  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("dims", nargs="*", type=int, default=[512, 512, 90])
ap.add_argument("--path", type=int, default=0)
ap.add_argument("--n-iter", type=int, default=50)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--halo", default="stored", choices=["stored", "press"])
ap.add_argument("--scheme", default="redblack", choices=["redblack", "twinned"])
ap.add_argument("--cpu", action="store_true", help="also time the reference's CPU solve (bounded sample)")
a = ap.parse_args()
im, jm, km = a.dims
P.runtime.set_sor_path(a.path)
grid = P.Grid.uniform(im, jm, km, 1.0)
fs = P.FlowState.create(grid, dt=1.0)
h = fs.handle()
fs._ensure_coeffs(h)
lib = N.load()
rng = np.random.default_rng(0)
rhs = np.zeros((im + 2, jm + 2, km + 2), np.float32)
rhs[1:-1, 1:-1, 1:-1] = rng.uniform(-1, 1, size=(im, jm, km)).astype(np.float32)
N.check(lib.lesb_upload(h.h, N.LESB_RHS, N.fptr(rhs)), "upload rhs")
p0 = np.zeros_like(rhs)
policy = N.LESB_HALO_STORED if a.halo == "stored" else N.LESB_HALO_PRESS
stream = torch.cuda.ExternalStream(lib.lesb_stream(h.h))
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
res = np.zeros(a.n_iter)
times = []
for r in range(a.reps + 1):
    N.check(lib.lesb_upload(h.h, N.LESB_P, N.fptr(p0)), "upload p0")
    with torch.cuda.stream(stream):
        flush.fill_(float(r))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    rb = a.scheme == "redblack"
    N.check(lib.lesb_sor_solve(h.h, a.n_iter, N.LESB_REDBLACK if rb else N.LESB_TWINNED, 1.7 if rb else 1.0, policy,
                               N.dptr(res)), "sor_solve")
    e1.record(stream)
    torch.cuda.synchronize()
    if r > 0:
        times.append(e0.elapsed_time(e1))
ms = sorted(times)[len(times) // 2]
n = im * jm * km
bpc = 12 if a.scheme == "redblack" else 24
peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0}
gbs = bpc * n * a.n_iter / (ms * 1e-3) / 1e9


def cpu_baseline():
    """The reference's own solve_pressure on host cores (bounded sample)."""
    import time

    ref = os.path.join(ROOT, "baseline", "_ref")
    if ref not in sys.path:
        sys.path.append(ref)
    try:
        from gmcf_mini import sor as rs
    except ImportError:
        return None
    assert rs.solve_pressure.__module__ == "gmcf_mini.sor", "drop-in installed: not the reference"
    c = rs.build_uniform_coeffs(rs.Grid.uniform(im, jm, km, 1.0))
    tw = a.scheme == "twinned"
    workers = os.cpu_count() if tw else 1
    it = 5 if n > 5e6 else 20
    t0 = time.perf_counter()
    rs.solve_pressure(p0, rhs, c, 1.0 if tw else 1.7, it, rs.Scheme.TWINNED if tw else rs.Scheme.REDBLACK,
                      workers=workers)
    sec = (time.perf_counter() - t0) / it
    return {"value": n / sec / 1e6, "unit": "M cell-iterations/s", "cores": workers, "kind": "reference",
            "us_per_iteration": sec * 1e6, "cpu_count": os.cpu_count(),
            "sample": f"{it} iterations of gmcf_mini.sor.solve_pressure ({a.scheme}, workers={workers}), "
                      "per-iteration time extrapolated"}
print(json.dumps({
    "config": (f"press-only {im}x{jm}x{km}, " + ("RB omega 1.7" if a.scheme == "redblack" else "TW omega 1.0") +
               f", {a.n_iter} iterations, halo {a.halo}"),
    "sor_kernel": ({1: "k_sor_rbt", 2: "k_sor_resident", 3: "k_sor_rb"}[lib.lesb_sor_path_in_use(h.h, 0)]
                   if a.scheme == "redblack" else ("k_sor_rbt (twinned sweep)" if lib.lesb_sor_path_in_use(h.h, 0) != 3
                                                   else "k_sor_tw")),
    "ms_per_solve": ms, "us_per_iteration": 1000 * ms / a.n_iter,
    "mcell_iter_per_s": n * a.n_iter / (ms * 1e-3) / 1e6,
    "roofline": {"bytes_per_cell_iteration": bpc, "achieved_gbs": gbs, "peak_gbs": peaks["hbm_gbs"],
                 "frac": gbs / peaks["hbm_gbs"]},
    "cpu_baseline": cpu_baseline() if a.cpu else None,
    "res_first_last": [float(res[0]), float(res[-1])],
    "times_ms": times,
}))
