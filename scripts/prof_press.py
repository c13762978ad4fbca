"""Profiling driver: repeated device-resident press (rhs = div/dt, RB SOR with
the press halo) on the benchmark grid.  Usage:
  python scripts/prof_press.py [im jm km] [--path 0|1|2] [--reps N] [--n-iter N]
Prints per-press device time (CUDA events on the domain stream)."""
import argparse, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np
import torch
import golden_inputs as gi
import paper_1504_02264_b200 as P
from paper_1504_02264_b200 import _native as N

ap = argparse.ArgumentParser()
ap.add_argument("dims", nargs="*", type=int, default=[150, 150, 90])
ap.add_argument("--path", type=int, default=0)
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--n-iter", type=int, default=50)
a = ap.parse_args()
im, jm, km = a.dims
P.runtime.set_sor_path(a.path)
st = gi.zero_state(im, jm, km, h=1.0)
rng = np.random.default_rng(0)
g = P.Grid(im, jm, km, st["dx1"], st["dy1"], st["dzn"])
fs = P.FlowState.create(g, dt=0.5, vn=0.8, cs=0.14)
fs.u[...] = rng.uniform(-1, 1, fs.u.shape).astype(np.float32)
h = fs.handle(); fs._ensure_coeffs(h)
lib = N.load()
stream = torch.cuda.ExternalStream(lib.lesb_stream(h.h))
res = np.zeros(a.n_iter)
print("sor path in use:", lib.lesb_sor_path_in_use(h.h, 0))
ts = []
for r in range(a.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    N.check(lib.lesb_press(h.h, a.n_iter, 0, 1.7, N.dptr(res)), "press")
    e1.record(stream)
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
print("press ms:", ["%.3f" % t for t in ts], "per pass us: %.2f" % (1000 * min(ts) / (2 * a.n_iter)))
