import os, sys, time
import numpy as np, torch
ROOT=os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path[:0]=[ROOT, ROOT+"/tests"]
import golden_inputs as gi
import paper_1504_02264_b200 as P
from paper_1504_02264_b200 import _native as N
st0 = gi.config2_state()
grid = P.Grid(150,150,90, st0["dx1"], st0["dy1"], st0["dzn"])
inflow = P.WindProfile(*gi.default_inflow(90))
fs = P.FlowState.create(grid, dt=0.5, vn=0.8, cs=0.14)
fs.mask[...] = st0["mask"]
h = fs.handle(); fs._ensure_coeffs(h)
lib = h.lib
arrs = [N.f32c(a) for a in (inflow.u, inflow.v, inflow.w)]
stage = N.C.c_int(-1)
N.check(lib.lesb_set_inflow(h.h, *[N.fptr(a) for a in arrs]), "inflow")
pristine = {n: getattr(fs, n).copy() for n in ("u","v","w","fgh","fgh_old","p")}
def reset():
    for n,a in pristine.items(): setattr(fs, n, a)
    fs.handle(); h.call("lesb_synchronize")
def run(kind, n=16):
    reset()
    t0=time.perf_counter()
    for _ in range(n):
        if kind=="sync": lib.lesb_step(h.h, *[N.fptr(a) for a in arrs], 50, 0, 1.7, None, N.C.byref(stage))
        elif kind=="async_each": lib.lesb_step_async(h.h, 50, 0, 1.7); lib.lesb_synchronize(h.h)
        else: lib.lesb_step_async(h.h, 50, 0, 1.7)
    lib.lesb_synchronize(h.h)
    return (time.perf_counter()-t0)/n*1e6
for kind in ("sync","async_each","async_batch"):
    run(kind)
    xs=[run(kind) for _ in range(5)]
    print(f"{kind:12s} per step us: min {min(xs):.1f} med {sorted(xs)[2]:.1f}")
