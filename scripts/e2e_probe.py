"""Where the e2e step time goes (config 2): les.step loop on a resident
state, the raw C-ABI step loop, the bulk window copies alone, and the
pipelined windows.  Host clock, after warm-up."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import golden_inputs as gi  # noqa: E402
import paper_1504_02264_b200 as P  # noqa: E402
from paper_1504_02264_b200 import _native as N  # noqa: E402

st0 = gi.config2_state()
grid = P.Grid(150, 150, 90, st0["dx1"], st0["dy1"], st0["dzn"])
inflow = P.WindProfile(*gi.default_inflow(90))
names = ("u", "v", "w", "fgh", "fgh_old", "p", "mask")
pinned = lambda n: torch.empty(st0[n].shape, dtype=torch.float32, pin_memory=True).numpy()  # noqa: E731
ins = {n: pinned(n) for n in names}
for n in names:
    ins[n][...] = st0[n]
outs = {n: pinned(n) for n in names[:6]}
fs = P.FlowState.create(grid, dt=0.5, vn=0.8, cs=0.14)


def t(fn, reps=5):
    best = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        best.append(time.perf_counter() - t0)
    return min(best) * 1e3, sorted(best)[len(best) // 2] * 1e3


def reset():
    for n in names:
        setattr(fs, n, ins[n])
    fs.handle()


reset()
for _ in range(3):
    P.les.step(fs, inflow)


def steps16():
    reset_dev()
    for _ in range(16):
        P.les.step(fs, inflow)


h = fs.handle()
arrs = [N.f32c(a) for a in (inflow.u, inflow.v, inflow.w)]
stage = N.C.c_int(-1)


def reset_dev():
    fs.stage(**ins)
    fs.commit_staged()
    h.call("lesb_synchronize")


def raw16():
    reset_dev()
    for _ in range(16):
        h.lib.lesb_step(h.h, *[N.fptr(a) for a in arrs], 50, 0, 1.7, None, N.C.byref(stage))


def up():
    fs.stage(**ins)
    h.call("lesb_copies_wait")


def down():
    fs.download_async(outs).wait()


def commit_only():
    fs.stage(**ins)
    h.call("lesb_copies_wait")
    t0 = time.perf_counter()
    fs.commit_staged()
    h.call("lesb_synchronize")
    return time.perf_counter() - t0


for name, fn in (("reset_dev (stage+commit+sync)", reset_dev), ("les.step x16 (+reset)", steps16),
                 ("lesb_step x16 raw (+reset)", raw16), ("upload 7 fields", up), ("download 6 fields", down)):
    fn()
    print(f"{name:34s} min {t(fn)[0]:8.3f} ms  median {t(fn)[1]:8.3f} ms", flush=True)


def steps16_with(copy):
    def fn():
        reset_dev()
        P.les.step(fs, inflow)
        copy()
        for _ in range(15):
            P.les.step(fs, inflow)
        h.call("lesb_copies_wait")
    return fn


per_step = []


def steps16_timed_with(copy):
    reset_dev()
    P.les.step(fs, inflow)
    copy()
    ts = []
    for _ in range(15):
        t0 = time.perf_counter()
        P.les.step(fs, inflow)
        ts.append((time.perf_counter() - t0) * 1e3)
    h.call("lesb_copies_wait")
    return ts


for name, cp in (("nothing", lambda: None), ("stage upload", lambda: fs.stage(**ins)),
                 ("download_async", lambda: fs.download_async(outs))):
    fn = steps16_with(cp)
    fn()
    print(f"16 steps with {name:16s} min {t(fn)[0]:8.3f} ms", flush=True)
    print("   per-step ms:", " ".join(f"{x:.3f}" for x in steps16_timed_with(cp)), flush=True)
