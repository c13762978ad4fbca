"""Per-pass phase timeline of the resident SOR kernel (LESB_RES_TRACE=1)."""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
os.environ["LESB_RES_TRACE"] = "1"
import numpy as np
import golden_inputs as gi
import paper_1504_02264_b200 as P
from paper_1504_02264_b200 import _native as N
im, jm, km = 150, 150, 90
st = gi.zero_state(im, jm, km, h=1.0)
g = P.Grid(im, jm, km, st["dx1"], st["dy1"], st["dzn"])
fs = P.FlowState.create(g, dt=0.5, vn=0.8, cs=0.14)
fs.u[...] = np.random.default_rng(0).uniform(-1, 1, fs.u.shape).astype(np.float32)
h = fs.handle(); fs._ensure_coeffs(h)
lib = N.load()
res = np.zeros(50)
for _ in range(3):
    N.check(lib.lesb_press(h.h, 50, 0, 1.7, N.dptr(res)), "press")
NST = 6
buf = np.zeros(200 * 100 * NST + 200 * 8, np.uint64)
fn = lib.lesb_debug_resident_trace
fn.restype = ctypes.c_longlong
n = fn(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_ulonglong)), buf.size)
nt = n // (100 * NST + 8)
t = buf[:nt * 100 * NST].reshape(nt, 100, NST).astype(np.int64)
t = t - t[:, 0, 0].min()
names = ["recv+barrier", "boundary", "barrier", "publish", "interior"]
d = [(t[:, :, q + 1] - t[:, :, q]) / 1e3 for q in range(NST - 1)]
gap = (t[:, 1:, 0] - t[:, :-1, NST - 1]) / 1e3
print("tiles", nt, "kernel span us", t[:, -1, NST - 1].max() / 1e3)
print("per-pass means over tiles/passes (us): " + "  ".join(
    "%s %.2f" % (nm, x[:, 2:].mean()) for nm, x in zip(names, d)) + "  end->next %.2f" % gap[:, 2:].mean())
per_pass = (t[:, 2:, 0].max(0)[1:] - t[:, 2:, 0].max(0)[:-1]) / 1e3
print("pass period (max start over tiles) us: mean %.2f min %.2f max %.2f" % (per_pass.mean(), per_pass.min(), per_pass.max()))
print("start skew across tiles at pass 50 (us): %.2f" % ((t[:, 50, 0].max() - t[:, 50, 0].min()) / 1e3))
comp = sum(d[1:])[:, 2:].mean(1)
order = np.argsort(comp)
print("per-tile work after receive (us): min %.2f median %.2f max %.2f" % (comp.min(), np.median(comp), comp.max()))
ext = buf[nt * 100 * NST: nt * 100 * NST + nt * 8].reshape(nt, 8).astype(np.int64)
if ext[:, 5].max() > 0:
    t00 = ext[:, 0].min()
    e = (ext[:, :8] - t00) / 1e3
    print("phases around the pass loop (us, mean over tiles): entry->loop %.2f  loop %.2f  write-back %.2f  "
          "grid sync %.2f  residuals %.2f  (kernel span %.2f)" % (
              (e[:, 1] - e[:, 0]).mean(), (e[:, 2] - e[:, 1]).mean(), (e[:, 3] - e[:, 2]).mean(),
              (e[:, 4] - e[:, 3]).mean(), (e[:, 5] - e[:, 4]).mean(), e[:, 5].max() - e[:, 0].min()))
    print("prologue (us, mean over tiles): tables + loads %.2f  initial publish %.2f  receive setup %.2f  "
          "(first tile entry -> last tile entry %.2f)" % ((e[:, 6] - e[:, 0]).mean(), (e[:, 7] - e[:, 6]).mean(),
                                                         (e[:, 1] - e[:, 7]).mean(), e[:, 0].max() - e[:, 0].min()))
