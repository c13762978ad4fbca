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
buf = np.zeros(200 * 100 * 4, np.uint64)
fn = lib.lesb_debug_resident_trace
fn.restype = ctypes.c_longlong
n = fn(buf.ctypes.data_as(ctypes.POINTER(ctypes.c_ulonglong)), buf.size)
nt = n // (100 * 4)
t = buf[:n].reshape(nt, 100, 4).astype(np.int64)
t0 = t[:, 0, 0].min()
t = t - t0
print("tiles", nt, "kernel span (first recv -> last interior end) us", (t[:, -1, 3].max()) / 1e3)
d_recv = (t[:, :, 1] - t[:, :, 0]) / 1e3
d_bnd = (t[:, :, 2] - t[:, :, 1]) / 1e3
d_int = (t[:, :, 3] - t[:, :, 2]) / 1e3
gap = (t[:, 1:, 0] - t[:, :-1, 3]) / 1e3
print("per-pass means over tiles/passes (us): recv+barrier %.2f  boundary %.2f  interior %.2f  end->next %.2f" %
      (d_recv[:, 2:].mean(), d_bnd[:, 2:].mean(), d_int[:, 2:].mean(), gap[:, 2:].mean()))
per_pass = (t[:, 2:, 0].max(0)[1:] - t[:, 2:, 0].max(0)[:-1]) / 1e3
print("pass period (max start over tiles) us: mean %.2f min %.2f max %.2f" % (per_pass.mean(), per_pass.min(), per_pass.max()))
print("tile 0 passes 10-14 (recv, bnd, int):", [(round(a, 2), round(b, 2), round(c, 2)) for a, b, c in zip(d_recv[0, 10:15], d_bnd[0, 10:15], d_int[0, 10:15])])
print("start skew across tiles at pass 50 (us): %.2f" % ((t[:, 50, 0].max() - t[:, 50, 0].min()) / 1e3))
comp = (d_bnd + d_int)[:, 2:].mean(1)
order = np.argsort(comp)
print("per-tile compute (bnd+int) us: min %.2f median %.2f max %.2f" % (comp.min(), np.median(comp), comp.max()))
print("slowest tiles:", [(int(t), round(float(comp[t]), 2)) for t in order[-6:]])
print("fastest tiles:", [(int(t), round(float(comp[t]), 2)) for t in order[:4]])
