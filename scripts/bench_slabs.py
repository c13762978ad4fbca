"""In-process x-slab step timing (SURVEY 8(e) streaming path): one domain vs
n slabs on one device with the streaming colour passes, the plane exchange
fused into the pass kernel (ghost planes) or a plane copy after every pass.

  python scripts/bench_slabs.py [IM JM KM] [--slabs 2] [--steps 16]

The slabs share one GPU here, so the number is the decomposition's overhead
(exchange, edge planes first, per-slab launches), not a multi-GPU speed-up.
Prints one JSON line; host-timed windows of synchronous steps (each step
ends with a host sync in both APIs)."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]

import golden_inputs as gi  # noqa: E402
import paper_1504_02264_b200 as P  # noqa: E402
from paper_1504_02264_b200.slabs import SlabGroup  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("dims", nargs="*", type=int, default=[600, 300, 90])
ap.add_argument("--slabs", type=int, default=2)
ap.add_argument("--steps", type=int, default=16)
a = ap.parse_args()
im, jm, km = a.dims
st = gi.config2_state(im, jm, km)
inflow = P.WindProfile(*gi.default_inflow(km))
P.runtime.set_sor_path(1)  # streaming passes on one domain too (the slabs' path)


def one_domain():
    g = P.Grid(im, jm, km, st["dx1"], st["dy1"], st["dzn"])
    fs = P.FlowState.create(g, dt=0.5, vn=0.8, cs=0.14)
    fs.mask[...] = st["mask"]
    for _ in range(2):
        P.les.step(fs, inflow)
    t0 = time.perf_counter()
    for _ in range(a.steps):
        P.les.step(fs, inflow)
    return (time.perf_counter() - t0) / a.steps


def slabs(env):
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        g = P.Grid(im, jm, km, st["dx1"], st["dy1"], st["dzn"])
        grp = SlabGroup(g, a.slabs, dt=0.5, vn=0.8, cs=0.14)
        grp.upload(st)
        for _ in range(2):
            grp.step(inflow)
        t0 = time.perf_counter()
        for _ in range(a.steps):
            grp.step(inflow)
        dt = (time.perf_counter() - t0) / a.steps
        grp.close()
        return dt
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


base = one_domain()
streams = slabs({"LESB_GROUP_PASSES": "1", "LESB_GHOST": "1", "LESB_GROUP_STREAMS": "1"})
serial = slabs({"LESB_GROUP_PASSES": "1", "LESB_GHOST": "1", "LESB_GROUP_STREAMS": "0"})
copies = slabs({"LESB_GROUP_PASSES": "1", "LESB_GHOST": "0"})
print(json.dumps({"grid": [im, jm, km], "slabs": a.slabs, "ms_per_step": {
    "one_domain": base * 1e3, "slabs_fused_exchange_own_streams": streams * 1e3,
    "slabs_fused_exchange_one_stream": serial * 1e3, "slabs_plane_copies_one_stream": copies * 1e3},
    "overhead_vs_one_domain": {"fused_own_streams": streams / base - 1, "fused_one_stream": serial / base - 1,
                               "copies_one_stream": copies / base - 1}}))
