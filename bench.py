"""Benchmark: DPRI-LES time steps/s on B200 (BASELINE.json metric).

Workload (BASELINE.json configs[1]): 150x150x90 grid,
h = 2, dt = 0.5, vn = 0.8, cs = 0.14, the 3x3 synthetic building array,
WRF-style log-law inflow, red-black SOR with 50 iterations (les.step
defaults).  Synthetic data.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

Arms
  (default)    the CUDA path.  `value` = steps/s with the state resident in
               HBM, each step one CUDA-graph replay timed with CUDA events on
               the domain stream, L2 flushed (256 MB write) before every
               timed step.  The reference dynamics blow up at step 19 with
               buildings, so the state is re-initialised
               (untimed device copy) every 16 steps; kernel cost is
               data-independent.
               `e2e` = the same steps through the public Python API
               (les.step on a FlowState), timed on the host clock over
               back-to-back 16-step windows (the longest that stays below
               the blow-up), each uploading the initial state from pinned
               host memory, running 16 steps (inflow H2D, stage flags +
               residual history D2H per step) and downloading the six fields
               to pinned host memory; the window copies run on their own
               streams under the steps (FlowState.stage / download_async).
               `e2e.serial_value`: the same with synchronous copies.
  reference    the reference on the host CPU: the unmodified gmcf_mini.les.step
               from baseline/_ref (scripts/install_reference.sh; the numpy
               port in oracle/ only when that is absent), a bounded sample
               of full-size config-2 steps on 1 core (the reference's
               red-black path is single-threaded numpy).

Multi-GPU (N > 1; `--gpus N` re-launches itself under torch.distributed.run
when WORLD_SIZE is unset): x-slab decomposition -- each
rank owns a 150x150x90 slab of a (150 N)x150x90 grid ("scaling": "weak"),
halo planes move by NCCL send/recv inside the step's CUDA graph; value
counts slab-steps over all ranks divided by the max-over-ranks time.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

METRIC = "LES time steps/sec and MLUPS at 1/2/4/8 B200; % of HBM-bandwidth roofline"
IM, JM, KM = 150, 150, 90
N_ITER = 50
REINIT = 16  # steps per state window (config 2 blows up at step 19)
E2E_MIN_WINDOWS = 8  # e2e: at least 8 windows (128 steps), so the exposed first upload / last download amortise
B_ITER = 12                     # SOR RB iteration, cn1 a scalar: p read + p write + rhs read
B_STEP = 216 + B_ITER * N_ITER  # algorithmic bytes / interior cell / step: 816 (SURVEY 8(d), cn1 scalarised)
WORKLOAD = "config2: 150x150x90, h=2, dt=0.5, 3x3 buildings, log-law inflow, RB SOR 50 iters"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    """SM clock and throttle reasons sampled DURING the timed region.

    NVML is polled every ~2 ms from a thread (a timed region of a few tens of
    ms still gets samples); nvidia-smi -lms 100 is the fallback when NVML is
    unavailable.  Only samples taken between __enter__ and __exit__ count."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []
        self.samples: list[tuple[float, float, int]] = []  # (sm MHz, max MHz, reason bits)
        self.nvml = None
        self.stop = threading.Event()
        self.t = None

    def _nvml_handle(self):
        import pynvml
        import torch
        pynvml.nvmlInit()
        try:
            p = torch.cuda.get_device_properties(self.device)
            bus = f"{p.pci_domain_id:08X}:{p.pci_bus_id:02X}:{p.pci_device_id:02X}.0"
            h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:  # noqa: BLE001
            h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
        return pynvml, h

    def _poll_nvml(self):
        nv, h = self.nvml
        bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
        self.bits = bits
        mx = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
        while not self.stop.is_set():
            try:
                sm = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                r = int(nv.nvmlDeviceGetCurrentClocksEventReasons(h))
                self.samples.append((sm, mx, r))
            except Exception:  # noqa: BLE001
                break
            time.sleep(0.002)

    def __enter__(self):
        try:
            self.nvml = self._nvml_handle()
            self.t = threading.Thread(target=self._poll_nvml, daemon=True)
            self.t.start()
            return self
        except Exception:  # noqa: BLE001
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:  # noqa: BLE001
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        self.stop.set()
        if self.nvml is not None and self.t is not None:
            self.t.join(timeout=2)
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:  # noqa: BLE001
                self.proc.kill()

    def summary(self):
        if self.nvml is not None and self.samples:
            sm = [x[0] for x in self.samples]
            reasons = sorted({nm for _, _, r in self.samples for nm, b in self.bits.items() if r & b})
            return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.samples[0][1], "reasons": reasons,
                    "samples": len(sm), "source": "nvml, 2 ms poll"}
        sm, mx, reasons = [], None, set()
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for nm, val in zip(self.NAMES, parts[3:7]):
                if val.lower() == "active":
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvidia-smi -lms 100"}


# ---------------------------------------------------------------------------
# CPU reference arm and CPU baseline: the unmodified reference (gmcf_mini,
# installed under baseline/_ref by scripts/install_reference.sh) when it is
# importable, else the numpy port in oracle/ (pinned bitwise to it)
# ---------------------------------------------------------------------------
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def cpu_info():
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_count": os.cpu_count(), "cpu_model": model}


def _reference_les():
    """gmcf_mini.les from baseline/_ref (or None).  The reference's own
    module-level step, never rebound here (install() is not called)."""
    if os.path.isdir(os.path.join(REF_DIR, "gmcf_mini")) and REF_DIR not in sys.path:
        sys.path.append(REF_DIR)
    try:
        import gmcf_mini.coupling as rc
        import gmcf_mini.les as rl
        import gmcf_mini.sor as rs
    except ImportError:
        return None
    if rl.step.__module__ != "gmcf_mini.les":
        raise RuntimeError("gmcf_mini.les.step is rebound (drop-in installed): not the reference")
    return rl, rs, rc


def cpu_sample(max_steps: int, budget_s: float):
    """Time full-size config-2 steps of the reference on one host core:
    returns (steps/s, steps timed, seconds, kind).  kind "reference" = the
    unmodified gmcf_mini.les.step (les.py:393-416), "port" = oracle/."""
    import golden_inputs as gi

    st = gi.config2_state(IM, JM, KM)
    inflow = gi.default_inflow(KM)  # == driver.generate_profile at the CLI defaults (tests/golden_inputs.py)
    ref = _reference_les()
    if ref is not None:
        rl, rs, rc = ref
        flow = rl.FlowState.create(rs.Grid.uniform(IM, JM, KM, 2.0), dt=0.5, vn=0.8, cs=0.14)
        flow.mask[...] = st["mask"]
        prof = rc.WindProfile(*inflow)
        kind = "reference"

        def one():
            rl.step(flow, prof, n_iter=N_ITER)
    else:
        from oracle import les_oracle as O

        o = O.OState.zeros(IM, JM, KM)
        for n in ("u", "v", "w", "fgh", "fgh_old", "p", "mask", "dx1", "dy1", "dzn"):
            getattr(o, n)[...] = st[n]
        kind = "port"

        def one():
            O.step(o, *inflow, n_iter=N_ITER)
    done = 0
    t0 = time.perf_counter()
    while done < max_steps:
        one()
        done += 1
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    return done / dt, done, dt, kind


def cpu_desc(n, secs, kind):
    what = ("the unmodified reference gmcf_mini.les.step (baseline/_ref)" if kind == "reference"
            else "the numpy port oracle/les_oracle.py (reference not importable)")
    return (f"{n} full {IM}x{JM}x{KM} RB50 config-2 steps of {what} in {secs:.1f}s, from a fresh state; "
            f"1 thread (the reference's red-black path is single-threaded numpy)")


def config_dict(world: int) -> dict:
    """The workload -- identical in both arms."""
    return {"workload": WORKLOAD, "grid": [IM, JM, KM], "n_iter": N_ITER, "scheme": "redblack",
            "global_grid": [IM * world, JM, KM],
            "parallelism": (f"x-slabs over {world} GPUs, {IM}x{JM}x{KM} per GPU" if world > 1 else "1 GPU"),
            "l2": "GPU arm: flushed before every timed step (256 MB device write, untimed)"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    if rank != 0:
        return
    for _ in range(min(args.warmup, 1)):
        cpu_sample(1, 0)
    rate, n, secs, kind = cpu_sample(max(1, args.steps), 90.0)
    sample = cpu_desc(n, secs, kind)
    line = {
        "impl": "reference", "metric": METRIC, "value": rate, "unit": "steps/s", "n_gpus": world,
        "steps": n, "warmup": min(args.warmup, 1), "ms_per_step": 1000.0 / rate, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_dict(world),
        "mlups": rate * IM * JM * KM / 1e6,
        "cpu_baseline": {"value": rate, "unit": "steps/s", "cores": 1, "kind": kind, "sample": sample,
                         **cpu_info()},
        "e2e": {"value": rate, "unit": "steps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# CUDA arm
# ---------------------------------------------------------------------------
def run_gpu(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    multi = world > 1 or args.slabs  # x-slab path (--slabs: on one rank, under torch.distributed.run)
    if multi:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)

    import golden_inputs as gi
    import paper_1504_02264_b200 as P
    from paper_1504_02264_b200 import _native as N

    P.runtime.set_device(local)
    lib = N.load()
    st0 = gi.config2_state(IM, JM, KM)
    inflow = P.WindProfile(*gi.default_inflow(KM))
    slab_dom = None
    if not multi:
        grid = P.Grid(IM, JM, KM, st0["dx1"], st0["dy1"], st0["dzn"])

        def make_state():
            fs = P.FlowState.create(grid, dt=0.5, vn=0.8, cs=0.14)
            fs.mask[...] = st0["mask"]
            return fs

        pristine = make_state()
        hp = pristine.handle()
        pristine._ensure_coeffs(hp)
        work = make_state()
        hw = work.handle()
        work._ensure_coeffs(hw)
    else:
        # x-slabs: every rank owns a 150x150x90 slab of a (150 N)x150x90 grid
        # with the 3x3 building array repeated per slab; halo planes move by
        # NCCL send/recv inside the step graph
        from paper_1504_02264_b200.slabs import SlabDomain, _Slab

        grid = P.Grid.uniform(IM * world, JM, KM, 2.0)
        gstate = gi.zero_state(IM * world, JM, KM)
        for r in range(world):
            gstate["mask"][1 + r * IM:1 + (r + 1) * IM] = st0["mask"][1:IM + 1]
        slab_dom = SlabDomain(grid, dt=0.5, vn=0.8, cs=0.14, device=local)
        slab_dom.upload(gstate)
        i0, i1 = slab_dom.bounds[rank]
        pristine = _Slab(grid, 0.5, 0.8, 0.14, i0, i1, local)
        for name in ("u", "v", "w", "fgh", "fgh_old", "p", "mask"):
            pristine.upload(name, gstate[name])

        class _H:
            def __init__(self, h):
                self.h = h

        hw, hp = _H(slab_dom.slab.h), _H(pristine.h)
    arrs = [N.f32c(getattr(inflow, c)) for c in ("u", "v", "w")]
    N.check(lib.lesb_set_inflow(hw.h, *[N.fptr(a) for a in arrs]), "set_inflow")
    # the timed steps replay the plain step graph; the phase split comes from
    # a separate, shorter run of the graph variant with event records between
    # the phases (instrumentation, not part of the measured steps)
    N.check(lib.lesb_set_timing(hw.h, 0), "set_timing")
    stream = torch.cuda.ExternalStream(lib.lesb_stream(hw.h))
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def reinit():
        N.check(lib.lesb_copy_state(hw.h, hp.h), "copy_state")

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)]
    phase_ms = np.zeros(4)
    since = 0
    reinit()
    # warm-up
    for _ in range(args.warmup):
        if since == REINIT:
            reinit()
            since = 0
        N.check(lib.lesb_step_async(hw.h, N_ITER, 0, 1.7), "step")
        since += 1
    torch.cuda.synchronize()
    # (after the warm-up: an x-slab maps its neighbours' buffers at its first
    # solve, which decides the solver path)
    kps = lib.lesb_kernels_per_step(hw.h, N_ITER, 0)  # asynchronous step, bookkeeping included
    sor_path = {1: "streaming colour passes, colour-split layout", 2: "shared-memory-resident persistent kernel",
                3: "streaming colour passes, natural layout"}[
        lib.lesb_sor_path_in_use(hw.h, 0)]
    if multi:
        dist.barrier()
    torch.cuda.synchronize()
    t_wall = time.perf_counter()
    with ClockSampler(local) as clk:
        for s in range(args.steps):
            if since == REINIT:
                reinit()
                since = 0
            with torch.cuda.stream(stream):
                flush.fill_(float(s))
                ev[s][0].record(stream)
            N.check(lib.lesb_step_async(hw.h, N_ITER, 0, 1.7), "step")
            with torch.cuda.stream(stream):
                ev[s][1].record(stream)
            since += 1
        torch.cuda.synchronize()
    wall = time.perf_counter() - t_wall
    # phase split: the instrumented graph, L2 flushed before each step as above
    N.check(lib.lesb_set_timing(hw.h, 1), "set_timing")
    n_ph = min(args.steps, 10)
    for s in range(n_ph + 1):
        if since == REINIT:
            reinit()
            since = 0
        with torch.cuda.stream(stream):
            flush.fill_(float(s))
        N.check(lib.lesb_step_async(hw.h, N_ITER, 0, 1.7), "step")
        since += 1
        if s > 0:  # (the first replay builds the instrumented graph)
            ph = np.zeros(4, np.float32)
            N.check(lib.lesb_last_step_times(hw.h, N.fptr(ph)), "times")
            phase_ms += ph
    torch.cuda.synchronize()
    N.check(lib.lesb_set_timing(hw.h, 0), "set_timing")
    if multi:
        dist.barrier()
    torch.cuda.synchronize()
    done = N.C.c_int(0)
    fstep = N.C.c_int(-1)
    fstage = N.C.c_int(-1)
    N.check(lib.lesb_poll_failure(hw.h, N.C.byref(done), N.C.byref(fstep), N.C.byref(fstage)), "poll")
    if fstep.value >= 0:
        raise RuntimeError(f"benchmark state went non-finite at step {fstep.value} ({fstage.value})")
    step_ms = [a.elapsed_time(b) for a, b in ev]
    dev_ms = float(sum(step_ms))
    if multi:
        t = torch.tensor([dev_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_ms = float(t.item())
    ms_per_step = dev_ms / args.steps
    value = world * args.steps / (dev_ms / 1000.0)  # slab-steps over all ranks / max time
    n_int = IM * JM * KM
    hbm, peak_kind = peaks()
    phase_ms /= n_ph
    # dominant kernel: the SOR solve (phase 2 = the solver launches between the
    # step's fused kernel and the press halo).  Algorithmic bytes: 12 B per
    # interior cell and iteration (SURVEY 8(d), cn1 scalar) x N x n_iter.
    sor_ms = phase_ms[2]
    b_solve = B_ITER * n_int * N_ITER
    achieved = b_solve / (sor_ms * 1e-3) / 1e9
    step_gbs = B_STEP * n_int / (ms_per_step * 1e-3) / 1e9
    sor_kernel = {2: "k_sor_resident", 1: "k_sor_rbt", 3: "k_sor_rb"}[lib.lesb_sor_path_in_use(hw.h, 0)]
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            traffic = json.load(f).get(f"{sor_kernel}@{IM}x{JM}x{KM}")
    except Exception:  # noqa: BLE001
        traffic = None

    # ---- e2e through the public API ----
    if args.no_e2e:
        e2e = {"value": None, "seconds": 0.0, "h2d": 0, "d2h": 0}
    elif slab_dom is None:
        e2e = e2e_run(P, N, gi, torch, grid, st0, inflow, args)
    else:
        e2e = e2e_slabs(slab_dom, gstate, inflow, torch, args, world)
    if multi and e2e["value"] is not None:
        t = torch.tensor([e2e["seconds"]], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e["value"] *= e2e["seconds"] / float(t.item())
        e2e["seconds"] = float(t.item())
        if "serial_seconds" in e2e:
            t = torch.tensor([e2e["serial_seconds"]], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e["serial_value"] *= e2e["serial_seconds"] / float(t.item())

    cpu = None
    if rank == 0 and not args.no_cpu:
        rate, n, secs, kind = cpu_sample(3, 20.0)
        cpu = {"value": rate, "unit": "steps/s", "cores": 1, "kind": kind, "sample": cpu_desc(n, secs, kind),
               **cpu_info()}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "steps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": config_dict(world),
            "method": {"reinit_every_steps": REINIT,
                       "timing": "CUDA events on the domain stream around each CUDA-graph step replay",
                       "sor_kernel": sor_path,
                       "exchange": "NCCL halo planes inside the step graph" if multi else None},
            "mlups": value * n_int / 1e6,
            "step_roofline": {"bytes_per_cell": B_STEP, "achieved_gbs": step_gbs, "peak_gbs": hbm,
                              "frac": step_gbs / hbm, "peak_kind": peak_kind},
            "phase_ms": {"velnw_bondv1": phase_ms[0], "velfg_feedbf_les_adam_rhs": phase_ms[1],
                         "sor_passes": phase_ms[2], "halo_and_residuals": phase_ms[3]},
            "roofline": {"kernel": (f"{sor_kernel} (whole {N_ITER}-iteration red-black solve, one launch)"
                                   if sor_kernel == "k_sor_resident" else
                                   f"{sor_kernel} ({2 * N_ITER} colour-pass launches with the layout pack / unpack "
                                   "and the residual reduction: the solve phase of the step)"),
                         "bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                         "traffic": traffic, "peak_kind": peak_kind,
                         "algorithmic_bytes_per_launch": b_solve, "bytes_per_cell_iteration": B_ITER,
                         "launch_ms": sor_ms,
                         "note": "working set (p, rhs: 17 MB) is L2/shared-memory resident at this size; "
                                 "the HBM-bound evidence is the 512x512x90 press-only line (DESIGN.md)"},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e["value"], "unit": "steps/s", "h2d_bytes_per_step": e2e["h2d"],
                    "d2h_bytes_per_step": e2e["d2h"],
                    **{k: e2e[k] for k in ("windows", "serial_value") if k in e2e}},
            "gpu_launches": kps * args.steps,
            "clocks": clk.summary(),
            "wall_s": wall,
        }
        if not multi and not args.grid and not args.no_extras:
            line["extras"] = side_lines()
        print(json.dumps(line), flush=True)
    if multi:
        dist.destroy_process_group()


def _last_json(cmd, timeout):
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=timeout)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    if r.returncode != 0 or not lines:
        raise RuntimeError(f"exit {r.returncode}: {(r.stderr or r.stdout)[-300:]}")
    return json.loads(lines[-1])


def side_lines():
    """The other BASELINE.json configurations that fit one GPU, measured after
    the headline run by the same tools the profiles use, so that they land in
    the driver's record: config 3 (press-only red-black solve, 512x512x90, the
    HBM-bound case) and the 300x300x90 step (the per-GPU size of the weak
    scaling runs).  Each in its own process; a failure is recorded, not raised."""
    out = {}
    try:
        d = _last_json([sys.executable, os.path.join(ROOT, "scripts", "bench_press.py"), "512", "512", "90",
                        "--path", "1", "--reps", "5"], 300)
        out["config3_press_only_512x512x90"] = {
            "kernel": d.get("sor_kernel"), "us_per_iteration": d["us_per_iteration"],
            "roofline_frac_12B": d["roofline"]["frac"], "achieved_gbs": d["roofline"]["achieved_gbs"],
            "halo": "stored", "n_iter": 50, "timing": "median of 5 device-timed solves, inputs resident"}
    except Exception as e:  # noqa: BLE001
        out["config3_press_only_512x512x90"] = {"error": str(e)[:300]}
    try:
        d = _last_json([sys.executable, os.path.abspath(__file__), "--grid", "300", "300", "90", "--steps", "20",
                        "--warmup", "5", "--no-cpu", "--no-e2e", "--no-extras"], 300)
        out["step_300x300x90"] = {"steps_per_s": d["value"], "ms_per_step": d["ms_per_step"],
                                  "step_roofline_frac": d["step_roofline"]["frac"],
                                  "sor_kernel": d["roofline"]["kernel"], "sor_roofline_frac": d["roofline"]["frac"],
                                  "clocks": d.get("clocks")}
    except Exception as e:  # noqa: BLE001
        out["step_300x300x90"] = {"error": str(e)[:300]}
    return out


def e2e_run(P, N, gi, torch, grid, st0, inflow, args):
    """Public-API steps with host buffers, timed on the host clock: windows of
    REINIT steps, each starting from the initial state copied from pinned host
    memory (FlowState.stage / commit_staged) and ending with the six fields
    copied to pinned host memory (FlowState.download_async); every step also
    copies its inflow in and its stage flags and residual history out
    (les.step).  The next window's upload is started after the window's first
    step and the window's download runs during the next window, so the copies
    overlap the steps; the first upload and the last download are exposed.
    `serial_value` is the same windows with synchronous copies (assignment,
    attribute reads) between them."""
    names = ("u", "v", "w", "fgh", "fgh_old", "p", "mask")
    pinned = lambda n: torch.empty(st0[n].shape, dtype=torch.float32, pin_memory=True).numpy()  # noqa: E731
    ins = {n: pinned(n) for n in names}
    for n in names:
        ins[n][...] = st0[n]
    outs = [{n: pinned(n) for n in names[:6]} for _ in range(2)]
    fs = P.FlowState.create(grid, dt=0.5, vn=0.8, cs=0.14)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def pipelined(n_windows):
        pend = [None, None]
        fs.stage(**ins)
        for w in range(n_windows):
            fs.commit_staged()
            P.les.step(fs, inflow)
            if w + 1 < n_windows:
                fs.stage(**ins)                # next window's initial state, during this window
            for _s in range(REINIT - 1):
                P.les.step(fs, inflow)
            b = w % 2
            if pend[b] is not None:
                pend[b].wait()                 # (window w-2's download: long done)
            pend[b] = fs.download_async(outs[b])
        for p in pend:
            if p is not None:
                p.wait()

    work = {n: pinned(n) for n in names}

    def serial():
        for n in names:
            setattr(fs, n, work[n])            # host arrays -> uploaded before the first step
        for _s in range(REINIT):
            P.les.step(fs, inflow)
        for n in names[:6]:
            getattr(fs, n)                     # device -> host (into work[n])

    def timed(fn, *a):
        flush.fill_(1.0)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn(*a)
        return time.perf_counter() - t0

    pipelined(1)                               # warm-up: graph capture
    n_windows = max(E2E_MIN_WINDOWS, -(-args.steps // REINIT))
    secs = timed(pipelined, n_windows)
    s_windows = max(1, args.steps // REINIT)
    s_secs = 0.0
    for _ in range(s_windows):
        for n in names:
            work[n][...] = st0[n]
        s_secs += timed(serial)
    h2d = sum(ins[n].nbytes for n in names) / REINIT + 3 * KM * 4
    d2h = sum(ins[n].nbytes for n in names[:6]) / REINIT + 4 + 8 * N_ITER
    return {"value": n_windows * REINIT / secs, "seconds": secs, "h2d": int(h2d), "d2h": int(d2h),
            "windows": n_windows, "serial_value": s_windows * REINIT / s_secs}


def e2e_slabs(dom, gstate, inflow, torch, args, world):
    """Public slab API with host buffers, e2e_run's windows on every rank:
    the rank's part of the initial state staged from pinned host memory
    during the previous window (SlabDomain.stage / commit_staged), its slab
    fields downloaded to pinned host memory during the next
    (SlabDomain.download_async); `serial_value`: upload / steps / download in
    sequence."""
    names = ("u", "v", "w", "fgh", "fgh_old", "p", "mask")
    ins = {}
    for n in names:
        ins[n] = torch.empty(gstate[n].shape, dtype=torch.float32, pin_memory=True).numpy()
        ins[n][...] = gstate[n]
    outs = [{n: torch.empty(dom.slab_shape(n), dtype=torch.float32, pin_memory=True).numpy() for n in names[:6]}
            for _ in range(2)]

    def pipelined(n_windows):
        pend = [None, None]
        dom.stage(ins)
        for w in range(n_windows):
            dom.commit_staged()
            dom.step(inflow)
            if w + 1 < n_windows:
                dom.stage(ins)
            for _s in range(REINIT - 1):
                dom.step(inflow)
            b = w % 2
            if pend[b] is not None:
                pend[b].wait()
            pend[b] = dom.download_async(outs[b])
        for p in pend:
            if p is not None:
                p.wait()

    def serial():
        dom.upload(gstate)
        for _s in range(REINIT):
            dom.step(inflow)
        for n in names[:6]:
            dom.slab.download(n, JM, KM)

    def timed(fn, *a):
        torch.cuda.synchronize()
        dom.dist.barrier()
        t0 = time.perf_counter()
        fn(*a)
        return time.perf_counter() - t0

    pipelined(1)
    n_windows = max(E2E_MIN_WINDOWS, -(-args.steps // REINIT))
    secs = timed(pipelined, n_windows)
    s_windows = max(1, args.steps // REINIT)
    s_secs = sum(timed(serial) for _ in range(s_windows))
    slab_bytes = {n: 4 * int(np.prod(dom.slab_shape(n))) for n in names}  # the rank's part, halo planes included
    h2d = sum(slab_bytes.values()) / REINIT + 3 * KM * 4
    d2h = sum(slab_bytes[n] for n in names[:6]) / REINIT + 4
    return {"value": world * n_windows * REINIT / secs, "seconds": secs, "h2d": int(h2d), "d2h": int(d2h),
            "windows": n_windows, "serial_value": world * s_windows * REINIT / s_secs, "serial_seconds": s_secs}


def main():
    global IM, JM, KM, WORKLOAD
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="cuda", choices=["cuda", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline sample")
    ap.add_argument("--no-e2e", action="store_true", help="skip the e2e measurement (profiling runs)")
    ap.add_argument("--slabs", action="store_true",
                    help="the x-slab (N-GPU) path even on one rank (launch under torch.distributed.run)")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the side lines (config 3 press-only at 512^2, the 300^2 step) measured after the run")
    ap.add_argument("--grid", type=int, nargs=3, metavar=("IM", "JM", "KM"),
                    help="another grid (per GPU) with config 2's buildings scaled to it; default config 2")
    args = ap.parse_args()
    if args.grid and tuple(args.grid) != (IM, JM, KM):
        IM, JM, KM = args.grid
        WORKLOAD = (f"config2 layout scaled to {IM}x{JM}x{KM}, h=2, dt=0.5, 3x3 buildings, log-law inflow, "
                    f"RB SOR 50 iters")
    if args.warmup < 3 and args.impl == "cuda":
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torchrun (the driver launches it
        # that way itself; a plain `python bench.py --gpus N` does the same)
        import socket

        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
