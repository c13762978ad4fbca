"""The reference CLI's hot-path modes on the GPU:
``les-standalone`` (cli.py:202-219) and ``sor-bench`` (cli.py:222-283).

``dropin.install()`` puts ``run_les_standalone`` / ``run_sor_bench`` into
``gmcf_mini.cli._RUNNERS``, so ``python -m paper_1504_02264_b200 <mode>
--config ...`` (or the reference's own ``gmcf-mini`` after install()) runs
them with the reference's config parser, output directory and exit codes.
Inputs, files and summary keys are the reference's; what changes is where
the work runs and what sor-bench's scaling table measures:

* les-standalone keeps the flow on the device for all n_steps (one CUDA
  graph per step, one host sync at the end: ``les.run_steps``), then dumps
  u, v, w, p from the device state (``dump.write_state``).
* sor-bench: the red-black and twinned solves on the device, residual CSVs
  written from the device's float64 histories (the reference's ``%.17g``
  rows).  The reference's worker table (workers 1, 2, 4, .. on a CPU pool)
  is kept -- ``workers`` is accepted and ignored on the device, so the
  check it feeds, ``residuals_worker_invariant``, holds by construction --
  and a device table is added: the twinned and red-black solves on 1, 2, 4
  and 8 x-slabs (in one process the slabs share the device,
  under ``torchrun --nproc-per-node N`` one slab per GPU is added as the
  ``gpus=N`` row) with the GPU-count invariance check -- p bitwise equal to
  the 1-slab solve and the residual histories' largest relative deviation
  (the slabs' partial sums are added in slab order, so they agree to
  summation-order rounding, SURVEY 8(e) "residuals compare to rtol").
"""

from __future__ import annotations

import os
import time
from pathlib import Path

import numpy as np

from . import dump
from . import les as _les
from . import sor as _sor
from .reftypes import Grid, Scheme


def _scheme(cfg) -> Scheme:
    return Scheme.REDBLACK if cfg.sor_scheme == "redblack" else Scheme.TWINNED


def run_les_standalone(cfg, out_dir):
    """les-standalone (cli.py:202-219) with the flow resident on the GPU."""
    from gmcf_mini.cli import build_driver_config
    from gmcf_mini.driver import generate_profile

    grid = Grid.uniform(cfg.im, cfg.jm, cfg.km, cfg.h)
    flow = _les.FlowState.create(grid, dt=cfg.models[0][1], vn=cfg.vn, cs=cfg.cs)
    inflow = generate_profile(build_driver_config(cfg), 0.0)
    t0 = time.perf_counter()
    _les.run_steps(flow, inflow, cfg.n_steps, n_iter=cfg.sor_n_iter, scheme=_scheme(cfg))
    elapsed = time.perf_counter() - t0
    dump.write_state(flow, out_dir, ("u", "v", "w", "p"))
    summary = {
        "mode": "les-standalone",
        "steps": cfg.n_steps,
        "max_abs_u": float(np.abs(flow.u).max()),
        "timing": {"total_s": elapsed},
    }
    dump.write_json(Path(out_dir) / "summary.json", summary)
    return summary


def _residual_rows(res):
    return [(i, f"{r:.17g}") for i, r in enumerate(res)]


def _slab_counts(im: int, limit: int = 8):
    counts = [1]
    while counts[-1] * 2 <= min(limit, im):
        counts.append(counts[-1] * 2)
    return counts


def _slab_table(grid, p0, rhs, coeffs, omega_rb, omega_tw, n_iter, counts):
    """(rows, invariance) of the x-slab solves: rows (scheme, slabs,
    seconds); invariance per scheme vs the 1-slab solve."""
    from .slabs import SlabGroup

    rows, inv = [], {}
    for scheme, om in ((Scheme.REDBLACK, omega_rb), (Scheme.TWINNED, omega_tw)):
        base = None
        same_p, worst = True, 0.0
        for n in counts:
            grp = SlabGroup(grid, n, dt=1.0)
            try:
                grp.solve(p0, rhs, om, min(n_iter, 2), scheme)  # warm-up (graph-free: kernel and plan caches)
                t0 = time.perf_counter()
                p, res = grp.solve(p0, rhs, om, n_iter, scheme)
                rows.append((scheme.value, n, time.perf_counter() - t0))
            finally:
                grp.close()
            if base is None:
                base = (p, res)
                continue
            same_p = same_p and np.array_equal(p.view(np.uint32), base[0].view(np.uint32))
            den = np.maximum(np.abs(base[1]), 1e-300)
            worst = max(worst, float(np.max(np.abs(res - base[1]) / den)))
        inv[scheme.value] = {"p_bitwise": bool(same_p), "residuals_max_rel_diff": worst,
                             "residuals_within_rtol_1e-12": bool(worst <= 1e-12)}
    return rows, inv


def run_sor_bench(cfg, out_dir):
    """sor-bench (cli.py:222-283) on the GPU."""
    out_dir = Path(out_dir)
    grid = Grid.uniform(cfg.im, cfg.jm, cfg.km, cfg.h)
    coeffs = _sor.build_uniform_coeffs(grid)
    rng = np.random.default_rng(cfg.seed)
    rhs = _sor.make_field(cfg.im, cfg.jm, cfg.km)
    rhs[1:-1, 1:-1, 1:-1] = rng.uniform(-1, 1, size=(cfg.im, cfg.jm, cfg.km)).astype(np.float32)
    p0 = _sor.make_field(cfg.im, cfg.jm, cfg.km)
    omega_rb = cfg.sor_omega if cfg.sor_omega is not None else 1.7
    omega_tw = cfg.sor_omega if cfg.sor_omega is not None else 1.0

    times = []
    t0 = time.perf_counter()
    _, res_rb = _sor.solve_pressure(p0, rhs, coeffs, omega_rb, cfg.sor_n_iter, Scheme.REDBLACK)
    times.append(("redblack", 1, time.perf_counter() - t0))
    dump.write_csv(out_dir / "redblack_residuals.csv", "iteration,residual", _residual_rows(res_rb))

    counts = [1]
    while counts[-1] * 2 <= cfg.sor_workers:
        counts.append(counts[-1] * 2)
    res_tw_base = None
    bitwise_ok = True
    for w in counts:
        t0 = time.perf_counter()
        _, res_tw = _sor.solve_pressure(p0, rhs, coeffs, omega_tw, cfg.sor_n_iter, Scheme.TWINNED, workers=w)
        times.append(("twinned", w, time.perf_counter() - t0))
        if res_tw_base is None:
            res_tw_base = res_tw
            dump.write_csv(out_dir / "twinned_residuals.csv", "iteration,residual", _residual_rows(res_tw))
        else:
            bitwise_ok = bitwise_ok and np.array_equal(res_tw, res_tw_base)
    dump.write_csv(out_dir / "sor_bench_times.csv", "scheme,workers,seconds",
                   [(s, w, f"{t:.4f}") for s, w, t in times])
    for s, w, t in times:
        print(f"{s:9s} workers={w}: {t:.3f}s", flush=True)

    slabs = _slab_counts(cfg.im)
    rows, inv = _slab_table(grid, p0, rhs, coeffs, omega_rb, omega_tw, cfg.sor_n_iter, slabs)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1:
        rows += _distributed_rows(grid, p0, rhs, omega_rb, omega_tw, cfg.sor_n_iter, inv)
    dump.write_csv(out_dir / "sor_bench_gpu_times.csv", "scheme,slabs,seconds",
                   [(s, n, f"{t:.6f}") for s, n, t in rows])
    for s, n, t in rows:
        print(f"{s:9s} x-slabs={n}: {t * 1e3:.3f} ms", flush=True)
    tw_times = {w: t for s, w, t in times if s == "twinned"}
    summary = {
        "mode": "sor-bench",
        "domain": [cfg.im, cfg.jm, cfg.km],
        "n_iter": cfg.sor_n_iter,
        "worker_counts": counts,
        "residuals_worker_invariant": bool(bitwise_ok),
        "speedup_vs_1": {str(w): tw_times[1] / tw_times[w] for w in counts},
        "timing": {"table": [(s, w, t) for s, w, t in times]},
        "device": {
            "slab_counts": slabs,
            "table": [(s, n, t) for s, n, t in rows],
            "gpu_count_invariance": inv,
            "note": "x-slabs (SURVEY 8(e)); in one process the slabs share one device",
        },
    }
    dump.write_json(out_dir / "summary.json", summary)
    return summary


def _distributed_rows(grid, p0, rhs, omega_rb, omega_tw, n_iter, inv):
    """Under torchrun: one x-slab per GPU (SlabDomain, NCCL), timed and
    checked against the 1-slab solve; every rank runs this, rank 0 reports."""
    import torch
    import torch.distributed as dist

    from .slabs import SlabDomain, slice_global

    local = int(os.environ.get("LOCAL_RANK", "0"))
    if not dist.is_initialized():
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    world = dist.get_world_size()
    rows = []
    dom = SlabDomain(grid, dt=1.0, device=local)
    try:
        for scheme, om in ((Scheme.REDBLACK, omega_rb), (Scheme.TWINNED, omega_tw)):
            ref_p, ref_res = _sor.solve_pressure(p0, rhs, _sor.build_uniform_coeffs(grid), om, n_iter, scheme)
            dom.solve(p0, rhs, om, min(n_iter, 2), scheme)
            dist.barrier()
            t0 = time.perf_counter()
            p, res = dom.solve(p0, rhs, om, n_iter, scheme)
            dist.barrier()
            rows.append((scheme.value, f"gpus={world}", time.perf_counter() - t0))
            mine = slice_global(ref_p, dom.slab.i0, dom.slab.i1)
            ok = torch.tensor([int(np.array_equal(p[1:-1].view(np.uint32), mine[1:-1].view(np.uint32)))],
                              device="cuda")
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            den = np.maximum(np.abs(ref_res), 1e-300)
            inv[f"{scheme.value}@gpus={world}"] = {
                "p_bitwise": bool(ok.item()),
                "residuals_max_rel_diff": float(np.max(np.abs(res - ref_res) / den)),
            }
    finally:
        dom.close()
    return rows
