"""Deterministic input builders shared by the golden generator and the tests.

Pure numpy, no reference import: the GPU box rebuilds exactly the inputs the
golden vectors were generated from.
"""

from __future__ import annotations

import zlib

import numpy as np

F32 = np.float32

# (tag, (im, jm, km), uniform spacing?)
STAGE_CASES = [
    ("s975", (9, 7, 5), True),
    ("s16", (16, 12, 10), True),
    ("s975nu", (9, 7, 5), False),
    ("s321", (3, 2, 1), True),
]
# (tag, (im, jm, km), h)
SOR_CASES = [
    ("r975", (9, 7, 5), 1.0),
    ("r886", (8, 8, 6), 2.0),
    ("r16", (16, 12, 10), 1.0),
    ("r111", (1, 1, 1), 1.0),
]
# (tag, (im, jm, km), n_steps)
STEP_CASES = [
    ("st975", (9, 7, 5), 10),
    ("st16tw", (16, 12, 10), 3),
    ("st24", (24, 10, 8), 10),
]
STEP_NITER = {"st975": 20, "st16tw": 15, "st24": 50}
STEP_SCHEME = {"st975": "redblack", "st16tw": "twinned", "st24": "redblack"}


def seed_of(tag: str) -> int:
    return zlib.crc32(tag.encode()) & 0x7FFFFFFF


def _spacing(n, rng, uniform, h=2.0):
    if uniform:
        return np.full(n, h, F32)
    return rng.uniform(1.0, 2.0, size=n).astype(F32)


def random_state(im, jm, km, seed, uniform=True, vel_scale=0.5):
    """Random u, v, w, p, fgh, fgh_old INCLUDING halos, a mask with a solid
    block and one fractional cell, and (optionally non-uniform) spacings."""
    rng = np.random.default_rng(seed)
    sh = (im + 2, jm + 2, km + 2)
    st = {"im": im, "jm": jm, "km": km, "dt": 0.5, "vn": 0.8, "cs": 0.14}
    for n in ("u", "v", "w"):
        st[n] = rng.uniform(-vel_scale, vel_scale, size=sh).astype(F32)
    st["p"] = rng.uniform(-1, 1, size=sh).astype(F32)
    st["fgh"] = rng.uniform(-1, 1, size=sh + (3,)).astype(F32)
    st["fgh_old"] = rng.uniform(-1, 1, size=sh + (3,)).astype(F32)
    m = np.zeros(sh, F32)
    i0, j0, k0 = max(1, im // 3), max(1, jm // 3), 1
    m[i0:i0 + max(1, im // 3), j0:j0 + max(1, jm // 3), k0:k0 + max(1, km // 2)] = 1.0
    m[im, jm, km] = 0.5
    st["mask"] = m
    st["dx1"] = _spacing(im + 3, rng, uniform)
    st["dy1"] = _spacing(jm + 2, rng, uniform)
    st["dzn"] = _spacing(km + 2, rng, uniform)
    return st


def random_inflow(km, seed):
    rng = np.random.default_rng(seed)
    return tuple(rng.uniform(-0.5, 1.0, size=km).astype(F32) for _ in range(3))


def sor_problem(im, jm, km, seed):
    """p0 with a random NON-ZERO halo (exercises the stored-halo policy) and rhs."""
    rng = np.random.default_rng(seed)
    sh = (im + 2, jm + 2, km + 2)
    p0 = rng.uniform(-1, 1, size=sh).astype(F32)
    rhs = rng.uniform(-1, 1, size=sh).astype(F32)
    return p0, rhs


def step_state(tag, im, jm, km):
    st = random_state(im, jm, km, seed=seed_of(tag), uniform=True, vel_scale=0.3)
    return st


def step_inflow(tag, km):
    return random_inflow(km, seed_of(tag) + 3)


def default_inflow(km, t_seconds=0.0):
    """driver.generate_profile with the CLI defaults (driver.py:44-57)."""
    import math

    z = 0.1 + 2.0 * np.arange(1, km + 1, dtype=np.float64)
    phase = 2.0 * math.pi * ((t_seconds % 600.0) / 600.0)
    gust = 1.0 + 0.2 * math.sin(phase)
    u = (0.05 / 0.41) * np.log(z / 0.1) * gust
    zeros = np.zeros(km, F32)
    return u.astype(F32), zeros, zeros.copy()


def zero_state(im, jm, km, h=2.0, dt=0.5, vn=0.8, cs=0.14):
    sh = (im + 2, jm + 2, km + 2)
    st = {"im": im, "jm": jm, "km": km, "dt": dt, "vn": vn, "cs": cs}
    for n in ("u", "v", "w", "p", "mask"):
        st[n] = np.zeros(sh, F32)
    st["fgh"] = np.zeros(sh + (3,), F32)
    st["fgh_old"] = np.zeros(sh + (3,), F32)
    st["dx1"] = np.full(im + 3, h, F32)
    st["dy1"] = np.full(jm + 2, h, F32)
    st["dzn"] = np.full(km + 2, h, F32)
    return st


def config1_state():
    st = zero_state(32, 32, 16)
    st["mask"][12:20, 12:20, 1:9] = 1.0
    return st


def config2_state(im=150, jm=150, km=90):
    """Config 2 (150x150x90, 3x3 buildings); other sizes scale the building
    layout to the grid (bench.py --grid)."""
    st = zero_state(im, jm, km)
    for bi in range(3):
        for bj in range(3):
            i0, j0 = (30 + 40 * bi) * im // 150, (30 + 40 * bj) * jm // 150
            h = (10 + 10 * ((bi + bj) % 3)) * km // 90
            st["mask"][i0:i0 + 16 * im // 150, j0:j0 + 16 * jm // 150, 1:1 + h] = 1.0
    return st
