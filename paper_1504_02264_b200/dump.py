"""GMCF field dumps straight from the device state.

Format (the reference's, dump.py:1-39): the 4 bytes ``GMCF``, the three
dimensions as little-endian uint32, then the field as row-major
little-endian float32; written to a temporary name and renamed, so a failed
run leaves the complete file or nothing.  ``write_state`` downloads each field
once (pitched D2H of the Python-visible array) and writes it; the files are
byte-identical to the reference's ``dump.write_field`` of the same array.
"""

from __future__ import annotations

import os
from pathlib import Path

import numpy as np

MAGIC = b"GMCF"


def _atomic(path: Path, chunks) -> None:
    tmp = path.with_name(path.name + ".tmp")
    with open(tmp, "wb") as f:
        for c in chunks:
            f.write(c)
    os.replace(tmp, path)


def write_field(path, arr: np.ndarray) -> None:
    path = Path(path)
    if arr.ndim != 3:
        raise ValueError(f"field dumps are 3-D, got shape {arr.shape}")
    head = MAGIC + np.asarray(arr.shape, dtype="<u4").tobytes()
    body = np.ascontiguousarray(arr, dtype="<f4")
    _atomic(path, (head, memoryview(body).cast("B")))


def write_json(path, obj) -> None:
    """JSON summary, indent 2 and a trailing newline, written atomically
    (dump.py:54-56)."""
    import json

    _atomic(Path(path), ((json.dumps(obj, indent=2) + "\n").encode(),))


def write_sidecar(path, entries: dict) -> None:
    """``key = value`` lines (dump.py:42-44)."""
    lines = [f"{k} = {v}" for k, v in entries.items()]
    _atomic(Path(path), (("\n".join(lines) + "\n").encode(),))


def write_csv(path, header: str, rows) -> None:
    """Comma-separated rows under a header line (dump.py:47-51): sor-bench's
    residual histories (``iteration,residual`` with ``%.17g`` values, as the
    device returns them) and timing tables."""
    lines = [header]
    lines.extend(",".join(str(c) for c in row) for row in rows)
    _atomic(Path(path), (("\n".join(lines) + "\n").encode(),))


def read_field(path) -> np.ndarray:
    raw = Path(path).read_bytes()
    if raw[:4] != MAGIC:
        raise ValueError(f"{path}: bad magic {raw[:4]!r}")
    dims = tuple(int(d) for d in np.frombuffer(raw[4:16], dtype="<u4"))
    data = np.frombuffer(raw[16:], dtype="<f4")
    if data.size != int(np.prod(dims)):
        raise ValueError(f"{path}: payload size {data.size} != dims {dims}")
    return data.reshape(dims).copy()


def write_state(state, out_dir, names=("u", "v", "w", "p")) -> list:
    """Dump fields of a (device) FlowState as ``<name>.gmcf`` files, as the
    reference's les-standalone and coupled modes do (cli.py:187-198, 210-211)."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    paths = []
    for n in names:
        p = out / f"{n}.gmcf"
        write_field(p, getattr(state, n))
        paths.append(p)
    return paths


# Checkpoint / resume (the reference has final dumps only).  A step
# reads u, v, w, p, fgh, fgh_old and the mask; the GMCF format is 3-D, so the
# two force fields are stored per component (``fgh.0.gmcf`` ...).
CHECKPOINT_FIELDS = ("u", "v", "w", "p", "mask", "fgh", "fgh_old")
_VECTOR_FIELDS = ("fgh", "fgh_old")


def write_checkpoint(state, out_dir) -> list:
    """Everything ``les.step`` reads from ``state`` as GMCF dumps plus a
    sidecar listing them; ``read_checkpoint`` restores it and the run then
    continues bitwise as if it had not stopped (tests/test_gpu_cli.py)."""
    out = Path(out_dir)
    out.mkdir(parents=True, exist_ok=True)
    paths, entries = [], {}
    for n in CHECKPOINT_FIELDS:
        arr = np.asarray(getattr(state, n))
        if n in _VECTOR_FIELDS:
            for m in range(arr.shape[-1]):
                p = out / f"{n}.{m}.gmcf"
                write_field(p, np.ascontiguousarray(arr[..., m]))
                paths.append(p)
                entries[f"{n}.{m}"] = p.name
        else:
            p = out / f"{n}.gmcf"
            write_field(p, arr)
            paths.append(p)
            entries[n] = p.name
    write_sidecar(out / "checkpoint.txt", entries)
    return paths


def read_checkpoint(state, in_dir) -> None:
    """Load ``write_checkpoint``'s files into ``state`` (a FlowState of the same
    grid: the shapes are checked); on the device state each field is uploaded
    at the next step."""
    src = Path(in_dir)
    g = state.grid
    shape = (g.im + 2, g.jm + 2, g.km + 2)
    for n in CHECKPOINT_FIELDS:
        if n in _VECTOR_FIELDS:
            comps = [read_field(src / f"{n}.{m}.gmcf") for m in range(3)]
            for c in comps:
                if c.shape != shape:
                    raise ValueError(f"{n}: checkpoint shape {c.shape} != state shape {shape}")
            arr = np.stack(comps, axis=-1)
        else:
            arr = read_field(src / f"{n}.gmcf")
            if arr.shape != shape:
                raise ValueError(f"{n}: checkpoint shape {arr.shape} != state shape {shape}")
        setattr(state, n, np.ascontiguousarray(arr, dtype=np.float32))
