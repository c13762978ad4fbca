"""bench.py keeps the driver contract: it compiles, and its CLI accepts the
driver's flags (the measurement itself needs a GPU)."""

import os
import py_compile
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_compiles_and_parses_flags():
    py_compile.compile(os.path.join(ROOT, "bench.py"), doraise=True)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--help"], capture_output=True, text=True,
                         timeout=120)
    assert out.returncode == 0, out.stderr
    for flag in ("--gpus", "--steps", "--warmup", "--impl", "--grid"):
        assert flag in out.stdout
