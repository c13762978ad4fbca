import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for p in (ROOT, os.path.join(ROOT, "tests")):
    if p not in sys.path:
        sys.path.insert(0, p)

# The unmodified reference (gmcf_mini), when present: the pip install under
# baseline/_ref travels to the GPU box; /root/reference exists only in the
# build container.  Appended, so the package's own modules win.  With it
# importable the drop-in shares the reference's own Scheme/Grid/WindProfile
# classes (reftypes.py), which is the configuration users run.
for p in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
    if os.path.isdir(os.path.join(p, "gmcf_mini")) and p not in sys.path:
        sys.path.append(p)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built liblesb200.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")
