"""pytest plugin: run the reference's own test suite (gmcf_mini's tests/)
with the CUDA drop-in installed.

``python -m pytest <reference tests> -p ref_suite_plugin`` calls
``paper_1504_02264_b200.install()`` before collection, so every
``les.step`` / stage / ``press`` / ``sor.solve_pressure`` /
``redblack_iteration`` / ``twinned_sweep`` call of the reference's tests --
on the reference's own numpy FlowState objects -- runs on the GPU through
the C ABI (the compat path: upload, run, copy the written fields back).
Each rebound function is wrapped in a counter; the counts are written to
``$LESB_REF_SUITE_COUNTS`` (JSON) at the end of the session, so a log shows
that the device path, not the reference's numpy, ran the tests.

Test infrastructure only: the reference suite is not shipped
with this repository; scripts/install_reference.sh puts a copy of it next
to the reference install under the git-ignored baseline/_ref.
"""

from __future__ import annotations

import functools
import json
import os

_COUNTS: dict = {}


def _counting(name, fn):
    @functools.wraps(fn)
    def wrapper(*a, **kw):
        _COUNTS[name] = _COUNTS.get(name, 0) + 1
        return fn(*a, **kw)

    return wrapper


def pytest_configure(config):
    import paper_1504_02264_b200 as P
    from paper_1504_02264_b200 import _native

    _native.load()  # fail loudly when the CUDA library is missing
    P.install()
    for (modname, n), _orig in list(P.dropin._saved.items()):
        if n.startswith("_RUNNERS:"):
            continue
        mod = _orig[0]
        setattr(mod, n, _counting(f"{modname}.{n}", getattr(mod, n)))


def pytest_sessionfinish(session, exitstatus):
    out = os.environ.get("LESB_REF_SUITE_COUNTS")
    if out:
        with open(out, "w") as f:
            json.dump({"exitstatus": int(exitstatus), "device_calls": _COUNTS}, f, indent=1, sort_keys=True)
    total = sum(_COUNTS.get(k, 0) for k in _COUNTS)
    print(f"\n[ref_suite_plugin] drop-in installed; {total} calls routed to the CUDA path: "
          + ", ".join(f"{k.split('.', 1)[1]}={v}" for k, v in sorted(_COUNTS.items())))
