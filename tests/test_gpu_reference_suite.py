"""the reference's own test suite (gmcf_mini tests/: test_les,
test_sor, test_acceptance, ...) run with the CUDA drop-in installed
(tests/ref_suite_plugin.py), i.e. every hot-path call of those tests -- on
the reference's own numpy FlowState objects -- goes through the C ABI.

The suite comes from baseline/_ref/_tests (scripts/install_reference.sh);
skipped when it is absent.  The log and the per-function device call counts
are written under gpurun_out/ref_suite/ when that directory exists.
"""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
SUITE = os.path.join(REF, "_tests")

# Every module runs.  Note on acceptance criterion 10 (a soft, non-gating
# timing check of the CPU worker pool's TWINNED speed-up, workers=1 vs 4):
# the drop-in accepts ``workers`` and ignores it (results are worker
# invariant by contract, SURVEY 8(b) Threading); the criterion still passes
# because its first call also pays the device setup, so its "speed-up"
# number means nothing on the GPU path.
MODULES = ["test_les.py", "test_sor.py", "test_acceptance.py", "test_cli.py", "test_coupling.py",
           "test_driver.py", "test_runtime.py", "test_config.py"]


@pytest.mark.skipif(not os.path.isdir(SUITE), reason="reference suite not installed (scripts/install_reference.sh)")
@pytest.mark.parametrize("module", MODULES)
def test_reference_suite_under_install(module, tmp_path):
    out_dir = os.path.join(ROOT, "gpurun_out", "ref_suite")
    os.makedirs(out_dir, exist_ok=True)
    counts = os.path.join(out_dir, module.replace(".py", "_counts.json"))
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([os.path.join(ROOT, "tests"), ROOT, REF, env.get("PYTHONPATH", "")])
    env["LESB_REF_SUITE_COUNTS"] = counts
    cmd = [sys.executable, "-m", "pytest", os.path.join(SUITE, module), "-p", "ref_suite_plugin", "-q",
           "-p", "no:cacheprovider", "-rs", "-s", "--rootdir", str(tmp_path)]
    res = subprocess.run(cmd, capture_output=True, text=True, env=env, cwd=str(tmp_path), timeout=1500)
    with open(os.path.join(out_dir, module.replace(".py", ".log")), "w") as f:
        f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    assert res.returncode == 0, res.stdout[-4000:] + res.stderr[-2000:]
    calls = json.load(open(counts))["device_calls"]
    if module in ("test_les.py", "test_sor.py", "test_acceptance.py", "test_cli.py"):
        assert sum(calls.values()) > 0, "no call reached the drop-in"
