"""The reference's own 206-test suite run against this package
(tests/ref_suite_plugin.py).  Needs the GPU (every
hot-path call is a CUDA kernel) and baseline/_ref (oracle/build_ref.sh).
Writes the per-test outcome summary to gpurun_out/ref_suite.json."""

import json
import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITE = os.path.join(ROOT, "baseline", "_ref", "ref_tests")

pytestmark = pytest.mark.gpu


def test_reference_suite_against_this_package():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    if not os.path.isdir(SUITE):
        pytest.skip("reference suite not installed (oracle/build_ref.sh)")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([os.path.join(ROOT, "tests"), ROOT]))
    r = subprocess.run([sys.executable, "-m", "pytest", SUITE, "-p", "ref_suite_plugin", "-p", "no:cacheprovider",
                        "-q", "-rfExX", "--no-header"], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=3000)
    tail = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-500:]
    counts = {k: int(v) for v, k in re.findall(r"(\d+) (passed|failed|xfailed|xpassed|error|errors|skipped)", tail)}
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "ref_suite.log"), "w") as fh:
        fh.write(r.stdout + r.stderr)
    with open(os.path.join(ROOT, "gpurun_out", "ref_suite.json"), "w") as fh:
        json.dump({"summary": tail, "counts": counts,
                   "details": [ln for ln in r.stdout.splitlines() if ln.startswith(("FAILED", "ERROR", "XFAIL", "XPASS"))]},
                  fh, indent=1)
    assert counts.get("failed", 0) == 0 and counts.get("error", 0) + counts.get("errors", 0) == 0, r.stdout[-6000:]
    assert counts.get("passed", 0) + counts.get("xpassed", 0) >= 190, tail
