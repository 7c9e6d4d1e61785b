"""compute-sanitizer over a small forward (SURVEY §5 race tooling): racecheck and synccheck
for the shared-memory protocols (the gate's block ranks and scans, the row movers, the
look-back-free level-1 scan), memcheck for out-of-bounds accesses -- on the SIMT fp32 path
and on the bf16 path with the tensor-core gate / FFN (tcgen05, TMA, mbarriers) and the
peer-store exchange.  Skipped when compute-sanitizer is not installed."""
import os
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SAN = shutil.which("compute-sanitizer") or ("/usr/local/cuda/bin/compute-sanitizer"
                                            if os.path.exists("/usr/local/cuda/bin/compute-sanitizer") else None)


@pytest.mark.skipif(SAN is None, reason="compute-sanitizer not available")
@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
@pytest.mark.parametrize("args", [["fp32"], ["bf16"], ["bf16", "peer"]])
def test_sanitizer_clean(tool, args):
    cmd = [SAN, "--tool", tool, "--error-exitcode", "97", "--target-processes", "all", sys.executable,
           os.path.join(ROOT, "tests", "sanitizer_case.py")] + args
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200)
    tail = (r.stdout + r.stderr)[-3000:]
    assert r.returncode == 0, tail
    assert "SANITIZER_CASE_OK" in r.stdout, tail
    assert "ERROR SUMMARY: 0 errors" in r.stdout + r.stderr or "RACECHECK SUMMARY: 0 hazards" in r.stdout + r.stderr, tail
