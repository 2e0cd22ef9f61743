"""compute-sanitizer memcheck over the small end-to-end cases of
tools/sanitize.py (every build route, both join bins, per-vertex, multi-part,
listings, MatrixMarket and TRIMCSR1 ingest).  racecheck/synccheck results of
the same cases: profiles/r01_compute_sanitizer.log."""
import os
import shutil
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_memcheck_clean(cuda_ok):
    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(cs):
        pytest.skip("compute-sanitizer not found")
    r = subprocess.run([cs, "--tool", "memcheck", "--error-exitcode", "3", sys.executable,
                        os.path.join(ROOT, "tools", "sanitize.py")], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "sanitize cases ok" in r.stdout, (r.stdout + r.stderr)[-3000:]
    assert "ERROR SUMMARY: 0 errors" in (r.stdout + r.stderr)
