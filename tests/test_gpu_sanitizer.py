"""compute-sanitizer over the product kernels (tools/sanitize_workload.py:
the streaming append route with ring relocations and arena repacks, the
onesweep look-back, the general rebuild, every walk variant, the auditor):
memcheck (out-of-bounds / misaligned accesses, leaks), racecheck (shared-
memory hazards) and synccheck (illegal barriers) must report 0 errors."""
import os
import re
import shutil
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _sanitizer():
    exe = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(exe):
        pytest.fail("compute-sanitizer not found (CUDA toolkit)")
    return exe


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck"])
def test_sanitizer_clean(tool):
    cmd = [_sanitizer(), "--tool", tool, "--error-exitcode", "99", "--print-limit", "20"]
    if tool == "memcheck":
        cmd += ["--leak-check", "no"]
    cmd += [sys.executable, os.path.join(ROOT, "tools", "sanitize_workload.py")]
    p = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=1500)
    out = p.stdout + p.stderr
    m = re.search(r"ERROR SUMMARY: (\d+) error", out) or re.search(r"SUMMARY: \d+ hazards displayed \((\d+) error", out)
    assert p.returncode == 0 and "sanitize workload ok" in out and m and int(m.group(1)) == 0, out[-4000:]
