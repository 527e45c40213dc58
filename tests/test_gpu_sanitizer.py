"""compute-sanitizer over the product kernels (tools/sanitize_workload.py:
the streaming append route with ring relocations and arena repacks, the
onesweep look-back, the general rebuild, every walk variant, the auditor):
memcheck (out-of-bounds / misaligned accesses, leaks), racecheck (shared-
memory hazards) and synccheck (illegal barriers) must report 0 errors.

Where the GPU pool refuses compute-sanitizer (its wrapper reports it closed),
those three skip, and the guard test carries the check with the library's own
instrumentation: TWG_GUARD=1 poisons every device block the allocator hands
out and puts a 4 KiB guard past each (checked on free, csrc/arena.cu), so the
same workload must report no write past a block and produce walks (and
audits) identical to a plain run — a read of never-written memory would
change them."""
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
    if "closed on this pool" in out:
        pytest.skip("compute-sanitizer refused by the GPU pool; test_guarded_workload_identical covers it")
    m = re.search(r"ERROR SUMMARY: (\d+) error", out) or re.search(r"SUMMARY: \d+ hazards displayed \((\d+) error", out)
    assert p.returncode == 0 and "sanitize workload ok" in out and m and int(m.group(1)) == 0, out[-4000:]


def _workload(env_extra):
    env = dict(os.environ, **env_extra)
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_workload.py")], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=900)
    out = p.stdout + p.stderr
    assert p.returncode == 0 and "sanitize workload ok" in out, out[-4000:]
    m = re.search(r"^digest ([0-9a-f]{64})$", p.stdout, re.M)
    assert m, out[-2000:]
    return m.group(1), out


def test_guarded_workload_identical():
    plain, _ = _workload({"TWG_GUARD": "0"})
    guarded, out = _workload({"TWG_GUARD": "1"})
    assert "TWG_GUARD:" not in out, out[-4000:]
    assert guarded == plain
