"""The reference's public C++ API (timewalk::EdgeStore, WindowManager,
generate_walks, replay_stream, samplers, primitives) compiled against our
headers and run on the GPU: the drop-in boundary exercised from C++."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_cpp_facade_known_answers():
    exe = os.path.join(ROOT, "build", "facade_test")
    if not os.path.exists(exe):
        subprocess.run(["make", "-C", ROOT, "facade_test"], check=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "checks passed" in r.stdout
