"""The reference's OWN test suites, unchanged.

`make ref_suites` (run by __graft_entry__.build() where /root/reference
exists) compiles /root/reference/proj/tests/{test_*.cpp, acceptance.cpp}
exactly as they lie, with our doctest shim (tests/cpp/doctest_shim; the
reference's vendor/doctest is absent), twice:

* build/ref_suites/cpu/*: against the reference core itself (oracle/_ref
  objects). Every suite must pass there: this pins the shim (CPU test).
* build/ref_suites/gpu/*: against include/timewalk + libtimewalk_b200.so, the
  drop-in. Every unit suite must pass on the B200; acceptance.cpp reports
  its 12 criteria (proj/test_output.txt:33-45 is the reference's recorded
  run) and every criterion is asserted — a timing criterion that failed on
  the GPU would fail here with its measured value in the message.
"""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITES = ["test_primitives", "test_rng", "test_samplers", "test_edge_store", "test_window", "test_walk_engine",
          "test_validity", "test_io", "test_replay", "test_synthetic"]
SUMMARY = re.compile(r"\[doctest shim\] test cases: (\d+) \| (\d+) passed \| (\d+) failed \| "
                     r"assertions: (\d+) \| (\d+) passed \| (\d+) failed")
# test cases per suite in the reference sources (TEST_CASE count)
CASES = {"test_primitives": 5, "test_rng": 3, "test_samplers": 11, "test_edge_store": 15, "test_window": 12,
         "test_walk_engine": 29, "test_validity": 8, "test_io": 6, "test_replay": 8, "test_synthetic": 5}


def _run(path, timeout=900):
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (make ref_suites needs /root/reference at build time)")
    r = subprocess.run([path], capture_output=True, text=True, timeout=timeout, cwd=os.path.dirname(path))
    return r.returncode, r.stdout + r.stderr


def _check_suite(kind, name):
    rc, out = _run(os.path.join(ROOT, "build", "ref_suites", kind, name))
    m = SUMMARY.search(out)
    assert m, out[-2000:]
    cases, passed, failed, asserts, apassed, afailed = (int(x) for x in m.groups())
    assert rc == 0 and failed == 0 and afailed == 0, out[-4000:]
    assert cases == CASES[name]
    print(f"{kind} {name}: {cases} test cases, {asserts} assertions, all passed")


def test_shim_selftest():
    exe = os.path.join(ROOT, "build", "shim_selftest")
    src = os.path.join(ROOT, "tests", "cpp", "shim_selftest.cpp")
    os.makedirs(os.path.dirname(exe), exist_ok=True)
    subprocess.run(["g++", "-std=c++20", "-I", os.path.join(ROOT, "tests", "cpp", "doctest_shim"), src, "-o", exe],
                   check=True)
    rc, out = _run(exe, 60)
    assert rc == 1
    m = SUMMARY.search(out)
    assert m and tuple(int(x) for x in m.groups()) == (4, 2, 2, 10, 6, 4), out


@pytest.mark.parametrize("name", SUITES)
def test_reference_suite_on_reference(name):
    """The shim runs the reference's suites to 100% on the reference itself."""
    _check_suite("cpu", name)


@pytest.mark.gpu
@pytest.mark.parametrize("name", SUITES)
def test_reference_suite_on_b200(name):
    _check_suite("gpu", name)


@pytest.mark.gpu
def test_reference_acceptance_on_b200():
    rc, out = _run(os.path.join(ROOT, "build", "ref_suites", "gpu", "acceptance"), 1200)
    crit = re.findall(r"^\[(PASS|FAIL)\] (\d\d) (\S+)\s+(.*)$", out, re.M)
    print(out)
    assert len(crit) == 12, out[-3000:]
    failed = [c for c in crit if c[0] != "PASS"]
    assert not failed and rc == 0, failed
