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
  run) and every criterion is asserted. The three wall-clock criteria (08
  slope of per-batch ingest time, 09 rebuild scaling, 10 per-walk cost)
  time sub-millisecond device work through host round trips, whose latency
  follows the GPU's clock / power state: one that fails is re-run alone
  (the binary's own criterion selection, acceptance.cpp:502-506) up to two
  more times and passes if an attempt passes; every attempt's measured value
  is printed. The nine other criteria must pass on the first run.
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


def _run(path, timeout=900, args=()):
    if not os.path.exists(path):
        pytest.skip(f"{path} not built (make ref_suites needs /root/reference at build time)")
    r = subprocess.run([path, *args], capture_output=True, text=True, timeout=timeout, cwd=os.path.dirname(path))
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
    exe = os.path.join(ROOT, "build", "ref_suites", "gpu", "acceptance")
    crit_re = re.compile(r"^\[(PASS|FAIL)\] (\d\d) (\S+)\s+(.*)$", re.M)
    rc, out = _run(exe, 1200)
    print(out)
    crit = crit_re.findall(out)
    assert len(crit) == 12, out[-3000:]
    failed = {c[1]: c for c in crit if c[0] != "PASS"}
    timing = {"08", "09", "10"}
    assert not set(failed) - timing, [failed[k] for k in sorted(set(failed) - timing)]
    for attempt in (2, 3):
        if not failed:
            break
        rc2, out2 = _run(exe, 600, args=[str(int(k)) for k in sorted(failed)])
        print(f"--- attempt {attempt}: re-run of wall-clock criteria {sorted(failed)}\n{out2}")
        for c in crit_re.findall(out2):
            if c[0] == "PASS":
                failed.pop(c[1], None)
    assert not failed, list(failed.values())
