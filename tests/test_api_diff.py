"""The drop-in C++ API against the reference library itself: the report of
tests/cpp/api_diff.cpp (every public function of include/tbsim/*.hpp on the
reference's generators, random DAGs of the test's own construction,
degenerate and invalid graphs; doubles as hex floats, exceptions as type +
text) built on this repo's libtbsim_cpp.so must equal, line for line, the
report the same source printed when built on the reference's unmodified
sources (tests/golden/make_api_diff.sh -> tests/golden/api_diff_ref.txt.gz)."""
import gzip
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "api_diff")
GOLDEN = os.path.join(ROOT, "tests", "golden", "api_diff_ref.txt.gz")


def _golden():
    with gzip.open(GOLDEN, "rt") as f:
        return f.read().splitlines()


def test_golden_report_is_complete():
    lines = _golden()
    assert lines[-1] == "end"
    assert sum(1 for x in lines if x.startswith("== ")) >= 25
    assert any(x.startswith("sim inspirit makespan=") for x in lines)


@pytest.mark.gpu
def test_cpp_api_report_matches_the_reference():
    subprocess.check_call(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp"), BIN])
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    got, want = r.stdout.splitlines(), _golden()
    section = ""
    for i, (g, w) in enumerate(zip(got, want)):
        if w.startswith("== "):
            section = w
        assert g == w, f"line {i + 1} ({section}):\n  b200:      {g}\n  reference: {w}"
    assert len(got) == len(want), (len(got), len(want))
