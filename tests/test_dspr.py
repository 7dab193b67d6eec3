"""The DSPR TCP front-end over the device center: protocol fuzz
(the reference's release-gate check 8, acceptance.cpp:436-545, restated in
tests/cpp/test_dspr_fuzz.cpp) and a TCP client's exchanges bit-exact against the elastic
kernel. The reference's own protocol / exchanger / worker suites run in
tests/test_reference_suites.py."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "_bin", "dspr_tests")

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not os.path.exists(BIN), reason="tests/cpp/_bin/dspr_tests not built")]


def test_dspr_suite():
    p = subprocess.run([BIN, "--test-suite=dspr"], capture_output=True, text=True, timeout=600)
    print(p.stdout[-3000:], p.stderr[-3000:])
    assert p.returncode == 0, p.stdout[-2000:] + p.stderr[-2000:]
