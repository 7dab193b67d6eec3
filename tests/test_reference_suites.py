"""The reference's own unit suites (proj/tests/test_{params,model,engine,simulator,data,
protocol,exchanger,worker}.cpp),
compiled UNMODIFIED against include/deepspark/ and linked with the B200 library
(oracle/Makefile `reftests`), run on the GPU. Every assertion the reference makes about
its own API — bit-exact one-step equality, replay of the elastic kernel, sync averaging,
the frozen convergence fixture — is checked against our implementation."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "reftests_b200")

pytestmark = pytest.mark.skipif(not os.path.exists(BIN), reason="oracle/_ref/reftests_b200 not built")


def run_suite(suite):
    p = subprocess.run([BIN, f"--test-suite={suite}"], capture_output=True, text=True, timeout=900,
                       env={**os.environ, "DEEPSPARK_LOG": "error"})
    print(p.stdout[-4000:])
    print(p.stderr[-4000:])
    return p


@pytest.mark.parametrize("suite", ["data", "protocol"])
def test_host_only_suites(suite):
    """test_data.cpp (dataset generation, partition, holdout, CSV, DSHD) and
    test_protocol.cpp (the DSPR wire codec) need no GPU."""
    p = run_suite(suite)
    assert p.returncode == 0, p.stderr[-2000:]


@pytest.mark.gpu
@pytest.mark.parametrize("suite", ["params", "model", "engine", "simulator", "exchanger", "worker"])
def test_reference_suite_on_b200(suite):
    p = run_suite(suite)
    assert p.returncode == 0, p.stderr[-3000:]
