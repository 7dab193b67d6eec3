"""Multi-GPU EASGD with the center sharded over the GPUs (needs >= 2 GPUs; skipped on a
single-GPU box). Deterministic mode must reproduce the CPU oracle's simulate() to within
1 ulp; async LockFree mode must stay finite and land within an accuracy band."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def ngpus():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


def run(world, *extra, script="mgpu_easgd.py"):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr=127.0.0.1", "--master-port=29517", os.path.join(ROOT, "tests", script), *extra]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    print(p.stdout[-3000:], p.stderr[-3000:])
    assert p.returncode == 0
    line = [l for l in p.stdout.splitlines() if l.startswith("MGPU_RESULT ")]
    assert line, "no result line"
    return json.loads(line[-1][len("MGPU_RESULT "):])


@pytest.mark.skipif(ngpus() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("kind", [1, 2])  # layered, fused
def test_deterministic_sharded_center(kind):
    r = run(min(ngpus(), 4), "--mode", "det", "--kind", str(kind))
    assert r["exchanges"] == r["expected_exchanges"]
    assert r["master_max_ulp"] <= 1 and r["workers_max_ulp"] <= 1
    assert r["snapshots_compared"] == 60 // 5 and r["snapshots_max_ulp"] <= 1
    assert r["acc_dev"] == r["acc_ref"]


@pytest.mark.skipif(ngpus() < 2, reason="needs >= 2 GPUs")
def test_deterministic_config1_two_gpus():
    r = run(2, "--mode", "det", "--big")
    assert r["master_max_ulp"] <= 1 and r["workers_max_ulp"] <= 1
    assert r["snapshots_compared"] == 200 // 10 and r["snapshots_max_ulp"] <= 1


@pytest.mark.skipif(ngpus() < 2, reason="needs >= 2 GPUs")
def test_async_lockfree_band():
    # BASELINE config 1's model and data (784-256-10, sep 0.1): accuracy is not saturated
    r = run(min(ngpus(), 4), "--mode", "async", "--big")
    assert r["finite"] and r["exchanges"] == r["expected_exchanges"]
    assert r["acc_ref"] < 0.99, "band test on a saturated run proves nothing"
    assert abs(r["acc_dev"] - r["acc_ref"]) <= 0.03


# ---- synchronous SGD: gradient "allreduce" fused into the update kernel over NVLink ----

@pytest.mark.skipif(ngpus() < 1, reason="needs a GPU")
def test_sync_single_rank_matches_oracle():
    r = run(1, script="mgpu_sync.py")
    assert r["rounds"] == r["i_max"]
    assert r["master_equal"] and r["loss_close"] and r["replicas_identical"]


@pytest.mark.skipif(ngpus() < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("wd", [0.0, 0.01])
def test_sync_multi_gpu_bit_identical(wd):
    r = run(min(ngpus(), 4), "--wd", str(wd), script="mgpu_sync.py")
    assert r["rounds"] == r["i_max"]
    assert r["replicas_identical"] and r["master_equal"] and r["loss_close"]


@pytest.mark.skipif(ngpus() < 2, reason="needs >= 2 GPUs")
def test_sync_config1_two_gpus():
    r = run(2, "--big", script="mgpu_sync.py")
    # 784-256-10, 100 rounds: CUDA's and glibc's exp/log may differ in the last f64 bit of
    # a softmax term; after f32 rounding and 100 SGD rounds that leaves a few-ulp
    # difference in a handful of master elements (observed: 1 of 203,530, 4 ulp).
    # Stated tolerance: <= 8 ulp per element, >= 99.99% of elements bit-identical.
    assert r["replicas_identical"] and r["loss_close"]
    assert r["master_max_ulp"] <= 8 and r["master_bit_identical"] >= 0.9999


@pytest.mark.skipif(ngpus() < 1, reason="needs a GPU")
def test_sync_engine_single_rank():
    r = run(1, "--engine", script="mgpu_sync.py")
    assert r["master_equal"] and r["loss_close"] and r["replicas_identical"]


@pytest.mark.skipif(ngpus() < 2, reason="needs >= 2 GPUs")
def test_sync_engine_multi_gpu():
    r = run(min(ngpus(), 4), "--engine", script="mgpu_sync.py")
    assert r["replicas_identical"] and r["master_equal"] and r["loss_close"]
