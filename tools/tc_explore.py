"""Scratch: measure the tensor-core engine's deviation from the f64 oracle (sets the
tolerances stated in tests/test_gpu_tc.py) and its step time."""
import ctypes as C
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
from oracle.oracle import Hyper, ModelSpec, Oracle  # noqa: E402
from paper_1602_08191_b200 import _lib as L  # noqa: E402
from test_gpu_engine import engine_log, engine_params, make_engine  # noqa: E402

orc = Oracle("dso")


def run_case(name, m, n, hp, with_master=None, sep=2.0, sigma=1.5):
    X, y = orc.gen_synthetic(n, m.n_features, m.n_classes, sep, sigma, 3)
    init = orc.init_params(m, 9)
    P = len(init)
    master0 = orc.init_params(m, 10)
    ref = orc.run_training_loop(m, X, y, m.n_classes, hp, 31, init, 2 if with_master else 0, master0)
    e = make_engine(L, m, X, y, m.n_classes, hp, 31, init, L.DS_ENGINE_TC)
    mh = None
    if with_master:
        mh = C.c_void_p()
        mode = L.DS_MODE_LOCKED if with_master == "locked" else L.DS_MODE_LOCKFREE
        L.check(L.lib.ds_master_create(C.byref(mh), 0, P, C.c_float(np.float32(hp.alpha)), mode, master0.ctypes.data))
        L.check(L.lib.ds_engine_attach_master(e, mh))
    t0 = time.time()
    L.check(L.lib.ds_engine_run(e, hp.i_max, 0, None))
    L.check(L.lib.ds_engine_sync(e))
    dt = time.time() - t0
    loss, cum, ex, per = engine_log(L, e, hp.i_max)
    params = engine_params(L, e, P)
    rl = np.abs(loss - ref["batch_loss"]) / np.abs(ref["batch_loss"])
    dp = np.abs(params - ref["final_params"]).max() / np.abs(ref["final_params"]).max()
    msg = f"{name:12s} master={with_master}: loss rel max {rl.max():.2e} (last {rl[-1]:.2e}), params max|d|/max|p| {dp:.2e}, ex equal {np.array_equal(ex, ref['exchanged'])}"
    if mh:
        snap = np.zeros(P, np.float32)
        L.check(L.lib.ds_master_snapshot(mh, snap.ctypes.data))
        dm = np.abs(snap - ref["master"]).max() / np.abs(ref["master"]).max()
        cnt = C.c_uint64()
        L.check(L.lib.ds_master_exchange_count(mh, C.byref(cnt)))
        msg += f", master {dm:.2e}, count {cnt.value}/{int(ref['exchanged'].sum())}"
    print(msg + f"  ({dt * 1e3:.1f} ms)", flush=True)
    L.lib.ds_engine_destroy(e)
    if mh:
        L.lib.ds_master_destroy(mh)


def timing(steps=20000):
    m = ModelSpec.mlp(784, [256], 10)
    X, y = orc.gen_synthetic(48000, 784, 10, 0.1, 1.0, 1)
    init = orc.init_params(m, 2)
    hp = Hyper(eta=0.05, alpha=0.1, tau=10, batch_size=32, i_max=steps)
    for kind in (L.DS_ENGINE_TC, L.DS_ENGINE_FUSED):
        e = make_engine(L, m, X, y, 10, hp, 5, init, kind)
        P = len(init)
        mh = C.c_void_p()
        L.check(L.lib.ds_master_create(C.byref(mh), 0, P, C.c_float(0.1), L.DS_MODE_LOCKFREE, init.ctypes.data))
        L.check(L.lib.ds_engine_attach_master(e, mh))
        L.check(L.lib.ds_engine_run(e, 100, 0, None))
        L.check(L.lib.ds_engine_sync(e))
        L.check(L.lib.ds_engine_reserve(e, steps))
        t0 = time.perf_counter()
        L.check(L.lib.ds_engine_run(e, steps, 0, None))
        L.check(L.lib.ds_engine_sync(e))
        dt = time.perf_counter() - t0
        loss, _, _, _ = engine_log(L, e, 100 + steps)
        print(f"kind {kind}: {dt / steps * 1e6:.2f} us/step = {32 * steps / dt / 1e6:.2f} M samples/s; "
              f"loss first/last {loss[0]:.4f} {loss[-1]:.4f}", flush=True)
        L.lib.ds_engine_destroy(e)
        L.lib.ds_master_destroy(mh)


def profile(steps=2000):
    m = ModelSpec.mlp(784, [256], 10)
    X, y = orc.gen_synthetic(48000, 784, 10, 0.1, 1.0, 1)
    init = orc.init_params(m, 2)
    hp = Hyper(eta=0.05, alpha=0.1, tau=10, batch_size=32, i_max=steps)
    path = os.path.join(ROOT, "gpurun_out", "tc_prof.txt")
    os.environ["DS_FUSED_PROFILE"] = path
    e = make_engine(L, m, X, y, 10, hp, 5, init, L.DS_ENGINE_TC)
    mh = C.c_void_p()
    L.check(L.lib.ds_master_create(C.byref(mh), 0, len(init), C.c_float(0.1), L.DS_MODE_LOCKFREE, init.ctypes.data))
    L.check(L.lib.ds_engine_attach_master(e, mh))
    L.check(L.lib.ds_engine_run(e, steps, 0, None))
    L.check(L.lib.ds_engine_sync(e))
    del os.environ["DS_FUSED_PROFILE"]
    print(open(path).read(), flush=True)
    L.lib.ds_engine_destroy(e)
    L.lib.ds_master_destroy(mh)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "prof":
        profile()
        timing()
        sys.exit(0)
    run_case("mlp20-16-3", ModelSpec.mlp(20, [16], 3), 300, Hyper(eta=0.05, tau=5, batch_size=16, i_max=40))
    run_case("mlp13-33-3", ModelSpec.mlp(13, [33], 3), 300, Hyper(eta=0.05, tau=5, batch_size=16, i_max=40))
    run_case("mlp-wd", ModelSpec.mlp(24, [40], 4), 300, Hyper(eta=0.05, tau=7, batch_size=32, i_max=40, weight_decay=0.01))
    for mm in (None, "lockfree", "locked"):
        run_case("mlp784", ModelSpec.mlp(784, [256], 10), 2000, Hyper(eta=0.05, tau=10, batch_size=32, i_max=100),
                 with_master=mm, sep=0.1, sigma=1.0)
    run_case("short-batch", ModelSpec.mlp(20, [33], 3), 70, Hyper(eta=0.05, tau=4, batch_size=32, i_max=12))
    timing()
