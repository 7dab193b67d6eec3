"""Time the cifar10_quick engine step (layered kernels) on one GPU; tool only.
  python tools/prof_cnn.py [--steps K] [--batch B]"""
import argparse
import ctypes as C
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--batch", type=int, default=100)
    ap.add_argument("--n", type=int, default=10000)
    a = ap.parse_args()
    import torch
    from paper_1602_08191_b200 import _lib as L
    from paper_1602_08191_b200.deepspark import DeepSpark, Model
    api = DeepSpark()
    X, y = api.gen_synthetic(a.n, 3072, 10, 1.0, 1.0, 1)
    w = api.init_params(Model.cifar10_quick(10), 2)
    h = (C.c_uint32 * 1)(0)
    d = L.ds_model_desc(2, 3072, 10, 0, h)
    hp = L.ds_hyper(0.01, 0.1, 10, a.batch, 10 ** 9, 0.0, 0.0, 0)
    e = C.c_void_p()
    L.check(L.lib.ds_engine_create(C.byref(e), 0, C.byref(d), X.ctypes.data, y.ctypes.data, len(y), 10, C.byref(hp),
                                   5, w.ctypes.data, L.DS_ENGINE_AUTO))
    m = C.c_void_p()
    L.check(L.lib.ds_master_create(C.byref(m), 0, len(w), C.c_float(0.1), L.DS_MODE_LOCKFREE, w.ctypes.data))
    L.check(L.lib.ds_engine_attach_master(e, m))
    L.check(L.lib.ds_engine_reserve(e, a.steps + 10))
    L.check(L.lib.ds_engine_run(e, 5, 0, None))
    L.check(L.lib.ds_engine_sync(e))
    sp = C.c_void_p()
    L.check(L.lib.ds_engine_stream(e, C.byref(sp)))
    st = torch.cuda.ExternalStream(sp.value)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    t0 = time.perf_counter()
    L.check(L.lib.ds_engine_run(e, a.steps, 0, None))
    t1 = time.perf_counter()
    e1.record(st)
    L.check(L.lib.ds_engine_sync(e))
    ms = e0.elapsed_time(e1)
    loss = np.zeros(a.steps + 5)
    z = np.zeros(a.steps + 5)
    L.check(L.lib.ds_engine_log(e, 0, a.steps + 5, loss.ctypes.data, z.ctypes.data, np.zeros(a.steps + 5, np.uint8).ctypes.data,
                                np.zeros(a.steps + 5, np.uint32).ctypes.data))
    print(f"cifar10_quick b={a.batch}: {ms / a.steps * 1e3:.1f} us/step, {a.batch * a.steps / ms * 1e3:.0f} samples/s, "
          f"host enqueue {1e6 * (t1 - t0) / a.steps:.1f} us/step; loss {loss[0]:.4f} -> {loss[-1]:.4f}")
    L.lib.ds_engine_destroy(e)
    L.lib.ds_master_destroy(m)


if __name__ == "__main__":
    main()
