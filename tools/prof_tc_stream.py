"""Stream-mode (host-fed, zero-copy ring) vs device-resident timing of one tensor-core
engine at config-1 shapes, with the per-phase profile (DS_FUSED_PROFILE=<file>) of each:
`python tools/prof_tc_stream.py [steps]`. Tool only."""
import ctypes as C
import os
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1602_08191_b200 import _lib as L  # noqa: E402
from paper_1602_08191_b200.deepspark import DeepSpark  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
api = DeepSpark()
X, y = api.gen_synthetic(24000, 784, 10, 0.1, 1.0, 1)
X = np.ascontiguousarray(X, np.float32)
y = np.ascontiguousarray(y, np.uint32)
hidden = (C.c_uint32 * 1)(256)
desc = L.ds_model_desc(1, 784, 10, 1, hidden)
P = 203530
init = np.random.default_rng(0).uniform(-0.05, 0.05, P).astype(np.float32)
h = L.ds_hyper(0.05, 0.1, 10, 32, 10 ** 9, 0.0, 0.0, 0)


def engine():
    e, m = C.c_void_p(), C.c_void_p()
    L.check(L.lib.ds_engine_create(C.byref(e), 0, C.byref(desc), X.ctypes.data, y.ctypes.data, len(y), 10,
                                   C.byref(h), 5, init.ctypes.data, L.DS_ENGINE_TC))
    L.check(L.lib.ds_master_create(C.byref(m), 0, P, C.c_float(0.1), L.DS_MODE_LOCKFREE, init.ctypes.data))
    L.check(L.lib.ds_engine_attach_master(e, m))
    L.check(L.lib.ds_engine_reserve(e, 2 * steps + 8))
    return e, m


e, m = engine()
L.check(L.lib.ds_engine_run(e, 300, 0, None))
L.check(L.lib.ds_engine_sync(e))
t0 = time.perf_counter()
L.check(L.lib.ds_engine_run(e, steps, 0, None))
L.check(L.lib.ds_engine_sync(e))
print(f"device-resident: {1e6 * (time.perf_counter() - t0) / steps:.2f} us/step (wall)", flush=True)
idx, sizes = api.sweep_batches(len(y), 32, 7, steps)
idx = np.ascontiguousarray(idx, np.uint32)
sizes = np.ascontiguousarray(sizes, np.uint32)
import torch  # noqa: E402
loss = torch.zeros(steps, dtype=torch.float64, pin_memory=True)
for rep in range(2):
    t0 = time.perf_counter()
    L.check(L.lib.ds_engine_stream_begin(e, steps, C.c_void_p(loss.data_ptr())))
    t1 = time.perf_counter()
    L.check(L.lib.ds_engine_stream_push_rows_n(e, X.ctypes.data, y.ctypes.data, idx.ctypes.data, sizes.ctypes.data,
                                               steps))
    t2 = time.perf_counter()
    L.check(L.lib.ds_engine_stream_end(e))
    t3 = time.perf_counter()
    print(f"stream rep {rep}: begin {1e3 * (t1 - t0):.2f} ms, pushes {1e6 * (t2 - t1) / steps:.2f} us/step, "
          f"end {1e3 * (t3 - t2):.2f} ms, total {1e6 * (t3 - t0) / steps:.2f} us/step", flush=True)
# host-only producer cost: the same gathers into a numpy ring (no device)
from paper_1602_08191_b200 import _lib  # noqa: E402,F401
t0 = time.perf_counter()
ring = np.empty((8, 32, 784), np.float32)
for s in range(min(steps, 2000)):
    ring[s % 8, :sizes[s]] = X[idx[s, :sizes[s]]]
print(f"numpy gather: {1e6 * (time.perf_counter() - t0) / min(steps, 2000):.2f} us/step", flush=True)
L.lib.ds_engine_destroy(e)
L.lib.ds_master_destroy(m)
