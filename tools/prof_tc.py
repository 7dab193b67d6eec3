"""One launch of the tensor-core MLP step (config-1 shapes: 784-256-10, b = 32, tau = 10,
LockFree center on the same GPU) for ncu captures: `python tools/prof_tc.py [steps]`."""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1602_08191_b200 import _lib as L  # noqa: E402
from paper_1602_08191_b200.deepspark import DeepSpark  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 300
api = DeepSpark()
X, y = api.gen_synthetic(48000, 784, 10, 0.1, 1.0, 1)
hidden = (C.c_uint32 * 1)(256)
desc = L.ds_model_desc(1, 784, 10, 1, hidden)
P = 203530
init = np.random.default_rng(0).uniform(-0.05, 0.05, P).astype(np.float32)
h = L.ds_hyper(0.05, 0.1, 10, 32, steps, 0.0, 0.0, 0)
e, m = C.c_void_p(), C.c_void_p()
L.check(L.lib.ds_engine_create(C.byref(e), 0, C.byref(desc), X.ctypes.data, y.ctypes.data, len(y), 10, C.byref(h), 5,
                               init.ctypes.data, L.DS_ENGINE_TC))
L.check(L.lib.ds_master_create(C.byref(m), 0, P, C.c_float(0.1), L.DS_MODE_LOCKFREE, init.ctypes.data))
L.check(L.lib.ds_engine_attach_master(e, m))
for _ in range(2):
    L.check(L.lib.ds_engine_run(e, steps, 0, None))
    L.check(L.lib.ds_engine_sync(e))
print("ok", steps)
