"""A few AlexNet-shaped engine steps (batch 128, 224x224x3, 1000 classes) for ncu launch
lists: python tools/prof_alex.py [steps]."""
import ctypes as C
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1602_08191_b200 import _lib as L  # noqa: E402
from paper_1602_08191_b200.deepspark import DeepSpark, Model  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
api = DeepSpark()
B, N, S, Cls = 128, 256, 224, 1000
F = 3 * S * S
X = torch.randn(N, F, device="cuda")
y = np.random.default_rng(1).integers(0, Cls, N).astype(np.uint32)
m = Model.alexnet(S, Cls)
init = api.init_params(m, 1)
d = L.ds_model_desc(3, F, Cls, 0, (C.c_uint32 * 1)(0))
hp = L.ds_hyper(0.01, 0.1, 10, B, 10 ** 9, 0.0, 0.0, 0)
e = C.c_void_p()
L.check(L.lib.ds_engine_create(C.byref(e), 0, C.byref(d), C.c_void_p(X.data_ptr()), y.ctypes.data, N, Cls,
                               C.byref(hp), 5, init.ctypes.data, L.DS_ENGINE_LAYERED))
L.check(L.lib.ds_engine_run(e, steps, 0, None))
L.check(L.lib.ds_engine_sync(e))
loss = np.zeros(steps)
L.check(L.lib.ds_engine_log(e, 0, steps, loss.ctypes.data, None, None, None))
print("losses", loss)
