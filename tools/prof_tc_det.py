"""BASELINE config 1's deterministic mode on one GPU (2 tensor-core workers in one launch, Locked
center, replayed simulate_async tickets) vs the async LockFree group, with the per-phase profile of
worker 0's CTA 0 (DS_FUSED_PROFILE=<file>): `python tools/prof_tc_det.py [steps]`. Tool only."""
import ctypes as C
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1602_08191_b200 import _lib as L  # noqa: E402
from paper_1602_08191_b200.deepspark import DeepSpark  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
api = DeepSpark()
P, W, tau = 203530, 2, 10
init = np.random.default_rng(0).uniform(-0.05, 0.05, P).astype(np.float32)
hidden = (C.c_uint32 * 1)(256)
desc = L.ds_model_desc(1, 784, 10, 1, hidden)
shards = [api.gen_synthetic(24000, 784, 10, 0.1, 1.0, 1 + k) for k in range(W)]
for mode in ("async", "det"):
    order_w, _ = api.exchange_order(W, tau, steps + 8, 1)
    m = C.c_void_p()
    L.check(L.lib.ds_master_create(C.byref(m), 0, P, C.c_float(0.1),
                                   L.DS_MODE_LOCKED if mode == "det" else L.DS_MODE_LOCKFREE, init.ctypes.data))
    h = L.ds_hyper(0.05, 0.1, tau, 32, steps + 8, 0.0, 0.0, 0)
    es = []
    for k in range(W):
        X, y = shards[k]
        e = C.c_void_p()
        L.check(L.lib.ds_engine_create(C.byref(e), 0, C.byref(desc), X.ctypes.data, y.ctypes.data, len(y), 10,
                                       C.byref(h), 5 + k, init.ctypes.data, L.DS_ENGINE_TC))
        L.check(L.lib.ds_engine_attach_master(e, m))
        if mode == "det":
            tk = np.nonzero(np.asarray(order_w) == k)[0].astype(np.uint64)
            L.check(L.lib.ds_engine_set_tickets(e, tk.ctypes.data, len(tk)))
        L.check(L.lib.ds_engine_reserve(e, steps + 8))
        es.append(e)
    arr = (C.c_void_p * W)(*[e.value for e in es])
    with open(os.environ.get("DS_FUSED_PROFILE", "/dev/null"), "a") as f:
        f.write(f"# {mode}\n")
    t0 = time.perf_counter()
    L.check(L.lib.ds_engine_run_group(arr, W, steps))
    for e in es:
        L.check(L.lib.ds_engine_sync(e))
    print(mode, f"{(time.perf_counter() - t0) / steps * 1e6:.2f} us/step (wall, incl. launch)")
    for e in es:
        L.lib.ds_engine_destroy(e)
    L.lib.ds_master_destroy(m)
