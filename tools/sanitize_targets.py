"""Small runs of the kernels with cross-CTA / cross-kernel synchronisation, for
compute-sanitizer (memcheck, racecheck, synccheck). Tool only, no torch:

  compute-sanitizer --tool racecheck python tools/sanitize_targets.py fused

targets:
  fused     mlp_kernel (DS_ENGINE_FUSED: grid barrier, reference-order f64 step) with a Locked
            master exchanged in-kernel, 12 steps
  tc        mlp_tc_kernel (DS_ENGINE_TC: cluster, mbarriers, TMA, tcgen05) with a LockFree
            master exchanged in-kernel, 12 steps; then two workers in one group launch
  exchange  exchange_kernel: Locked single-device, sharded (two shards of one GPU, device
            ticket dispenser) and ticketed exchanges
  sync      round_kernel: a synchronous group of 3 ranks on one GPU, SGD and EASGD rounds
"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1602_08191_b200 import _lib as L  # noqa: E402
from paper_1602_08191_b200.deepspark import DeepSpark  # noqa: E402

api = DeepSpark()


def engine(kind, X, y, F, H, NC, steps, batch, init, seed=5):
    hidden = (C.c_uint32 * 1)(H)
    desc = L.ds_model_desc(1, F, NC, 1, hidden)
    h = L.ds_hyper(0.05, 0.1, 5, batch, steps, 0.0, 0.0, 0)
    e = C.c_void_p()
    L.check(L.lib.ds_engine_create(C.byref(e), 0, C.byref(desc), X.ctypes.data, y.ctypes.data, len(y), NC,
                                   C.byref(h), seed, init.ctypes.data, kind))
    return e, (hidden, desc, h)


def model_run(kind, mode, group):
    F, H, NC = 784, 256, 10
    X, y = api.gen_synthetic(2000, F, NC, 0.1, 1.0, 1)
    P = F * H + H + NC * H + NC
    init = np.random.default_rng(0).uniform(-0.05, 0.05, P).astype(np.float32)
    m = C.c_void_p()
    L.check(L.lib.ds_master_create(C.byref(m), 0, P, C.c_float(0.1), mode, init.ctypes.data))
    es = []
    for k in range(2 if group else 1):
        e, keep = engine(kind, X, y, F, H, NC, 12, 32, init, seed=5 + k)
        L.check(L.lib.ds_engine_attach_master(e, m))
        es.append((e, keep))
    if group:
        arr = (C.c_void_p * len(es))(*[e.value for e, _ in es])
        L.check(L.lib.ds_engine_run_group(arr, len(es), 12))
    else:
        L.check(L.lib.ds_engine_run(es[0][0], 12, 0, None))
    for e, _ in es:
        L.check(L.lib.ds_engine_sync(e))
        L.lib.ds_engine_destroy(e)
    snap = np.zeros(P, np.float32)
    L.check(L.lib.ds_master_snapshot(m, snap.ctypes.data))
    assert np.isfinite(snap).all()
    L.lib.ds_master_destroy(m)


def exchange_run():
    n = 1 << 16
    rng = np.random.default_rng(1)
    m0 = rng.standard_normal(n).astype(np.float32)
    w = rng.standard_normal(n).astype(np.float32)
    wd, outd = C.c_void_p(), C.c_void_p()
    L.check(L.lib.ds_device_alloc(0, 4 * n, C.byref(wd)))
    L.check(L.lib.ds_device_alloc(0, 4 * n, C.byref(outd)))
    L.check(L.lib.ds_memcpy(wd, w.ctypes.data, 4 * n, None))
    m = C.c_void_p()
    L.check(L.lib.ds_master_create(C.byref(m), 0, n, C.c_float(0.1), L.DS_MODE_LOCKED, m0.ctypes.data))
    for _ in range(3):
        L.check(L.lib.ds_master_exchange(m, wd, outd, None))
    for t in range(3):
        L.check(L.lib.ds_master_exchange_ticketed(m, wd, outd, t, None))
    snap = np.zeros(n, np.float32)
    L.check(L.lib.ds_master_snapshot(m, snap.ctypes.data))
    L.lib.ds_master_destroy(m)
    hs, recs = [], []
    for r in range(2):
        h = C.c_void_p()
        L.check(L.lib.ds_master_create_sharded(C.byref(h), 0, n, C.c_float(0.1), L.DS_MODE_LOCKED, r, 2,
                                               m0.ctypes.data))
        rec = (C.c_uint8 * L.DS_IPC_RECORD_BYTES)()
        L.check(L.lib.ds_master_export(h, rec))
        hs.append(h)
        recs.append(bytes(rec))
    allrec = (C.c_uint8 * (2 * L.DS_IPC_RECORD_BYTES)).from_buffer_copy(b"".join(recs))
    for h in hs:
        L.check(L.lib.ds_master_attach(h, allrec))
    for k in range(4):
        L.check(L.lib.ds_master_exchange(hs[k % 2], wd, outd, None))
    L.check(L.lib.ds_master_snapshot(hs[0], snap.ctypes.data))
    assert np.isfinite(snap).all()
    for h in hs:
        L.lib.ds_master_destroy(h)
    L.lib.ds_device_free(wd)
    L.lib.ds_device_free(outd)


def sync_run():
    n, world = 100_003, 3
    rng = np.random.default_rng(2)
    syncs, recs = [], []
    for k in range(world):
        s = C.c_void_p()
        L.check(L.lib.ds_sync_create(C.byref(s), 0, n, k, world))
        rec = (C.c_uint8 * L.DS_IPC_RECORD_BYTES)()
        L.check(L.lib.ds_sync_export(s, rec))
        syncs.append(s)
        recs.append(bytes(rec))
    allrec = (C.c_uint8 * (world * L.DS_IPC_RECORD_BYTES)).from_buffer_copy(b"".join(recs))
    for s in syncs:
        L.check(L.lib.ds_sync_attach(s, allrec))
    bufs = []
    for _ in range(2 * world + 1):
        p = C.c_void_p()
        L.check(L.lib.ds_device_alloc(0, 4 * n, C.byref(p)))
        v = rng.standard_normal(n).astype(np.float32)
        L.check(L.lib.ds_memcpy(p, v.ctypes.data, 4 * n, None))
        bufs.append(p)
    flags = C.c_void_p()
    L.check(L.lib.ds_device_alloc(0, 4, C.byref(flags)))
    L.check(L.lib.ds_memset(flags, 0, 4, None))
    reps = (C.c_void_p * world)(*[bufs[k].value for k in range(world)])
    works = (C.c_void_p * world)(*[bufs[world + k].value for k in range(world)])
    group = (C.c_void_p * world)(*[s.value for s in syncs])
    for _ in range(2):
        for k in range(world):
            slot = C.c_void_p()
            L.check(L.lib.ds_sync_begin(syncs[k], C.byref(slot), None))
            L.check(L.lib.ds_memcpy(slot, bufs[-1], 4 * n, None))
        L.check(L.lib.ds_sync_reduce_update_group(group, world, reps, C.c_float(0.01), C.c_float(1e-4), flags, None))
        L.check(L.lib.ds_sync_easgd_update_group(group, world, works, reps, C.c_float(0.2), flags, None))
    L.check(L.lib.ds_stream_sync(None))
    for s in syncs:
        L.lib.ds_sync_destroy(s)
    for p in bufs:
        L.lib.ds_device_free(p)
    L.lib.ds_device_free(flags)


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    if what in ("fused", "all"):
        model_run(L.DS_ENGINE_FUSED, L.DS_MODE_LOCKED, False)
    if what in ("tc", "all"):
        model_run(L.DS_ENGINE_TC, L.DS_MODE_LOCKFREE, False)
        model_run(L.DS_ENGINE_TC, L.DS_MODE_LOCKED, True)
    if what in ("exchange", "all"):
        exchange_run()
    if what in ("sync", "all"):
        sync_run()
    print("ok", what, flush=True)
