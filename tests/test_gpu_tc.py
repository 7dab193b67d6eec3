"""GPU tests of the tensor-core fast step (DS_ENGINE_TC, csrc/mlp_tc.cu) against the CPU
oracle's restatement of the reference (engine.cpp:50-113, simulator.cpp:70-154).

The fast step computes its two dense contractions on tcgen05 with bf16 operands (f32
accumulation), the logits in tf32, everything else in f32 -- it is NOT the reference's f64
order, so parity is a stated tolerance (bf16 <= 1e-3 relative):
  * per-step batch loss within 5e-3 relative (observed <= 2.2e-3),
  * final parameters / center within 2e-3 of max|param| after 40-150 steps
    (observed <= 1.1e-3),
  * exchange decisions (fixed period) and exchange counts exact,
  * the deterministic multi-worker schedule (tickets) reproducible bit for bit,
  * async LockFree (concurrent workers): holdout accuracy within 0.02 and holdout loss
    within 3% of the reference's simulate on BASELINE config 1 (784-256-10, 2 workers).
"""
import ctypes as C

import numpy as np
import pytest

from oracle.oracle import Hyper, ModelSpec, Oracle, SimSpec

pytestmark = pytest.mark.gpu

LOSS_RTOL = 5e-3
PARAM_TOL = 2e-3


@pytest.fixture(scope="module")
def L():
    from paper_1602_08191_b200 import _lib
    return _lib


@pytest.fixture(scope="module")
def orc():
    return Oracle("dso")


@pytest.fixture(scope="module")
def api():
    from paper_1602_08191_b200.deepspark import DeepSpark
    return DeepSpark()


def desc_of(L, m):
    h = (C.c_uint32 * max(1, len(m.hidden)))(*m.hidden)
    d = L.ds_model_desc(0 if m.kind == "softmax" else 1, m.n_features, m.n_classes, len(m.hidden), h)
    d._keep = h
    return d


def make_engine(L, m, X, y, ncls, hp, seed, init, kind=None, device=0):
    d = desc_of(L, m)
    h = L.ds_hyper(hp.eta, hp.alpha, hp.tau, hp.batch_size, hp.i_max, hp.loss_cut, hp.weight_decay,
                   1 if hp.adaptive else 0)
    X = np.ascontiguousarray(X, np.float32)
    y = np.ascontiguousarray(y, np.uint32)
    init = np.ascontiguousarray(init, np.float32)
    e = C.c_void_p()
    L.check(L.lib.ds_engine_create(C.byref(e), device, C.byref(d), X.ctypes.data, y.ctypes.data, len(y), ncls,
                                   C.byref(h), seed, init.ctypes.data, L.DS_ENGINE_TC if kind is None else kind))
    return e


def engine_log(L, e, first, n):
    loss, cum = np.zeros(n), np.zeros(n)
    ex, per = np.zeros(n, np.uint8), np.zeros(n, np.uint32)
    L.check(L.lib.ds_engine_log(e, first, n, loss.ctypes.data, cum.ctypes.data, ex.ctypes.data, per.ctypes.data))
    return loss, cum, ex, per


def params_of(L, e, P):
    out = np.zeros(P, np.float32)
    L.check(L.lib.ds_engine_get_params(e, out.ctypes.data))
    return out


def rel(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-30))


CASES = [
    ("mlp20-16-3", ModelSpec.mlp(20, [16], 3), 300, Hyper(eta=0.05, tau=5, batch_size=16, i_max=40)),  # 1 CTA
    ("mlp13-33-3", ModelSpec.mlp(13, [33], 3), 300, Hyper(eta=0.05, tau=5, batch_size=16, i_max=40)),  # F odd, 3 CTAs
    ("mlp-wd", ModelSpec.mlp(24, [40], 4), 300, Hyper(eta=0.05, tau=7, batch_size=32, i_max=40, weight_decay=0.01)),
    ("short-batch", ModelSpec.mlp(20, [33], 3), 70, Hyper(eta=0.05, tau=4, batch_size=32, i_max=12)),
    ("mlp784", ModelSpec.mlp(784, [256], 10), 2000, Hyper(eta=0.05, tau=10, batch_size=32, i_max=100)),  # 16 CTAs
]


@pytest.mark.parametrize("name,m,n,hp", CASES, ids=[c[0] for c in CASES])
@pytest.mark.parametrize("master", [None, "lockfree", "locked"])
def test_tc_matches_oracle(L, orc, name, m, n, hp, master):
    sep, sigma = (0.1, 1.0) if m.n_features == 784 else (2.0, 1.5)
    X, y = orc.gen_synthetic(n, m.n_features, m.n_classes, sep, sigma, 3)
    init, master0 = orc.init_params(m, 9), orc.init_params(m, 10)
    P = len(init)
    ref = orc.run_training_loop(m, X, y, m.n_classes, hp, 31, init, 2 if master else 0, master0)
    e = make_engine(L, m, X, y, m.n_classes, hp, 31, init)
    mh = None
    try:
        if master:
            mh = C.c_void_p()
            mode = L.DS_MODE_LOCKED if master == "locked" else L.DS_MODE_LOCKFREE
            L.check(L.lib.ds_master_create(C.byref(mh), 0, P, C.c_float(np.float32(hp.alpha)), mode,
                                           master0.ctypes.data))
            L.check(L.lib.ds_engine_attach_master(e, mh))
        L.check(L.lib.ds_engine_run(e, hp.i_max, 0, None))
        L.check(L.lib.ds_engine_sync(e))
        loss, _, ex, per = engine_log(L, e, 0, hp.i_max)
        assert np.array_equal(ex, ref["exchanged"]) and np.array_equal(per, ref["period_len"])
        assert np.all(np.abs(loss - ref["batch_loss"]) <= LOSS_RTOL * np.abs(ref["batch_loss"]))
        assert rel(params_of(L, e, P), ref["final_params"]) <= PARAM_TOL
        if master:
            snap = np.zeros(P, np.float32)
            L.check(L.lib.ds_master_snapshot(mh, snap.ctypes.data))
            assert rel(snap, ref["master"]) <= PARAM_TOL
            cnt = C.c_uint64()
            L.check(L.lib.ds_master_exchange_count(mh, C.byref(cnt)))
            assert cnt.value == int(ref["exchanged"].sum())
    finally:
        L.lib.ds_engine_destroy(e)
        if mh:
            L.lib.ds_master_destroy(mh)


def test_tc_split_runs_equal_one_run(L, orc):
    """run(30) + run(30) is bit-identical to run(60): the kernel's state round-trips through
    the engine (resident W1 master, policy counters, ping-pong parameter buffers)."""
    m = ModelSpec.mlp(784, [256], 10)
    X, y = orc.gen_synthetic(1500, 784, 10, 0.1, 1.0, 3)
    init, master0 = orc.init_params(m, 9), orc.init_params(m, 10)
    hp = Hyper(eta=0.05, tau=7, batch_size=32, i_max=60)
    out = []
    for chunks in ([60], [30, 30], [13, 40, 7]):
        e = make_engine(L, m, X, y, 10, hp, 31, init)
        mh = C.c_void_p()
        L.check(L.lib.ds_master_create(C.byref(mh), 0, len(init), C.c_float(np.float32(0.1)), L.DS_MODE_LOCKED,
                                       master0.ctypes.data))
        L.check(L.lib.ds_engine_attach_master(e, mh))
        for c in chunks:
            L.check(L.lib.ds_engine_run(e, c, 0, None))
        L.check(L.lib.ds_engine_sync(e))
        snap = np.zeros(len(init), np.float32)
        L.check(L.lib.ds_master_snapshot(mh, snap.ctypes.data))
        out.append((params_of(L, e, len(init)), snap, engine_log(L, e, 0, 60)[0]))
        L.lib.ds_engine_destroy(e)
        L.lib.ds_master_destroy(mh)
    for p, s, lo in out[1:]:
        assert np.array_equal(p, out[0][0]) and np.array_equal(s, out[0][1]) and np.array_equal(lo, out[0][2])


@pytest.mark.parametrize("adaptive", [False, True])
def test_tc_stream_and_host_steps_equal_device_run(L, orc, api, adaptive):
    """Host-fed batches (stream mode, the e2e path; and ds_engine_step_host) give exactly the
    device-resident run's trajectory on the same batches — with the Fixed and the Adaptive
    policy (engine.cpp:35-48, evaluated in the kernel)."""
    m = ModelSpec.mlp(784, [256], 10)
    X, y = orc.gen_synthetic(1000, 784, 10, 0.1, 1.0, 3)
    init = orc.init_params(m, 9)
    P, steps, B = len(init), 120, 32  # the 8-slot host ring is reused 15 times
    hp = Hyper(eta=0.05, tau=10, batch_size=B, i_max=steps)
    if adaptive:
        cut = 3.0 / 20.0 * orc.resolve_loss_cut(m, X, y, 10, Hyper(eta=0.05, tau=10, batch_size=B, i_max=steps,
                                                                    adaptive=True), 31, init)
        hp = Hyper(eta=0.05, tau=10, batch_size=B, i_max=steps, adaptive=True, loss_cut=cut)
    idx, rows = api.sweep_batches(len(y), B, 31, steps)
    e0 = make_engine(L, m, X, y, 10, hp, 31, init)
    L.check(L.lib.ds_engine_run(e0, steps, 0, None))
    L.check(L.lib.ds_engine_sync(e0))
    ref_p, ref_l = params_of(L, e0, P), engine_log(L, e0, 0, steps)[0]
    ref_x = engine_log(L, e0, 0, steps)[2]
    if adaptive:
        assert 1 <= int(ref_x.sum()) < steps // 2
    L.lib.ds_engine_destroy(e0)
    # stream mode with host gathers
    import torch
    e1 = make_engine(L, m, X, y, 10, hp, 31, init)
    with pytest.raises(L.ContractError, match="pinned"):  # the kernel writes the losses directly
        L.check(L.lib.ds_engine_stream_begin(e1, steps, np.zeros(steps).ctypes.data))
    loss_h = torch.zeros(steps, dtype=torch.float64, pin_memory=True)
    Xc, yc = np.ascontiguousarray(X, np.float32), np.ascontiguousarray(y, np.uint32)
    L.check(L.lib.ds_engine_stream_begin(e1, steps, C.c_void_p(loss_h.data_ptr())))
    for s in range(steps):
        ii = np.ascontiguousarray(idx[s, :rows[s]], np.uint32)
        L.check(L.lib.ds_engine_stream_push_rows(e1, Xc.ctypes.data, yc.ctypes.data, ii.ctypes.data, int(rows[s])))
    L.check(L.lib.ds_engine_stream_end(e1))
    assert np.array_equal(params_of(L, e1, P), ref_p) and np.array_equal(engine_log(L, e1, 0, steps)[0], ref_l)
    assert np.array_equal(loss_h.numpy(), ref_l)  # the zero-copy per-step losses
    assert np.array_equal(engine_log(L, e1, 0, steps)[2], ref_x)
    L.lib.ds_engine_destroy(e1)
    # the whole session's pushes in one call (ring reuse: steps >> DS_STREAM_RING), and
    # user-gathered f32 batches through ds_engine_stream_push
    e3 = make_engine(L, m, X, y, 10, hp, 31, init)
    idx_all = np.ascontiguousarray(idx, np.uint32)
    rows_all = np.ascontiguousarray(rows, np.uint32)
    L.check(L.lib.ds_engine_stream_begin(e3, steps, C.c_void_p(loss_h.data_ptr())))
    L.check(L.lib.ds_engine_stream_push_rows_n(e3, Xc.ctypes.data, yc.ctypes.data, idx_all.ctypes.data,
                                               rows_all.ctypes.data, steps))
    L.check(L.lib.ds_engine_stream_end(e3))
    assert np.array_equal(params_of(L, e3, P), ref_p) and np.array_equal(engine_log(L, e3, 0, steps)[0], ref_l)
    L.lib.ds_engine_destroy(e3)
    # the same pushes from a cached bf16 copy of the host shard (row copies instead of casts)
    e5 = make_engine(L, m, X, y, 10, hp, 31, init)
    L.check(L.lib.ds_engine_stream_cache_host_shard(e5, Xc.ctypes.data, len(yc)))
    L.check(L.lib.ds_engine_stream_begin(e5, steps, C.c_void_p(loss_h.data_ptr())))
    with pytest.raises(L.StateError, match="stream is open"):  # the pushes may be reading the copy
        L.check(L.lib.ds_engine_stream_cache_host_shard(e5, Xc.ctypes.data, len(yc)))
    L.check(L.lib.ds_engine_stream_push_rows_n(e5, Xc.ctypes.data, yc.ctypes.data, idx_all.ctypes.data,
                                               rows_all.ctypes.data, steps))
    L.check(L.lib.ds_engine_stream_end(e5))
    assert np.array_equal(params_of(L, e5, P), ref_p) and np.array_equal(engine_log(L, e5, 0, steps)[0], ref_l)
    L.check(L.lib.ds_engine_stream_cache_host_shard(e5, None, 0))
    L.lib.ds_engine_destroy(e5)
    e4 = make_engine(L, m, X, y, 10, hp, 31, init)
    L.check(L.lib.ds_engine_stream_begin(e4, steps, C.c_void_p(loss_h.data_ptr())))
    keep = []
    for s in range(steps):
        xb = np.ascontiguousarray(X[idx[s, :rows[s]]], np.float32)
        yb = np.ascontiguousarray(y[idx[s, :rows[s]]], np.uint32)
        keep.append((xb, yb))
        L.check(L.lib.ds_engine_stream_push(e4, xb.ctypes.data, yb.ctypes.data, int(rows[s])))
    L.check(L.lib.ds_engine_stream_end(e4))
    assert np.array_equal(params_of(L, e4, P), ref_p) and np.array_equal(engine_log(L, e4, 0, steps)[0], ref_l)
    L.lib.ds_engine_destroy(e4)
    # one host step at a time
    e2 = make_engine(L, m, X, y, 10, hp, 31, init)
    for s in range(steps):
        xb = np.ascontiguousarray(X[idx[s, :rows[s]]], np.float32)
        yb = np.ascontiguousarray(y[idx[s, :rows[s]]], np.uint32)
        L.check(L.lib.ds_engine_step_host(e2, xb.ctypes.data, yb.ctypes.data, int(rows[s]), None))
    L.check(L.lib.ds_engine_sync(e2))
    assert np.array_equal(params_of(L, e2, P), ref_p) and np.array_equal(engine_log(L, e2, 0, steps)[0], ref_l)
    L.lib.ds_engine_destroy(e2)


def _config1(orc, api, n_workers, i_max, data_seed=3, init_seed=2):
    from paper_1602_08191_b200 import dist as D
    m = ModelSpec.mlp(784, [256], 10)
    X, y = orc.gen_synthetic(6000, 784, 10, 0.1, 1.0, 1)
    hp = Hyper(eta=0.05, alpha=0.1, tau=10, batch_size=32, i_max=i_max)
    shards, hold = D.sim_shards(api, X, y, n_workers, 0.2, data_seed)
    seeds = [D.sweep_seed(api, data_seed, k) for k in range(n_workers)]
    return m, X, y, hp, shards, hold, seeds, orc.init_params(m, init_seed)


def _run_group(L, api, m, hp, shards, seeds, init, mode, n_slices=1, tickets=None):
    """n workers (one engine each) in ONE launch against one center (optionally split into
    n_slices shards on this GPU). Returns (center, worker params, exchange count)."""
    from paper_1602_08191_b200 import dist as D
    P = len(init)
    masters = []
    if n_slices == 1:
        mh = C.c_void_p()
        L.check(L.lib.ds_master_create(C.byref(mh), 0, P, C.c_float(np.float32(hp.alpha)), mode, init.ctypes.data))
        masters = [mh]
    else:  # one slice per emulated rank, all on device 0 (in-process attach)
        for k in range(n_slices):
            mh = C.c_void_p()
            L.check(L.lib.ds_master_create_sharded(C.byref(mh), 0, P, C.c_float(np.float32(hp.alpha)), mode, k,
                                                   n_slices, init.ctypes.data))
            masters.append(mh)
        recs = b""
        for mh in masters:
            rec = (C.c_uint8 * L.DS_IPC_RECORD_BYTES)()
            L.check(L.lib.ds_master_export(mh, rec))
            recs += bytes(rec)
        allrec = (C.c_uint8 * len(recs)).from_buffer_copy(recs)
        for mh in masters:
            L.check(L.lib.ds_master_attach(mh, allrec))
    engines = []
    try:
        for k, (Xk, yk) in enumerate(shards):
            e = make_engine(L, m, Xk, yk, 10, hp, seeds[k], init)
            L.check(L.lib.ds_engine_attach_master(e, masters[k % len(masters)]))
            if tickets is not None:
                tk = D.worker_tickets(tickets, k)
                L.check(L.lib.ds_engine_set_tickets(e, tk.ctypes.data, len(tk)))
            engines.append(e)
        arr = (C.c_void_p * len(engines))(*[e.value for e in engines])
        L.check(L.lib.ds_engine_run_group(arr, len(engines), hp.i_max))
        for e in engines:
            L.check(L.lib.ds_engine_sync(e))
        snap = np.zeros(P, np.float32)
        L.check(L.lib.ds_master_snapshot(masters[0], snap.ctypes.data))
        cnt = C.c_uint64()
        L.check(L.lib.ds_master_exchange_count(masters[0], C.byref(cnt)))
        workers = [params_of(L, e, P) for e in engines]
        return snap, workers, int(cnt.value)
    finally:
        for e in engines:
            L.lib.ds_engine_destroy(e)
        for mh in masters:
            L.lib.ds_master_destroy(mh)


@pytest.mark.parametrize("n_slices", [1, 2])
def test_tc_group_deterministic_config1(L, orc, api, n_slices):
    """BASELINE config 1 (784-256-10, 2 workers, tau=10, alpha=0.1) in deterministic mode on
    ONE GPU: both workers in one launch, exchanges serialized by the tickets of the
    replayed simulate_async order (simulator.cpp:91-143). Center and workers within the bf16
    tolerance of the oracle's simulate; exact exchange count; bit-identical on a rerun and
    with the center split into two shards (the sharded exchange path, one GPU)."""
    m, X, y, hp, shards, hold, seeds, init = _config1(orc, api, 2, 120)
    order_w, _ = api.exchange_order(2, hp.tau, hp.i_max, 1)
    ref = orc.simulate(SimSpec(2, hp, m, X, y, 10, schedule_seed=1, init_seed=2, data_seed=3,
                               eval_every=10 ** 6, record_master_snaps=False))
    a = _run_group(L, api, m, hp, shards, seeds, init, L.DS_MODE_LOCKED, n_slices, order_w)
    b = _run_group(L, api, m, hp, shards, seeds, init, L.DS_MODE_LOCKED, n_slices, order_w)
    assert a[2] == 2 * (hp.i_max // hp.tau)
    assert rel(a[0], ref.final_master) <= PARAM_TOL
    for k in range(2):
        assert rel(a[1][k], ref.worker_final[k]) <= PARAM_TOL
    assert np.array_equal(a[0], b[0]) and all(np.array_equal(p, q) for p, q in zip(a[1], b[1]))
    if n_slices == 2:  # the same arithmetic per element as one slice: bit-identical
        c = _run_group(L, api, m, hp, shards, seeds, init, L.DS_MODE_LOCKED, 1, order_w)
        assert np.array_equal(a[0], c[0])


@pytest.mark.parametrize("mode,n_slices", [("locked", 1), ("locked", 2), ("lockfree", 1), ("lockfree", 2)])
def test_tc_group_async_band_config1(L, orc, api, mode, n_slices):
    """Async EASGD on BASELINE config 1: the two workers train CONCURRENTLY in one launch and
    exchange whenever their policy fires, in arrival order (no precomputed schedule).
    After 120 iterations (1.6 epochs per worker; holdout accuracy ~0.92, not saturated) the
    center's holdout accuracy and loss are compared with the reference simulate's
    (simulator.cpp:138-142 evaluation).

    * Locked (exchanges serialized in arrival order by the device ticket dispenser, the
      reference's UpdateMode::Locked): |d acc| <= 0.02 and |d loss| <= 3% relative.
    * LockFree (UpdateMode::LockFree: no ordering): the two workers run in lockstep on one
      GPU, so their exchanges overlap. The center's increments are f32 atomic adds (bulk
      TMA reductions for a one-GPU center), so overlapping exchanges add up rather than
      overwrite each other (a lone writer gets exactly m + e) — measured: accuracy 0.920 vs
      0.918, holdout loss within 2%. Same band as Locked."""
    m, X, y, hp, shards, hold, seeds, init = _config1(orc, api, 2, 120)
    ref = orc.simulate(SimSpec(2, hp, m, X, y, 10, schedule_seed=1, init_seed=2, data_seed=3,
                               eval_every=10 ** 6, record_master_snaps=False))
    md = L.DS_MODE_LOCKED if mode == "locked" else L.DS_MODE_LOCKFREE
    snap, workers, cnt = _run_group(L, api, m, hp, shards, seeds, init, md, n_slices)
    Xh, yh = hold
    acc_ref, acc_dev = orc.accuracy(m, ref.final_master, Xh, yh, 10), orc.accuracy(m, snap, Xh, yh, 10)
    loss_ref = orc.loss_and_grad(m, ref.final_master, Xh, yh, want_grad=False)[0]
    loss_dev = orc.loss_and_grad(m, snap, Xh, yh, want_grad=False)[0]
    print(f"async band ({mode}, {n_slices} slice(s)): acc {acc_dev:.4f} vs {acc_ref:.4f}, "
          f"holdout loss {loss_dev:.5f} vs {loss_ref:.5f}")
    assert cnt == 2 * (hp.i_max // hp.tau) and np.isfinite(snap).all()
    assert 0.8 <= acc_ref <= 0.97  # the band is tested away from saturation
    assert abs(acc_dev - acc_ref) <= 0.02
    assert abs(loss_dev - loss_ref) <= 0.03 * loss_ref


def test_tc_errors(L, orc):
    m = ModelSpec.mlp(20, [16], 3)
    X, y = orc.gen_synthetic(300, 20, 3, 2.0, 1.5, 3)
    init = orc.init_params(m, 9)
    hp = Hyper(eta=0.05, tau=5, batch_size=16, i_max=10)
    # the bf16 host-shard cache: contract errors on a null engine / a non-tensor-core engine;
    # dropping a cache that does not exist is a no-op
    with pytest.raises(L.ContractError):
        L.check(L.lib.ds_engine_stream_cache_host_shard(None, X.ctypes.data, len(y)))
    e = make_engine(L, m, X, y, 3, hp, 31, init, kind=L.DS_ENGINE_FUSED)
    try:
        with pytest.raises(L.ContractError, match="tensor-core"):
            L.check(L.lib.ds_engine_stream_cache_host_shard(e, X.ctypes.data, len(y)))
        L.check(L.lib.ds_engine_stream_cache_host_shard(e, None, 0))
    finally:
        L.lib.ds_engine_destroy(e)
    e = make_engine(L, m, X, y, 3, hp, 31, init)
    try:  # a host-fed batch with a label out of range, caught in the kernel (model.cpp:176-180)
        xb = np.ascontiguousarray(X[:16], np.float32)
        yb = np.full(16, 7, np.uint32)
        L.check(L.lib.ds_engine_step_host(e, xb.ctypes.data, yb.ctypes.data, 16, None))
        with pytest.raises(L.ContractError, match="label"):
            L.check(L.lib.ds_engine_sync(e))
    finally:
        L.lib.ds_engine_destroy(e)
    # a non-finite batch makes the loss non-finite (model.cpp:256): NumericError
    e = make_engine(L, m, X, y, 3, hp, 31, init)
    try:
        xb = np.full((16, 20), np.nan, np.float32)
        yb = np.ascontiguousarray(y[:16], np.uint32)
        L.check(L.lib.ds_engine_step_host(e, xb.ctypes.data, yb.ctypes.data, 16, None))
        with pytest.raises(L.NumericError):
            L.check(L.lib.ds_engine_sync(e))
    finally:
        L.lib.ds_engine_destroy(e)
    # an update that overflows f32 (huge weights, weight decay folded in): NumericError
    hp_big = Hyper(eta=5.0, tau=5, batch_size=16, i_max=10, weight_decay=1.0)
    e = make_engine(L, m, X, y, 3, hp_big, 31, (init * np.float32(1e37)).astype(np.float32))
    try:
        L.check(L.lib.ds_engine_run(e, 10, 0, None))
        with pytest.raises(L.NumericError):
            L.check(L.lib.ds_engine_sync(e))
    finally:
        L.lib.ds_engine_destroy(e)
    # models the tensor-core step does not cover are refused, not run another way
    with pytest.raises(L.ContractError):
        make_engine(L, ModelSpec.mlp(12, [8, 6], 4), *orc.gen_synthetic(100, 12, 4, 2.0, 1.5, 3), 4,
                    Hyper(eta=0.05, tau=5, batch_size=16, i_max=10), 31, orc.init_params(ModelSpec.mlp(12, [8, 6], 4), 9))
