"""The device center's concurrency contract on ONE GPU, through the product C-ABI.

The reference's exchanger properties (test_exchanger.cpp), restated for a device center
that host threads drive concurrently, each on its own CUDA stream:

* concurrent Locked exchanges == SOME serialization, bit for bit (test_exchanger.cpp:168-193):
  the single-device Locked master serializes on its own stream; the sharded master (two
  shards of one GPU, one handle per "rank") orders by the device ticket dispenser;
* deterministic tickets enqueued out of order still apply in ticket order
  (simulator.cpp:105-143's serialization, here without a second GPU);
* LockFree with a single writer is bit-identical to Locked (test_exchanger.cpp:228-242);
* concurrent LockFree writers stay finite and inside the per-element hull of everything
  ever sent (test_exchanger.cpp:244-290), at the reference's dim 4 and at 1M elements
  where the kernels really interleave;
* snapshot / exchange_count wait only for the master's client streams (no device-wide
  synchronize): an unrelated stream blocked on a host-side event does not stall them.
"""
import ctypes as C
import itertools
import threading

import numpy as np
import pytest

from oracle.oracle import Oracle

pytestmark = pytest.mark.gpu
ALPHA = 0.1


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1602_08191_b200 import _lib as L
    return torch, L, Oracle("dso")


def _vecs(n, dim, seed):
    rng = np.random.default_rng(seed)
    return [(rng.standard_normal(dim) * (k + 1)).astype(np.float32) for k in range(n)]


def _replay(orc, m0, workers, order):
    m = m0.copy()
    for k in order:
        _, m = orc.easgd_update(workers[k], m, ALPHA)
    return m


def _master(L, dim, mode, init):
    m = C.c_void_p()
    L.check(L.lib.ds_master_create(C.byref(m), 0, dim, C.c_float(ALPHA), mode, init.ctypes.data))
    return m


def _sharded(L, dim, mode, init, n=3):
    """n shards of one center on cuda:0, one handle (and master stream) per 'rank',
    attached to each other."""
    hs, recs = [], []
    for r in range(n):
        h = C.c_void_p()
        L.check(L.lib.ds_master_create_sharded(C.byref(h), 0, dim, C.c_float(ALPHA), mode, r, n,
                                               C.c_void_p(init.ctypes.data)))
        rec = (C.c_uint8 * L.DS_IPC_RECORD_BYTES)()
        L.check(L.lib.ds_master_export(h, rec))
        hs.append(h)
        recs.append(bytes(rec))
    allrec = (C.c_uint8 * (n * L.DS_IPC_RECORD_BYTES)).from_buffer_copy(b"".join(recs))
    for h in hs:
        L.check(L.lib.ds_master_attach(h, allrec))
    return hs


def _run_threads(fns):
    errs = []

    def wrap(f):
        try:
            f()
        except Exception as e:  # noqa: BLE001 - surfaced below
            errs.append(e)
    ts = [threading.Thread(target=wrap, args=(f,)) for f in fns]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if errs:
        raise errs[0]


@pytest.mark.parametrize("dim", [6, 100_003])
@pytest.mark.parametrize("sharded", [False, True])
def test_locked_concurrent_matches_some_serialization(env, dim, sharded):
    torch, L, orc = env
    m0 = _vecs(1, dim, 99)[0]
    workers = _vecs(3, dim, dim)
    handles = _sharded(L, dim, L.DS_MODE_LOCKED, m0) if sharded else [_master(L, dim, L.DS_MODE_LOCKED, m0)]
    streams = [torch.cuda.Stream() for _ in range(3)]
    bufs = [torch.from_numpy(w).cuda() for w in workers]
    torch.cuda.synchronize()
    outs = [torch.empty_like(b) for b in bufs]

    def go(k):
        h = handles[k % len(handles)]
        L.check(L.lib.ds_master_exchange(h, C.c_void_p(bufs[k].data_ptr()), C.c_void_p(outs[k].data_ptr()),
                                         C.c_void_p(streams[k].cuda_stream)))
    try:
        _run_threads([lambda k=k: go(k) for k in range(3)])
        for s in streams:
            s.synchronize()
        got = np.zeros(dim, np.float32)
        L.check(L.lib.ds_master_snapshot(handles[0], got.ctypes.data))
        cnt = C.c_uint64()
        L.check(L.lib.ds_master_exchange_count(handles[0], C.byref(cnt)))
        assert cnt.value == 3
    finally:
        for h in handles:
            L.lib.ds_master_destroy(h)
    matched = None
    for order in itertools.permutations(range(3)):
        if np.array_equal(got.view(np.uint32), _replay(orc, m0, workers, order).view(np.uint32)):
            matched = order
            break
    assert matched is not None, "the center is not any serialization of the three exchanges"
    # each worker got back w - alpha (w - m_before) for the center it saw in that order
    m = m0.copy()
    for k in matched:
        w_exp, m = orc.easgd_update(workers[k], m, ALPHA)
        assert np.array_equal(outs[k].cpu().numpy().view(np.uint32), w_exp.view(np.uint32))


@pytest.mark.parametrize("sharded", [False, True])
def test_tickets_out_of_order_apply_in_ticket_order(env, sharded):
    torch, L, orc = env
    dim = 1000  # one CTA per shard: the waiting kernels never crowd out the ones they wait for
    m0 = _vecs(1, dim, 5)[0]
    workers = _vecs(3, dim, 6)
    handles = _sharded(L, dim, L.DS_MODE_LOCKED, m0) if sharded else [_master(L, dim, L.DS_MODE_LOCKED, m0)]
    streams = [torch.cuda.Stream() for _ in range(3)]
    bufs = [torch.from_numpy(w).cuda() for w in workers]
    torch.cuda.synchronize()
    tickets = [2, 0, 1]  # worker k's global exchange number
    try:
        if sharded:  # ticket 2 first, then 1, then 0, each on its own handle's stream: the
            # device-side seq waits order them
            for k in sorted(range(3), key=lambda k: -tickets[k]):
                L.check(L.lib.ds_master_exchange_ticketed(handles[k], C.c_void_p(bufs[k].data_ptr()),
                                                          C.c_void_p(bufs[k].data_ptr()), tickets[k],
                                                          C.c_void_p(streams[k].cuda_stream)))
        else:  # host threads race; the single-device master admits them in ticket order
            _run_threads([lambda k=k: L.check(L.lib.ds_master_exchange_ticketed(
                handles[0], C.c_void_p(bufs[k].data_ptr()), C.c_void_p(bufs[k].data_ptr()), tickets[k],
                C.c_void_p(streams[k].cuda_stream))) for k in range(3)])
        for s in streams:
            s.synchronize()
        got = np.zeros(dim, np.float32)
        L.check(L.lib.ds_master_snapshot(handles[0], got.ctypes.data))
    finally:
        for h in handles:
            L.lib.ds_master_destroy(h)
    order = sorted(range(3), key=lambda k: tickets[k])
    assert np.array_equal(got.view(np.uint32), _replay(orc, m0, workers, order).view(np.uint32))


def test_lockfree_single_writer_equals_locked(env):
    torch, L, orc = env
    dim = 4099
    m0 = _vecs(1, dim, 1)[0]
    sent = _vecs(4, dim, 2)
    results = []
    for mode in (L.DS_MODE_LOCKED, L.DS_MODE_LOCKFREE):
        h = _master(L, dim, mode, m0)
        try:
            for w in sent:
                b = torch.from_numpy(w).cuda()
                L.check(L.lib.ds_master_exchange(h, C.c_void_p(b.data_ptr()), C.c_void_p(b.data_ptr()), None))
            got = np.zeros(dim, np.float32)
            L.check(L.lib.ds_master_snapshot(h, got.ctypes.data))
            cnt = C.c_uint64()
            L.check(L.lib.ds_master_exchange_count(h, C.byref(cnt)))
            assert cnt.value == 4
        finally:
            L.lib.ds_master_destroy(h)
        results.append(got)
    assert np.array_equal(results[0].view(np.uint32), results[1].view(np.uint32))
    assert np.array_equal(results[0].view(np.uint32), _replay(orc, m0, sent, range(4)).view(np.uint32))


@pytest.mark.parametrize("dim", [4, 1 << 20])
def test_lockfree_concurrent_stays_in_hull(env, dim):
    torch, L, orc = env
    writers, rounds = 4, 50
    m0 = _vecs(1, dim, 11)[0]
    sent = _vecs(writers, dim, 12)
    h = _master(L, dim, L.DS_MODE_LOCKFREE, m0)
    streams = [torch.cuda.Stream() for _ in range(writers)]
    bufs = [torch.from_numpy(w).cuda() for w in sent]
    torch.cuda.synchronize()

    def go(k):
        st = C.c_void_p(streams[k].cuda_stream)
        for _ in range(rounds):  # w = client.exchange(w)
            L.check(L.lib.ds_master_exchange(h, C.c_void_p(bufs[k].data_ptr()), C.c_void_p(bufs[k].data_ptr()), st))
    try:
        _run_threads([lambda k=k: go(k) for k in range(writers)])
        got = np.zeros(dim, np.float32)
        L.check(L.lib.ds_master_snapshot(h, got.ctypes.data))  # waits for the client streams
        cnt = C.c_uint64()
        L.check(L.lib.ds_master_exchange_count(h, C.byref(cnt)))
        # the count is one relaxed increment per exchange kernel: exact
        assert cnt.value == writers * rounds
    finally:
        L.lib.ds_master_destroy(h)
    assert np.isfinite(got).all()
    allv = np.stack([m0] + sent).astype(np.float64)
    lo, hi = allv.min(0), allv.max(0)
    slack = 1e-5 * np.maximum(1.0, np.maximum(np.abs(lo), np.abs(hi)))
    assert (got >= lo - slack).all() and (got <= hi + slack).all()
    big_m = np.abs(np.stack(sent)).max()
    assert (np.abs(got.astype(np.float64) - m0) <= ALPHA * 2.0 * big_m * writers * rounds).all()
    for b in bufs:  # the workers' returned vectors are blends too
        wv = b.cpu().numpy()
        assert np.isfinite(wv).all() and (wv >= lo - slack).all() and (wv <= hi + slack).all()


def test_snapshot_does_not_wait_for_unrelated_streams(env):
    """Another component's busy stream must not block the master's snapshot or count
    (round 1 used cudaDeviceSynchronize there)."""
    import time
    torch, L, orc = env
    dim = 1000
    m0 = _vecs(1, dim, 3)[0]
    w0 = _vecs(1, dim, 4)[0]
    h = _master(L, dim, L.DS_MODE_LOCKFREE, m0)
    mine, other = torch.cuda.Stream(), torch.cuda.Stream()
    try:
        w = torch.from_numpy(w0).cuda()
        torch.cuda.synchronize()
        L.check(L.lib.ds_master_exchange(h, C.c_void_p(w.data_ptr()), C.c_void_p(w.data_ptr()),
                                         C.c_void_p(mine.cuda_stream)))
        with torch.cuda.stream(other):  # ~2 s of device sleeps on an unrelated stream
            for _ in range(20):
                torch.cuda._sleep(200_000_000)
        t0 = time.perf_counter()
        got = np.zeros(dim, np.float32)
        L.check(L.lib.ds_master_snapshot(h, got.ctypes.data))
        cnt = C.c_uint64()
        L.check(L.lib.ds_master_exchange_count(h, C.byref(cnt)))
        dt = time.perf_counter() - t0
        other_busy = not other.query()
        other.synchronize()
        assert other_busy, "the unrelated stream finished before the snapshot; the check proves nothing"
        assert dt < 0.5 and cnt.value == 1
        _, m1 = orc.easgd_update(w0, m0, ALPHA)
        assert np.array_equal(got.view(np.uint32), m1.view(np.uint32))
    finally:
        L.lib.ds_master_destroy(h)
