"""Red-zone checks of the C-ABI kernels that write caller buffers (compute-sanitizer is
closed on the GPU pool; this is the memcheck substitute for out-of-bounds writes).

Every output vector sits inside a larger allocation at an unaligned offset, the guard
floats on both sides hold a NaN pattern, and after the call the guards must be intact
while the payload is correct. Sizes cover the scalar tails and vector bodies of the
grid-stride loops (1, 3, 33, 4099, 1000003)."""
import ctypes as C

import numpy as np
import pytest

from oracle.oracle import Oracle

pytestmark = pytest.mark.gpu
GUARD = 64
SENT = np.uint32(0x7FC0DEAD)


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1602_08191_b200 import _lib as L
    from paper_1602_08191_b200 import dist as D
    return torch, L, D, Oracle("dso")


class Zoned:
    """n floats at offset `off` (floats) inside a guarded device allocation."""

    def __init__(self, torch, n, off, init=None):
        self.n, self.off = n, off
        host = np.full(n + 2 * GUARD + off, SENT, np.uint32)
        if init is not None:
            host[GUARD + off:GUARD + off + n] = np.asarray(init, np.float32).view(np.uint32)
        self.t = torch.from_numpy(host.view(np.int32)).cuda()

    @property
    def ptr(self):
        return C.c_void_p(self.t.data_ptr() + 4 * (GUARD + self.off))

    def payload(self):
        return self.t.cpu().numpy().view(np.uint32)[GUARD + self.off:GUARD + self.off + self.n].view(np.float32)

    def guards_ok(self):
        h = self.t.cpu().numpy().view(np.uint32)
        return bool((h[:GUARD + self.off] == SENT).all() and (h[GUARD + self.off + self.n:] == SENT).all())


SIZES = [1, 3, 33, 4099, 1000003]


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("off", [0, 1, 3])
def test_elastic_and_sgd_stay_in_bounds(env, n, off):
    torch, L, D, orc = env
    rng = np.random.default_rng(n + off)
    w, m, g = (rng.standard_normal(n).astype(np.float32) for _ in range(3))
    wz, mz, gz, oz = Zoned(torch, n, off, w), Zoned(torch, n, off + 1, m), Zoned(torch, n, off, g), Zoned(torch, n, off + 2)
    L.check(L.lib.ds_elastic_update(wz.ptr, mz.ptr, n, C.c_float(0.1), None))
    L.check(L.lib.ds_sgd_step_checked(oz.ptr, wz.ptr, gz.ptr, n, 0.05, None))
    torch.cuda.synchronize()
    ew, em = orc.easgd_update(w, m, 0.1)
    assert np.array_equal(wz.payload().view(np.uint32), ew.view(np.uint32))
    assert np.array_equal(mz.payload().view(np.uint32), em.view(np.uint32))
    assert np.array_equal(oz.payload().view(np.uint32), orc.sgd_step(ew, g, 0.05).view(np.uint32))
    assert all(z.guards_ok() for z in (wz, mz, gz, oz))


@pytest.mark.parametrize("n", SIZES)
def test_master_exchange_stays_in_bounds(env, n):
    torch, L, D, orc = env
    rng = np.random.default_rng(n)
    m0, w = rng.standard_normal(n).astype(np.float32), rng.standard_normal(n).astype(np.float32)
    for mode in (L.DS_MODE_LOCKED, L.DS_MODE_LOCKFREE):
        wz, oz = Zoned(torch, n, 1, w), Zoned(torch, n, 3)
        h = C.c_void_p()
        L.check(L.lib.ds_master_create(C.byref(h), 0, n, C.c_float(0.1), mode, m0.ctypes.data))
        try:
            L.check(L.lib.ds_master_exchange(h, wz.ptr, oz.ptr, None))
            torch.cuda.synchronize()
        finally:
            L.lib.ds_master_destroy(h)
        ew, _ = orc.easgd_update(w, m0, 0.1)
        assert np.array_equal(oz.payload().view(np.uint32), ew.view(np.uint32))
        assert wz.guards_ok() and oz.guards_ok()


@pytest.mark.parametrize("n", SIZES)
def test_sync_group_stays_in_bounds(env, n):
    torch, L, D, orc = env
    world = 3
    rng = np.random.default_rng(n + 7)
    x0 = rng.standard_normal(n).astype(np.float32)
    grads = [rng.standard_normal(n).astype(np.float32) for _ in range(world)]
    reps = [Zoned(torch, n, k, x0) for k in range(world)]  # offsets 0, 1, 2: vector and scalar paths
    syncs = D.local_sync_group(L, 0, n, world)
    flags = torch.zeros(1, dtype=torch.int32, device="cuda")
    try:
        for k in range(world):
            slot = C.c_void_p()
            L.check(L.lib.ds_sync_begin(syncs[k], C.byref(slot), None))
            L.check(L.lib.ds_memcpy(slot, grads[k].ctypes.data, 4 * n, None))
        group = (C.c_void_p * world)(*[s.value for s in syncs])
        preps = (C.c_void_p * world)(*[r.ptr.value for r in reps])
        L.check(L.lib.ds_sync_reduce_update_group(group, world, preps, C.c_float(0.05), C.c_float(0.0),
                                                  C.c_void_p(flags.data_ptr()), None))
        works = [Zoned(torch, n, 2 - k, x0 + 0.5) for k in range(world)]
        pw = (C.c_void_p * world)(*[w.ptr.value for w in works])
        L.check(L.lib.ds_sync_easgd_update_group(group, world, pw, preps, C.c_float(0.2),
                                                 C.c_void_p(flags.data_ptr()), None))
        torch.cuda.synchronize()
    finally:
        for s in syncs:
            L.lib.ds_sync_destroy(s)
    assert int(flags.item()) == 0
    x1 = orc.sync_sgd_round(x0, grads, 0.05)
    xs, c2 = orc.sync_easgd_round([(x0 + 0.5).astype(np.float32)] * world, x1, 0.2)
    for r in reps:
        assert r.guards_ok() and np.array_equal(r.payload().view(np.uint32), c2.view(np.uint32))
    for k, w in enumerate(works):
        assert w.guards_ok() and np.array_equal(w.payload().view(np.uint32), xs[k].view(np.uint32))


@pytest.mark.parametrize("rows,F", [(1, 1), (7, 33), (32, 784)])
def test_gather_rows_stays_in_bounds(env, rows, F):
    torch, L, D, orc = env
    N = 100
    rng = np.random.default_rng(rows * F)
    X = rng.standard_normal((N, F)).astype(np.float32)
    y = rng.integers(0, 10, N).astype(np.uint32)
    idx = rng.integers(0, N, rows).astype(np.uint32)
    Xd = torch.from_numpy(X).cuda()
    yd = torch.from_numpy(y.view(np.int32)).cuda()
    idd = torch.from_numpy(idx.view(np.int32)).cuda()
    bx, by = Zoned(torch, rows * F, 1), Zoned(torch, rows, 3)
    L.check(L.lib.ds_gather_rows(bx.ptr, by.ptr, C.c_void_p(Xd.data_ptr()), C.c_void_p(yd.data_ptr()),
                                 C.c_void_p(idd.data_ptr()), rows, F, None))
    torch.cuda.synchronize()
    assert np.array_equal(bx.payload().reshape(rows, F), X[idx])
    assert np.array_equal(by.payload().view(np.uint32), y[idx])
    assert bx.guards_ok() and by.guards_ok()
