"""Bit-exactness of the elementwise hot kernels at the sizes the bench runs (SURVEY §7
gate 1: 1M-500M elements), where the grid-stride loops take many passes and the float4
bodies dominate:

* ds_elastic_update (the exchange leg's kernel, 256M in bench.py) at 64M and 500M;
* ds_master_exchange (exchange_kernel, single-device and two-shard LockFree) at 64M;
* ds_sgd_step_checked at 64M and 500M.

Inputs are generated on the device; the CPU oracle (oracle/ds_oracle.c) checks the
results in 32M-element chunks so host memory stays bounded.
"""
import ctypes as C

import numpy as np
import pytest

from oracle.oracle import Oracle

pytestmark = pytest.mark.gpu
CHUNK = 32 << 20


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1602_08191_b200 import _lib as L
    return torch, L, Oracle("dso")


def _need(torch, nbytes):
    free, _ = torch.cuda.mem_get_info()
    if free < nbytes:
        pytest.skip(f"needs {nbytes / 2**30:.1f} GiB free on the device")


def _mixed(torch, n, seed):
    """normal values with a spread of magnitudes (products and differences that round)."""
    g = torch.Generator(device="cuda").manual_seed(seed)
    v = torch.randn(n, device="cuda", generator=g)
    scale = torch.exp2(torch.randint(-20, 21, (n,), device="cuda", generator=g).float())
    return v.mul_(scale)


def _chunks(n):
    for a in range(0, n, CHUNK):
        yield a, min(n, a + CHUNK)


@pytest.mark.parametrize("n", [64 << 20, 500_000_000])
def test_elastic_update_bit_exact_large(env, n):
    torch, L, orc = env
    _need(torch, 4 * n * 2 + (2 << 30))
    w = _mixed(torch, n, 1)
    m = _mixed(torch, n, 2)
    w0, m0 = w.cpu(), m.cpu()  # pageable host copies of the inputs
    alpha = np.float32(0.1)
    L.check(L.lib.ds_elastic_update(C.c_void_p(w.data_ptr()), C.c_void_p(m.data_ptr()), n, C.c_float(alpha), None))
    torch.cuda.synchronize()
    for a, b in _chunks(n):
        ew, em = orc.easgd_update(w0[a:b].numpy(), m0[a:b].numpy(), float(alpha))
        assert np.array_equal(w[a:b].cpu().numpy().view(np.uint32), ew.view(np.uint32)), f"w chunk {a}"
        assert np.array_equal(m[a:b].cpu().numpy().view(np.uint32), em.view(np.uint32)), f"m chunk {a}"


@pytest.mark.parametrize("shards", [1, 2])
def test_master_exchange_bit_exact_large(env, shards):
    torch, L, orc = env
    n = 64 << 20
    _need(torch, 4 * n * 3 + (2 << 30))
    w = _mixed(torch, n, 3)
    m0 = _mixed(torch, n, 4)
    out = torch.empty_like(w)
    hs = []
    try:
        if shards == 1:
            h = C.c_void_p()
            L.check(L.lib.ds_master_create(C.byref(h), 0, n, C.c_float(0.1), L.DS_MODE_LOCKFREE,
                                           C.c_void_p(m0.data_ptr())))
            hs.append(h)
        else:
            recs = []
            for r in range(shards):
                h = C.c_void_p()
                L.check(L.lib.ds_master_create_sharded(C.byref(h), 0, n, C.c_float(0.1), L.DS_MODE_LOCKFREE, r,
                                                       shards, C.c_void_p(m0.data_ptr())))
                rec = (C.c_uint8 * L.DS_IPC_RECORD_BYTES)()
                L.check(L.lib.ds_master_export(h, rec))
                hs.append(h)
                recs.append(bytes(rec))
            allrec = (C.c_uint8 * (shards * L.DS_IPC_RECORD_BYTES)).from_buffer_copy(b"".join(recs))
            for h in hs:
                L.check(L.lib.ds_master_attach(h, allrec))
        L.check(L.lib.ds_master_exchange(hs[0], C.c_void_p(w.data_ptr()), C.c_void_p(out.data_ptr()), None))
        torch.cuda.synchronize()
        got_m = np.zeros(n, np.float32)
        L.check(L.lib.ds_master_snapshot(hs[0], got_m.ctypes.data))
    finally:
        for h in hs:
            L.lib.ds_master_destroy(h)
    wh, mh = w.cpu().numpy(), m0.cpu().numpy()
    for a, b in _chunks(n):
        ew, em = orc.easgd_update(wh[a:b], mh[a:b], 0.1)
        assert np.array_equal(out[a:b].cpu().numpy().view(np.uint32), ew.view(np.uint32)), f"w chunk {a}"
        assert np.array_equal(got_m[a:b].view(np.uint32), em.view(np.uint32)), f"m chunk {a}"


@pytest.mark.parametrize("n", [64 << 20, 500_000_000])
def test_sgd_step_bit_exact_large(env, n):
    torch, L, orc = env
    _need(torch, 4 * n * 3 + (2 << 30))
    x = _mixed(torch, n, 5)
    g = torch.randn(n, device="cuda", generator=torch.Generator(device="cuda").manual_seed(6))
    out = torch.empty_like(x)
    eta = 0.013
    L.check(L.lib.ds_sgd_step_checked(C.c_void_p(out.data_ptr()), C.c_void_p(x.data_ptr()),
                                      C.c_void_p(g.data_ptr()), n, eta, None))
    torch.cuda.synchronize()
    for a, b in _chunks(n):
        e = orc.sgd_step(x[a:b].cpu().numpy(), g[a:b].cpu().numpy(), eta)
        assert np.array_equal(out[a:b].cpu().numpy().view(np.uint32), e.view(np.uint32)), f"chunk {a}"
