"""GPU parity of the C-ABI kernels against the CPU oracle (oracle/ds_oracle.c).

Bar: the elastic and SGD updates are bit-exact (pure f32 arithmetic
with the reference's rounding points). loss_and_grad is the reference's f64 algorithm
in the same per-element order; only CUDA's double tanh/exp/log differ from glibc's, so
the f32 gradients are compared bit-exact with a tolerance of at most 1 ulp on a tiny
fraction of elements, and the f64 loss to 1e-15 relative.
"""
import ctypes as C

import numpy as np
import pytest

from oracle.oracle import Oracle, ModelSpec, Hyper

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def T():
    import torch
    return torch


@pytest.fixture(scope="module")
def L():
    from paper_1602_08191_b200 import _lib
    return _lib


@pytest.fixture(scope="module")
def orc():
    return Oracle("dso")


def dev(T, a):
    return T.from_numpy(np.ascontiguousarray(a)).cuda()


def ptr(t):
    return C.c_void_p(t.data_ptr())


def ulps(a, b):
    a = np.asarray(a, np.float32).view(np.int32).astype(np.int64)
    b = np.asarray(b, np.float32).view(np.int32).astype(np.int64)
    ka = np.where(a < 0, np.int64(-2**31) - a, a)
    kb = np.where(b < 0, np.int64(-2**31) - b, b)
    return np.abs(ka - kb)


def rand_pairs(n, seed):
    rng = np.random.default_rng(seed)
    kind = rng.integers(0, 3, n)
    w = rng.standard_normal(n)
    m = rng.standard_normal(n)
    big = kind == 1
    w[big] *= 2.0 ** rng.uniform(-30, 30, big.sum())
    m[big] *= 2.0 ** rng.uniform(-30, 30, big.sum())
    canc = kind == 2
    w[canc] *= 1e6
    m[canc] = -w[canc] + rng.standard_normal(canc.sum())
    return w.astype(np.float32), m.astype(np.float32)


def test_elastic_kats(T, L, orc):
    # test_params.cpp:41-68
    for w, m, a, ew, em in [([1, 2], [0, 0], 0.1, [0.9, 1.8], [0.1, 0.2]), ([6], [2], 0.25, [5], [3]),
                            ([6], [2], 0.5, [4], [4]), ([3.75, -1.25], [3.75, -1.25], 0.3, [3.75, -1.25], [3.75, -1.25])]:
        wd = dev(T, np.array(w, np.float32))
        md = dev(T, np.array(m, np.float32))
        L.check(L.lib.ds_elastic_update(ptr(wd), ptr(md), len(w), C.c_float(np.float32(a)), None))
        T.cuda.synchronize()
        assert (wd.cpu().numpy() == np.array(ew, np.float32)).all()
        assert (md.cpu().numpy() == np.array(em, np.float32)).all()


@pytest.mark.parametrize("n", [1, 3, 4, 1000, 10007, 1 << 20])
@pytest.mark.parametrize("offset", [0, 1])
def test_elastic_bitexact(T, L, orc, n, offset):
    w, m = rand_pairs(n + offset, 2024 + n)
    alpha = 0.1
    ew, em = orc.easgd_update(w[offset:], m[offset:], alpha)
    wd, md = dev(T, w), dev(T, m)
    L.check(L.lib.ds_elastic_update(C.c_void_p(wd.data_ptr() + 4 * offset), C.c_void_p(md.data_ptr() + 4 * offset),
                                    n, C.c_float(np.float32(alpha)), None))
    T.cuda.synchronize()
    assert np.array_equal(wd.cpu().numpy()[offset:].view(np.uint32), ew.view(np.uint32))
    assert np.array_equal(md.cpu().numpy()[offset:].view(np.uint32), em.view(np.uint32))


def test_elastic_exchange_out(T, L, orc):
    n = 100003
    w, m = rand_pairs(n, 7)
    ew, em = orc.easgd_update(w, m, 0.25)
    wd, md = dev(T, w), dev(T, m)
    out = T.empty_like(wd)
    L.check(L.lib.ds_elastic_exchange(ptr(wd), ptr(md), ptr(out), n, C.c_float(0.25), None))
    T.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy().view(np.uint32), ew.view(np.uint32))
    assert np.array_equal(md.cpu().numpy().view(np.uint32), em.view(np.uint32))
    assert np.array_equal(wd.cpu().numpy(), w)  # worker input untouched


@pytest.mark.parametrize("n", [2, 5, 65536 + 3])
def test_sgd_bitexact(T, L, orc, n):
    rng = np.random.default_rng(n)
    x = rng.standard_normal(n).astype(np.float32)
    g = rng.standard_normal(n).astype(np.float32)
    for eta in (0.5, 0.05, 0.013):
        expect = orc.sgd_step(x, g, eta)
        xd, gd = dev(T, x), dev(T, g)
        out = T.empty_like(xd)
        L.check(L.lib.ds_sgd_step_checked(ptr(out), ptr(xd), ptr(gd), n, eta, None))
        assert np.array_equal(out.cpu().numpy().view(np.uint32), expect.view(np.uint32))


def test_sgd_errors(T, L):
    x = dev(T, np.array([1.0], np.float32))
    g = dev(T, np.array([1.0], np.float32))
    out = T.empty_like(x)
    for eta in (0.0, -0.5):
        with pytest.raises(L.ContractError):
            L.check(L.lib.ds_sgd_step_checked(ptr(out), ptr(x), ptr(g), 1, eta, None))
    nan = dev(T, np.array([np.nan], np.float32))
    inf = dev(T, np.array([np.inf], np.float32))
    with pytest.raises(L.ContractError):
        L.check(L.lib.ds_sgd_step_checked(ptr(out), ptr(nan), ptr(g), 1, 0.1, None))
    with pytest.raises(L.ContractError):
        L.check(L.lib.ds_sgd_step_checked(ptr(out), ptr(x), ptr(inf), 1, 0.1, None))
    big = dev(T, np.array([3e38], np.float32))
    neg = dev(T, np.array([-3e38], np.float32))
    with pytest.raises(L.NumericError):  # test_params.cpp:122-125 overflow
        L.check(L.lib.ds_sgd_step_checked(ptr(out), ptr(big), ptr(neg), 1, 1.0, None))


def desc_of(L, m: ModelSpec):
    h = (C.c_uint32 * max(1, len(m.hidden)))(*m.hidden)
    d = L.ds_model_desc(0 if m.kind == "softmax" else 1, m.n_features, m.n_classes, len(m.hidden), h)
    d._keep = h
    return d


def gpu_loss_and_grad(T, L, m, params, X, y, want_grad=True):
    d = desc_of(L, m)
    ws_b = C.c_uint64()
    L.check(L.lib.ds_loss_and_grad_workspace(C.byref(d), len(y), C.byref(ws_b)))
    ws = T.empty(max(8, ws_b.value) // 8, dtype=T.float64, device="cuda")
    pd, Xd, yd = dev(T, params), dev(T, X), dev(T, y.astype(np.int32))
    g = T.zeros_like(pd) if want_grad else None
    loss = T.zeros(1, dtype=T.float64, device="cuda")
    flags = T.zeros(1, dtype=T.int32, device="cuda")
    L.check(L.lib.ds_loss_and_grad(C.byref(d), ptr(pd), ptr(Xd), ptr(yd), len(y), ptr(g) if g is not None else None,
                                   ptr(loss), ptr(ws), ptr(flags), None))
    T.cuda.synchronize()
    return loss.item(), (g.cpu().numpy() if g is not None else None), int(flags.item())


def test_loss_grad_zero_params_kat(T, L):
    # test_model.cpp:93-110: softmax(2,2), zero params, x=[1,2], y=0
    m = ModelSpec.softmax(2, 2)
    loss, g, fl = gpu_loss_and_grad(T, L, m, np.zeros(6, np.float32), np.array([[1.0, 2.0]], np.float32),
                                    np.array([0], np.uint32))
    assert fl == 0
    assert abs(loss - np.log(2.0)) <= 1e-15 * np.log(2.0)
    assert list(g) == [-0.5, -1.0, 0.5, 1.0, -0.5, 0.5]


@pytest.mark.parametrize("spec", [ModelSpec.softmax(20, 2), ModelSpec.mlp(20, [16], 3), ModelSpec.mlp(4, [8, 16], 3),
                                  ModelSpec.mlp(784, [256], 10)])
@pytest.mark.parametrize("rows", [1, 7, 32])
def test_loss_grad_matches_oracle(T, L, orc, spec, rows):
    X, y = orc.gen_synthetic(max(rows, 40), spec.n_features, spec.n_classes, 2.0, 1.0, 11)
    X, y = X[:rows], y[:rows]
    p = orc.init_params(spec, 5)
    el, eg = orc.loss_and_grad(spec, p, X, y)
    gl, gg, fl = gpu_loss_and_grad(T, L, spec, p, X, y)
    assert fl == 0
    assert abs(gl - el) <= 1e-14 * abs(el)
    d = ulps(gg, eg)
    assert d.max() <= 1, f"max ulp {d.max()}"
    assert (d > 0).mean() <= 1e-3
    # loss_only path (model.cpp:265-275)
    lo, _ = orc.loss_and_grad(spec, p, X, y, want_grad=False)
    gl2, _, _ = gpu_loss_and_grad(T, L, spec, p, X, y, want_grad=False)
    assert abs(gl2 - lo) <= 1e-14 * abs(lo)


def test_label_out_of_range_flag(T, L, orc):
    m = ModelSpec.softmax(3, 2)
    _, _, fl = gpu_loss_and_grad(T, L, m, np.zeros(8, np.float32), np.ones((2, 3), np.float32), np.array([0, 2], np.uint32))
    assert fl & L.FLAG_LABEL_RANGE


def test_momentum_update(T, L):
    """SURVEY §8 a21 (not in the reference): mu = 0 is bit-identical to sgd_update; mu > 0
    matches the Caffe-form recurrence evaluated with numpy float32 (separate roundings)."""
    rng = np.random.default_rng(3)
    n = 100003
    x = rng.standard_normal(n).astype(np.float32)
    g = rng.standard_normal(n).astype(np.float32)
    v0 = rng.standard_normal(n).astype(np.float32)
    eta, wd = np.float32(0.05), np.float32(0.01)
    for mu in (0.0, 0.9):
        xd, gd, vd = dev(T, x), dev(T, g), dev(T, v0.copy())
        out = T.empty_like(xd)
        fl = T.zeros(1, dtype=T.int32, device="cuda")
        L.check(L.lib.ds_sgd_momentum_update(ptr(out), ptr(xd), ptr(vd), ptr(gd), n, C.c_float(eta), C.c_float(mu),
                                             C.c_float(wd), ptr(fl), None))
        T.cuda.synchronize()
        g1 = (g + wd * x).astype(np.float32)
        v = (np.float32(mu) * v0 + g1).astype(np.float32) if mu else g1
        ref = (x - eta * v).astype(np.float32)
        assert np.array_equal(out.cpu().numpy().view(np.uint32), ref.view(np.uint32))
        assert np.array_equal(vd.cpu().numpy().view(np.uint32), v.view(np.uint32))
        if mu == 0.0:
            out2 = T.empty_like(xd)
            L.check(L.lib.ds_sgd_update(ptr(out2), ptr(xd), ptr(gd), n, C.c_float(eta), C.c_float(wd), ptr(fl), None))
            T.cuda.synchronize()
            assert T.equal(out, out2)
