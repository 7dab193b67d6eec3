"""AlexNet-shaped convnet (model kind 3, BASELINE config 4) on the B200 against the f64 CPU
restatement (oracle/ds_oracle_alex.c, pinned by central differences in test_oracle.py and
against PyTorch float64 autograd to 1 ulp in test_oracle_cnn_torch.py).

NOT IN THE REFERENCE (no reference implementation to pin against). Every contraction runs on the
tcgen05 tensor cores with tf32 operands and f32 accumulation (csrc/gemm_tc.cu,
csrc/alexnet.cu). Two bars:
  * f32-accurate products (DS_GEMM_3XTF32=1: each GEMM as three tf32 GEMMs on hi/lo
    operand splits) isolate the implementation from tf32 rounding: batch loss within 2e-5
    relative, every layer's gradient within 2e-4 relative norm (cosine >= 0.99999) of the
    f64 oracle — the evidence that the layer algebra is right (measured, tools/alex_tol.py:
    1.4e-5 .. 5e-5 at S = 55 and S = 224; the tensor core's f32 accumulation is not IEEE
    round-to-nearest, so the residual grows with K);
  * the production tf32 path: batch loss within 5e-4 relative (measured 9e-7 .. 5e-6 at
    batch >= 2, 1.6e-4 for a single row);
    the classifier layer's gradient within 1e-2 relative norm (measured 3e-3 .. 6e-3);
    every other layer within 0.12 relative norm, cosine >= 0.99 (measured 0.036 .. 0.090,
    the same against the f64 oracle as against the GPU's own 3xTF32 products, and the
    same at batch 2, 13, 32 and 64). That residual is not accumulation error: tf32 operand
    rounding (2^-11) flips ReLU masks and max-pool winners whose pre-activations tie to
    within 5e-4, and each flip moves one position's whole gradient contribution — a flip
    rate of ~1e-3 gives sqrt(2e-3) ~ 5% relative norm independent of batch. Only
    f32-accurate forward products remove it (the 3xTF32 bar above);
  * predictions: argmax agreement with the oracle >= 0.99 (measured 1.0 on 200 rows);
  * determinism: two identical calls are bit-identical (fixed-order split-K reductions).
"""
import ctypes as C

import numpy as np
import pytest

from oracle.oracle import ModelSpec, Oracle

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


def desc(L, side, c):
    h = (C.c_uint32 * 1)(0)
    d = L.ds_model_desc(3, 3 * side * side, c, 0, h)
    d._keep = h
    return d


def layer_bounds(orc, side, c):
    m = ModelSpec.alexnet(side, c)
    P = orc.param_dim(m)
    q5 = 256 * ((((((side - 11) // 4 + 1) - 2) // 2 + 1 - 2) // 2 + 1 - 2) // 2 + 1) ** 2
    sizes = [34944, 307456, 885120, 663936, 442624, 4096 * q5 + 4096, 4096 * 4096 + 4096, c * 4096 + c]
    b = np.cumsum([0] + sizes)
    assert b[-1] == P
    return [(int(b[i]), int(b[i + 1])) for i in range(8)]


def gpu_lag(T, L, d, params, X, y, want_grad=True):
    wsb = C.c_uint64()
    L.check(L.lib.ds_loss_and_grad_workspace(C.byref(d), len(y), C.byref(wsb)))
    ws = T.empty(max(8, wsb.value), dtype=T.uint8, device="cuda")
    pd = T.from_numpy(np.ascontiguousarray(params)).cuda()
    Xd = T.from_numpy(np.ascontiguousarray(X)).cuda()
    yd = T.from_numpy(np.ascontiguousarray(y).astype(np.int32)).cuda()
    g = T.zeros_like(pd) if want_grad else None
    loss = T.zeros(1, dtype=T.float64, device="cuda")
    flags = T.zeros(1, dtype=T.int32, device="cuda")
    L.check(L.lib.ds_loss_and_grad(C.byref(d), C.c_void_p(pd.data_ptr()), C.c_void_p(Xd.data_ptr()),
                                   C.c_void_p(yd.data_ptr()), len(y),
                                   C.c_void_p(g.data_ptr()) if g is not None else None,
                                   C.c_void_p(loss.data_ptr()), C.c_void_p(ws.data_ptr()),
                                   C.c_void_p(flags.data_ptr()), None))
    T.cuda.synchronize()
    return loss.item(), (g.cpu().numpy() if g is not None else None), int(flags.item())


def compare(orc, side, c, lg, gg, lr, gr, exact):
    assert abs(lg - lr) <= (2e-5 if exact else 5e-4) * abs(lr), (lg, lr)
    bounds = layer_bounds(orc, side, c)
    for li, (a, b) in enumerate(bounds):
        ref, got = gr[a:b].astype(np.float64), gg[a:b].astype(np.float64)
        rn = np.linalg.norm(got - ref) / np.linalg.norm(ref)
        cos = float(ref @ got / (np.linalg.norm(ref) * np.linalg.norm(got) + 1e-300))
        if exact:
            assert rn <= 2e-4 and cos >= 0.99999, (li, rn, cos)
        elif li == len(bounds) - 1:  # classifier: no ReLU / pool downstream of its inputs' use
            assert rn <= 1e-2 and cos >= 0.9999, (li, rn, cos)
        else:
            assert rn <= 0.12 and cos >= 0.99, (li, rn, cos)


@pytest.fixture(params=["tf32", "exact"])
def mode(request, monkeypatch):
    if request.param == "exact":
        monkeypatch.setenv("DS_GEMM_3XTF32", "1")
    return request.param


@pytest.mark.parametrize("batch", [1, 6, 13])
def test_small_side_loss_and_grad(T, L, orc, batch, mode):
    side, c = 55, 5
    m = ModelSpec.alexnet(side, c)
    w = orc.init_params(m, 3)
    X, y = orc.gen_synthetic(batch, 3 * side * side, c, 1.0, 1.0, 21)
    X = np.ascontiguousarray(X * 5.0, dtype=np.float32)
    lr, gr = orc.loss_and_grad(m, w, X, y)
    lg, gg, flags = gpu_lag(T, L, desc(L, side, c), w, X, y)
    assert flags == 0
    compare(orc, side, c, lg, gg, lr, gr, mode == "exact")


def test_full_size_loss_and_grad(T, L, orc, mode):
    """224 x 224 x 3 input, 1000 classes, P = 60,965,224 (config 4 shapes), 2 rows."""
    side, c = 224, 1000
    m = ModelSpec.alexnet(side, c)
    w = orc.init_params(m, 4)
    X, y = orc.gen_synthetic(2, 3 * side * side, c, 1.0, 1.0, 5)
    lr, gr = orc.loss_and_grad(m, w, X, y)
    lg, gg, flags = gpu_lag(T, L, desc(L, side, c), w, X, y)
    assert flags == 0
    compare(orc, side, c, lg, gg, lr, gr, mode == "exact")


def test_deterministic_and_loss_only(T, L, orc):
    side, c = 67, 10
    m = ModelSpec.alexnet(side, c)
    w = orc.init_params(m, 5)
    X, y = orc.gen_synthetic(32, 3 * side * side, c, 1.0, 1.0, 8)
    d = desc(L, side, c)
    l1, g1, _ = gpu_lag(T, L, d, w, X, y)
    l2, g2, _ = gpu_lag(T, L, d, w, X, y)
    l3, _, _ = gpu_lag(T, L, d, w, X, y, want_grad=False)
    assert l1 == l2 == l3
    assert np.array_equal(g1.view(np.uint32), g2.view(np.uint32))


def test_predict_matches_oracle(T, L, orc):
    side, c = 55, 7
    m = ModelSpec.alexnet(side, c)
    w = orc.init_params(m, 6)
    X, y = orc.gen_synthetic(200, 3 * side * side, c, 1.0, 1.0, 9)
    X = np.ascontiguousarray(X * 5.0, dtype=np.float32)
    ref = orc.predict(m, w, X)
    d = desc(L, side, c)
    pd = T.from_numpy(w).cuda()
    Xd = T.from_numpy(X).cuda()
    pred = T.zeros(len(y), dtype=T.int32, device="cuda")
    L.check(L.lib.ds_predict(C.byref(d), C.c_void_p(pd.data_ptr()), C.c_void_p(Xd.data_ptr()), len(y),
                             C.c_void_p(pred.data_ptr()), None))
    T.cuda.synchronize()
    got = pred.cpu().numpy()
    agree = (got == ref).mean()
    assert agree >= 0.99, agree


def test_engine_training_tracks_oracle(T, L, orc, mode, monkeypatch):
    """run_training_loop with a Locked master exchange every tau steps through the layered
    engine (CUDA-graph replay in tf32 mode); exact mode tracks the f64 oracle to 1e-5."""
    if mode == "exact":
        monkeypatch.setenv("DS_ENGINE_NO_GRAPH", "1")
    from oracle.oracle import Hyper
    side, c = 55, 5
    m = ModelSpec.alexnet(side, c)
    X, y = orc.gen_synthetic(24, 3 * side * side, c, 1.0, 1.0, 7)
    X = np.ascontiguousarray(X * 5.0, dtype=np.float32)
    w = orc.init_params(m, 2)
    hp = Hyper(eta=0.01, alpha=0.1, tau=3, batch_size=4, i_max=8)
    d = desc(L, side, c)
    h = L.ds_hyper(hp.eta, hp.alpha, hp.tau, hp.batch_size, hp.i_max, 0.0, 0.0, 0)
    e = C.c_void_p()
    yk = y.astype(np.uint32)
    L.check(L.lib.ds_engine_create(C.byref(e), 0, C.byref(d), X.ctypes.data, yk.ctypes.data, len(y), c, C.byref(h),
                                   99, w.ctypes.data, L.DS_ENGINE_AUTO))
    mst = C.c_void_p()
    L.check(L.lib.ds_master_create(C.byref(mst), 0, len(w), C.c_float(0.1), L.DS_MODE_LOCKED, w.ctypes.data))
    L.check(L.lib.ds_engine_attach_master(e, mst))
    L.check(L.lib.ds_engine_run(e, hp.i_max, 0, None))
    L.check(L.lib.ds_engine_sync(e))
    params = np.zeros_like(w)
    L.check(L.lib.ds_engine_get_params(e, params.ctypes.data))
    loss = np.zeros(hp.i_max)
    ex = np.zeros(hp.i_max, np.uint8)
    L.check(L.lib.ds_engine_log(e, 0, hp.i_max, loss.ctypes.data, None, ex.ctypes.data, None))
    snap = np.zeros_like(w)
    L.check(L.lib.ds_master_snapshot(mst, snap.ctypes.data))
    L.lib.ds_engine_destroy(e)
    L.lib.ds_master_destroy(mst)
    ref = orc.run_training_loop(m, X, y, c, hp, 99, w, exchange_mode=2, master=w)
    assert list(ex) == list(ref["exchanged"])
    tol = 1e-5 if mode == "exact" else 5e-3
    assert np.allclose(loss, ref["batch_loss"], rtol=tol, atol=0)
    scale = np.abs(w).max()
    assert np.abs(params - ref["final_params"]).max() <= tol * scale
    assert np.abs(snap - ref["master"]).max() <= tol * scale
