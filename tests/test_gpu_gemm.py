"""tcgen05 tf32 GEMM (csrc/gemm_tc.cu, ds_gemm_tf32) against a float64 PyTorch reference.

Bar (stated tolerance, tf32 operands with f32 accumulation): elementwise
|D - D64| <= 4e-3 * (|A| . |B|^T) + 1e-6, i.e. each product may carry the tf32 operand
rounding (2 x 2^-11, truncation allowed) plus f32 accumulation error. A layout or
descriptor bug shows up as O(1) relative errors, far outside this band.
"""
import ctypes as C

import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def L():
    from paper_1602_08191_b200 import _lib
    return _lib


def run(L, torch, M, N, K, lda=None, ldb=None, ldd=None, scale=1.0, bias_n=False, bias_m=False, relu=False, splits=1,
        seed=0, tol=4e-3):
    g = torch.Generator(device="cuda").manual_seed(seed)
    lda, ldb, ldd = lda or K, ldb or K, ldd or N
    A = torch.randn(M, lda, device="cuda", generator=g)
    B = torch.randn(N, ldb, device="cuda", generator=g)
    D = torch.full((M, ldd), float("nan"), device="cuda")
    bn = torch.randn(N, device="cuda", generator=g) if bias_n else None
    bm = torch.randn(M, device="cuda", generator=g) if bias_m else None
    part = torch.empty(max(1, splits) * M * N, device="cuda") if splits > 1 else None
    ptr = lambda t: C.c_void_p(t.data_ptr()) if t is not None else None  # noqa: E731
    L.check(L.lib.ds_gemm_tf32(ptr(A), lda, ptr(B), ldb, ptr(D), ldd, M, N, K, C.c_float(scale), ptr(bn), ptr(bm),
                               int(relu), splits, ptr(part), None))
    torch.cuda.synchronize()
    a, b = A[:, :K].double(), B[:, :K].double()
    ref = scale * (a @ b.T)
    if bn is not None:
        ref += bn.double()[None, :]
    if bm is not None:
        ref += bm.double()[:, None]
    if relu:
        ref = ref.clamp_min(0)
    bound = tol * abs(scale) * (a.abs() @ b.abs().T) + 1e-6
    got = D[:, :N].double()
    err = (got - ref).abs()
    assert torch.isfinite(got).all()
    assert (err <= bound).all(), f"max err {err.max().item():.3e}, worst ratio {(err / bound).max().item():.2f}"
    if ldd > N:
        assert torch.isnan(D[:, N:]).all()  # columns past N untouched
    return err.max().item()


@pytest.mark.parametrize("M,N,K", [(128, 64, 32), (128, 128, 64), (256, 256, 256), (300, 96, 363), (77, 200, 40),
                                   (1000, 10, 4096), (5, 130, 17)])
def test_shapes(L, M, N, K):
    import torch
    lda = (K + 3) // 4 * 4
    run(L, torch, M, N, K, lda=lda, ldb=lda)


def test_epilogue_and_strides(L):
    import torch
    run(L, torch, 333, 192, 1200, lda=2400, ldb=1204, ldd=256, scale=0.5, bias_n=True, relu=True)
    run(L, torch, 190, 100, 96, bias_m=True, scale=-2.0)


@pytest.mark.parametrize("M,N,K", [(128 * 500, 48, 64), (128 * 700 + 5, 96, 72), (128 * 320, 128, 40),
                                   (128 * 300 + 17, 192, 96), (128 * 300, 256, 64), (128 * 3, 200, 5000)])
def test_persistent_tiles(L, M, N, K):
    """More tiles than co-resident CTAs for every tile width (each persistent CTA walks several
    tiles through both TMEM accumulator buffers), ragged M, short and long K."""
    import torch
    lda = (K + 3) // 4 * 4
    run(L, torch, M, N, K, lda=lda, ldb=lda, bias_n=True, relu=True, seed=M % 7)


@pytest.mark.parametrize("splits", [2, 4, 9])
def test_split_k(L, splits):
    import torch
    run(L, torch, 128, 512, 9216, splits=splits, bias_n=True, relu=True)
    run(L, torch, 256, 363, 640, splits=splits, scale=1.0 / 128)


def test_fc6_shape_and_throughput(L):
    """AlexNet fc6 forward shape (batch 128, 9216 -> 4096) plus a timing print."""
    import torch
    run(L, torch, 128, 4096, 9216, splits=4)
    M, N, K = 4096, 9216, 1024
    A = torch.randn(M, K, device="cuda")
    B = torch.randn(N, K, device="cuda")
    D = torch.empty(M, N, device="cuda")
    args = (C.c_void_p(A.data_ptr()), K, C.c_void_p(B.data_ptr()), K, C.c_void_p(D.data_ptr()), N, M, N, K,
            C.c_float(1.0), None, None, 0, 1, None, None)
    for _ in range(3):
        L.check(L.lib.ds_gemm_tf32(*args))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        L.check(L.lib.ds_gemm_tf32(*args))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"ds_gemm_tf32 {M}x{N}x{K}: {2 * M * N * K / ms / 1e9:.1f} TFLOP/s")


def test_3xtf32_mode_is_f32_accurate(L, monkeypatch):
    """DS_GEMM_3XTF32=1 (the parity-diagnostic mode): hi/lo operand splits give f32-level
    products, |err| <= 2e-6 * (|A| . |B|^T)."""
    import torch
    monkeypatch.setenv("DS_GEMM_3XTF32", "1")
    run(L, torch, 300, 96, 363, lda=364, ldb=364, tol=2e-6)
    run(L, torch, 333, 192, 1200, lda=2400, ldb=1204, ldd=256, scale=0.5, bias_n=True, relu=True, tol=2e-6)
