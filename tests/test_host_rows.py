"""The host half of the tensor-core stream mode (csrc/host_rows.cpp, ds_host_rows_to_bf16):
gather_batch (model.cpp:12-21) plus the bf16 operand cast, run on the CPU. It must give the
device cast's bits (__float2bfloat16_rn: round to nearest even, NaN -> 0x7FFF, denormals
kept), including where the AVX-512 BF16 fast path has to fall back (denormals, NaN, Inf).
No GPU needed."""
import ctypes as C

import numpy as np
import pytest


@pytest.fixture(scope="module")
def L():
    from paper_1602_08191_b200 import _lib
    return _lib


def bf16_rn(x: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    nan = (u & 0x7FFFFFFF) > 0x7F800000
    return np.where(nan, np.uint16(0x7FFF), r)


@pytest.mark.parametrize("F,pitch", [(784, 784), (37, 40), (1, 8), (96, 96)])
def test_gather_cast_bits(L, F, pitch):
    rng = np.random.default_rng(F)
    n = 50
    X = rng.standard_normal((n, F)).astype(np.float32) * np.exp2(rng.integers(-20, 20, (n, F))).astype(np.float32)
    flat = X.reshape(-1)
    k = flat.size
    # specials: denormals, +-0, +-inf, NaNs with payloads, ties (exact halfway points)
    sp = np.array([1e-40, -3e-39, 0.0, -0.0, np.inf, -np.inf], np.float32)
    flat[rng.integers(0, k, 200)] = sp[rng.integers(0, len(sp), 200)]
    nans = rng.integers(0, k, 20)
    flat[nans] = np.array([0x7FC00001, 0xFFA00000, 0x7F800001] * 7, np.uint32)[:20].view(np.float32)
    ties = rng.integers(0, k, 50)
    flat[ties] = (rng.integers(0, 1 << 16, 50).astype(np.uint32) << 16 | 0x8000).view(np.float32)
    idx = rng.integers(0, n, 32).astype(np.uint32)
    dst = np.full((32, pitch), 0xABCD, np.uint16)
    assert L.lib.ds_host_rows_to_bf16(X.ctypes.data, F, idx.ctypes.data, 32, dst.ctypes.data, pitch) == 0
    assert np.array_equal(dst[:, :F], bf16_rn(X[idx]))
    assert (dst[:, F:] == 0xABCD).all()  # padding untouched
    dst2 = np.zeros((n, pitch), np.uint16)
    assert L.lib.ds_host_rows_to_bf16(X.ctypes.data, F, None, n, dst2.ctypes.data, pitch) == 0
    assert np.array_equal(dst2[:, :F], bf16_rn(X))


def test_contract(L):
    X = np.zeros((2, 4), np.float32)
    d = np.zeros((2, 4), np.uint16)
    assert L.lib.ds_host_rows_to_bf16(X.ctypes.data, 4, None, 2, d.ctypes.data, 3) != 0  # pitch < F
    assert L.lib.ds_host_rows_to_bf16(None, 4, None, 2, d.ctypes.data, 4) != 0
