"""DSHD shard ingestion: ds_shard_info_read / ds_shard_load /
ds_engine_create_from_shard against the reference's format and checks.

Fixtures: tests/golden/ref_small.dshd was written by the UNMODIFIED reference's
write_shard (shard.cpp:40-73) from gen_synthetic data kept in ref_small_dshd.npz
(tests/golden/make_golden.py). The corruption cases follow test_data.cpp:254-289; the
messages and error classes are read_shard's (shard.cpp:75-125: FormatError / IoError).
Bar: bit-exact features and labels.
"""
import ctypes as C
import os
import struct

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden", "ref_small.dshd")


@pytest.fixture(scope="module")
def L():
    from paper_1602_08191_b200 import _lib
    return _lib


@pytest.fixture(scope="module")
def gold():
    g = np.load(os.path.join(HERE, "golden", "ref_small_dshd.npz"))
    return g["X"], g["y"]


def write_dshd(path, X, y, seed=1, magic=0x44534844, version=1, n=None, f=None, c=None):
    """The DSHD layout (shard.hpp:9-16), written independently of any implementation."""
    n = len(y) if n is None else n
    f = X.shape[1] if f is None else f
    c = int(y.max()) + 1 if c is None else c
    body = np.empty((len(y), X.shape[1] + 1), np.uint32)
    body[:, :-1] = np.ascontiguousarray(X, np.float32).view(np.uint32)
    body[:, -1] = y
    with open(path, "wb") as fh:
        fh.write(struct.pack("<IIIIIQ", magic, version, n, f, c, seed))
        fh.write(body.tobytes())


def info_of(L, path):
    info = L.ds_shard_info()
    L.check(L.lib.ds_shard_info_read(path.encode(), C.byref(info)))
    return info


def test_reference_written_header(L, gold, tmp_path):
    X, y = gold
    info = info_of(L, GOLD)
    assert (info.n_samples, info.n_features, info.n_classes, info.seed) == (37, 9, 4, 0xFEED)
    assert os.path.getsize(GOLD) == 28 + 37 * (9 * 4 + 4)  # dshd::file_size
    # our independent writer produces the reference's bytes
    with open(GOLD, "rb") as fh:
        ref_bytes = fh.read()
    p = str(tmp_path / "mine.dshd")
    write_dshd(p, X, y, seed=0xFEED, c=4)
    with open(p, "rb") as fh:
        assert fh.read() == ref_bytes


@pytest.mark.parametrize("case,err,msg", [
    ("truncated", "FormatError", "truncated header"),
    ("magic", "FormatError", "bad magic"),
    ("version", "FormatError", "unsupported version"),
    ("empty", "FormatError", "empty shard"),
    ("zerodim", "FormatError", "zero dimension"),
    ("short", "FormatError", "size mismatch"),
    ("long", "FormatError", "size mismatch"),
    ("missing", "IoError", "cannot open"),
])
def test_header_rejections(L, gold, tmp_path, case, err, msg):
    X, y = gold
    p = str(tmp_path / f"{case}.dshd")
    if case == "truncated":
        open(p, "wb").write(b"DSHD" * 3)
    elif case == "magic":
        write_dshd(p, X, y, magic=0x12345678)
    elif case == "version":
        write_dshd(p, X, y, version=2)
    elif case == "empty":
        open(p, "wb").write(struct.pack("<IIIIIQ", 0x44534844, 1, 0, 9, 4, 0))
    elif case == "zerodim":
        write_dshd(p, X, y, c=0)
    elif case == "short":
        write_dshd(p, X, y)
        os.truncate(p, os.path.getsize(p) - 1)
    elif case == "long":
        write_dshd(p, X, y)
        open(p, "ab").write(b"\0")
    else:
        p = str(tmp_path / "nope.dshd")
    with pytest.raises(getattr(L, err)) as ei:
        info_of(L, p)
    assert msg in str(ei.value)


@pytest.mark.gpu
def test_load_reference_shard_bit_exact(L, gold):
    import torch
    X, y = gold
    Xd = torch.full((40, 9), float("nan"), device="cuda")
    yd = torch.zeros(40, dtype=torch.int32, device="cuda")
    info = L.ds_shard_info()
    L.check(L.lib.ds_shard_load(GOLD.encode(), C.c_void_p(Xd.data_ptr()), C.c_void_p(yd.data_ptr()), 40,
                                C.byref(info), None))
    assert info.n_samples == 37
    assert np.array_equal(Xd[:37].cpu().numpy().view(np.uint32), X.view(np.uint32))
    assert np.array_equal(yd[:37].cpu().numpy().view(np.uint32), y)
    assert torch.isnan(Xd[37:]).all()  # nothing past the shard was touched


@pytest.mark.gpu
def test_load_rejects_label_and_capacity(L, gold, tmp_path):
    import torch
    X, y = gold
    bad = y.copy()
    bad[5], bad[30] = 9, 11
    p = str(tmp_path / "label.dshd")
    write_dshd(p, X, bad, c=4)
    Xd = torch.empty((37, 9), device="cuda")
    yd = torch.empty(37, dtype=torch.int32, device="cuda")
    with pytest.raises(L.FormatError) as ei:
        L.check(L.lib.ds_shard_load(p.encode(), C.c_void_p(Xd.data_ptr()), C.c_void_p(yd.data_ptr()), 37, None,
                                    None))
    assert "label 9 out of range at sample 5" in str(ei.value)  # the first offender, as shard.cpp:115-120
    with pytest.raises(L.ContractError):
        L.check(L.lib.ds_shard_load(GOLD.encode(), C.c_void_p(Xd.data_ptr()), C.c_void_p(yd.data_ptr()), 36, None,
                                    None))


@pytest.mark.gpu
def test_load_multi_chunk(L, tmp_path):
    """A shard larger than the 64 MiB pipeline slot (several chunks, both slots reused),
    odd row width so rows straddle every alignment."""
    import time
    import torch
    rng = np.random.default_rng(3)
    n, f = 60_000, 785
    X = rng.standard_normal((n, f), dtype=np.float32)
    y = rng.integers(0, 10, n).astype(np.uint32)
    p = str(tmp_path / "big.dshd")
    write_dshd(p, X, y, c=10)
    Xd = torch.empty((n, f), device="cuda")
    yd = torch.empty(n, dtype=torch.int32, device="cuda")
    t0 = time.perf_counter()
    L.check(L.lib.ds_shard_load(p.encode(), C.c_void_p(Xd.data_ptr()), C.c_void_p(yd.data_ptr()), n, None, None))
    dt = time.perf_counter() - t0
    assert np.array_equal(Xd.cpu().numpy().view(np.uint32), X.view(np.uint32))
    assert np.array_equal(yd.cpu().numpy().view(np.uint32), y)
    t0 = time.perf_counter()
    L.check(L.lib.ds_shard_load(p.encode(), C.c_void_p(Xd.data_ptr()), C.c_void_p(yd.data_ptr()), n, None, None))
    dt2 = time.perf_counter() - t0
    print(f"ds_shard_load: {os.path.getsize(p) / dt / 1e9:.2f} GB/s first call, {os.path.getsize(p) / dt2 / 1e9:.2f} "
          f"GB/s second call, file (page cache) -> HBM ({os.path.getsize(p) >> 20} MiB)")


@pytest.mark.gpu
def test_engine_from_shard_matches_host_engine(L, tmp_path):
    """SgdEngine over the DSHD file == SgdEngine over the same arrays passed from the host:
    identical TrainLog and parameters (bit-exact)."""
    from oracle.oracle import ModelSpec, Oracle
    orc = Oracle("dso")
    m = ModelSpec.mlp(20, [16], 3)
    X, y = orc.gen_synthetic(300, 20, 3, 2.0, 1.0, 5)
    p = str(tmp_path / "train.dshd")
    write_dshd(p, X, y, c=3)
    init = orc.init_params(m, 2)
    h = (C.c_uint32 * 1)(16)
    desc = L.ds_model_desc(1, 20, 3, 1, h)
    hp = L.ds_hyper(0.05, 0.1, 5, 16, 40, 0.0, 0.0, 0)
    out = []
    for from_file in (False, True):
        e = C.c_void_p()
        if from_file:
            L.check(L.lib.ds_engine_create_from_shard(C.byref(e), 0, C.byref(desc), p.encode(), C.byref(hp), 9,
                                                      init.ctypes.data, L.DS_ENGINE_LAYERED))
        else:
            L.check(L.lib.ds_engine_create(C.byref(e), 0, C.byref(desc), X.ctypes.data, y.ctypes.data, len(y), 3,
                                           C.byref(hp), 9, init.ctypes.data, L.DS_ENGINE_LAYERED))
        L.check(L.lib.ds_engine_run(e, 40, 0, None))
        L.check(L.lib.ds_engine_sync(e))
        loss = np.zeros(40)
        L.check(L.lib.ds_engine_log(e, 0, 40, loss.ctypes.data, None, None, None))
        par = np.zeros(len(init), np.float32)
        L.check(L.lib.ds_engine_get_params(e, par.ctypes.data))
        L.lib.ds_engine_destroy(e)
        out.append((loss, par))
    assert np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][1].view(np.uint32), out[1][1].view(np.uint32))
