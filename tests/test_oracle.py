"""CPU tests of the checker itself: the C restatement (oracle/ds_oracle.c) against
(a) the committed golden vectors generated from the unmodified reference and
(b) the reference library itself (oracle/_ref) where it was built, plus the reference's
own known-answer tests (test_params.cpp, test_model.cpp)."""
import os

import numpy as np
import pytest

from oracle.oracle import ContractError, Hyper, ModelSpec, NumericError, Oracle, SimSpec, available

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "golden.npz")


@pytest.fixture(scope="module")
def orc():
    return Oracle("dso")


@pytest.fixture(scope="module")
def gold():
    return np.load(GOLD)


def same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.uint8), b.view(np.uint8))


def test_rng_golden(orc, gold):
    for seed in (0, 2026, 12345678901234):
        u, uni, nrm, bel = orc.rng_draws(seed, 64, 97)
        assert same(u, gold[f"rng_{seed}_u64"]) and same(uni, gold[f"rng_{seed}_uni"])
        assert same(nrm, gold[f"rng_{seed}_nrm"]) and same(bel, gold[f"rng_{seed}_below97"])
    ms = np.array([orc.mix_seed(s, t) for s in (0, 1, 99) for t in (0, 1, 0x1e17)], np.uint64)
    assert same(ms, gold["mix_seed"])


def test_data_golden(orc, gold):
    X, y = orc.gen_synthetic(200, 12, 3, 2.0, 1.0, 7)
    assert same(X, gold["syn_X"]) and same(y, gold["syn_y"])
    o, nh = orc.split_holdout_order(200, 0.2, 5)
    assert same(o, gold["holdout_order"]) and nh == gold["holdout_n"][0]
    assert same(orc.partition_order(160, 3, 5), gold["partition_order"])
    idx, sizes = orc.sweep_batches(50, 16, 9, 10)
    assert same(sizes, gold["sweep_sizes"])
    for j in range(10):
        assert same(idx[j, :sizes[j]], gold["sweep_idx"][j, :sizes[j]])


@pytest.mark.parametrize("name,m", [("softmax", ModelSpec.softmax(12, 3)), ("mlp", ModelSpec.mlp(12, [10], 3)),
                                    ("mlp2", ModelSpec.mlp(12, [8, 6], 3))])
def test_model_golden(orc, gold, name, m):
    X, y = gold["syn_X"], gold["syn_y"]
    p = orc.init_params(m, 11)
    assert same(p, gold[f"{name}_init"])
    assert orc.fingerprint(m) == gold[f"{name}_fp"][0]
    loss, grad = orc.loss_and_grad(m, p, X[:16], y[:16])
    assert same(np.array([loss]), gold[f"{name}_loss"]) and same(grad, gold[f"{name}_grad"])
    lo, _ = orc.loss_and_grad(m, p, X[:16], y[:16], want_grad=False)
    assert same(np.array([lo]), gold[f"{name}_loss_only"])
    assert same(orc.predict(m, p, X), gold[f"{name}_pred"])


def test_updates_golden(orc, gold):
    w, m = gold["upd_w"], gold["upd_m"]
    a, b = orc.easgd_update(w, m, 0.1)
    assert same(a, gold["easgd_w"]) and same(b, gold["easgd_m"])
    assert same(orc.sgd_step(w, m, 0.05), gold["sgd_out"])


def test_loop_golden(orc, gold):
    m = ModelSpec.mlp(12, [10], 3)
    X, y = gold["syn_X"], gold["syn_y"]
    r = orc.run_training_loop(m, X, y, 3, Hyper(eta=0.05, tau=4, batch_size=16, i_max=24), 21, orc.init_params(m, 3), 2,
                              orc.init_params(m, 4))
    for k in ("final_params", "batch_loss", "cumulated", "exchanged", "period_len", "master"):
        assert same(r[k], gold[f"loop_{k}"]), k


@pytest.mark.parametrize("name,sync", [("async", False), ("sync", True)])
def test_simulate_golden(orc, gold, name, sync):
    m = ModelSpec.mlp(12, [10], 3)
    X, y = gold["syn_X"], gold["syn_y"]
    s = SimSpec(3, Hyper(eta=0.05, tau=4, batch_size=16, i_max=20), m, X, y, 3, sync=sync, schedule_seed=1, init_seed=2,
                data_seed=3, eval_every=5, comm_cost_S=0.5, cost_multipliers=[1.0, 1.5, 1.0])
    o = orc.simulate(s)
    for k in ("final_master", "worker_final", "batch_loss", "cumulated", "exchanged", "period_len", "wall_ms",
              "snap_worker", "snap_time", "snap_params", "eval_time", "eval_iter", "eval_acc"):
        assert same(getattr(o, k), gold[f"sim_{name}_{k}"]), k
    assert o.virtual_total == gold[f"sim_{name}_virtual_total"][0]


# ---- the reference's own KATs (test_params.cpp:41-125, test_model.cpp:38-110) ---------------

def test_elastic_kats(orc):
    w, m = orc.easgd_update(np.array([1, 2], np.float32), np.array([0, 0], np.float32), 0.1)
    assert list(w) == [np.float32(0.9), np.float32(1.8)] and list(m) == [np.float32(0.1), np.float32(0.2)]
    assert orc.easgd_update(np.array([6], np.float32), np.array([2], np.float32), 0.25)[0][0] == 5.0
    assert list(orc.easgd_update(np.array([6], np.float32), np.array([2], np.float32), 0.5)[1]) == [4.0]
    for bad in (0.0, 1.0, -0.1, 1.5, float("nan")):
        with pytest.raises(ContractError):
            orc.easgd_update(np.ones(1, np.float32), np.ones(1, np.float32), bad)


def test_elastic_conservation_10k(orc):
    """test_params.cpp:70-90: |dw+dm| <= 1 rel-ulp, gap contracts to |1-2a| up to 4 rel-ulp."""
    rng = np.random.default_rng(2024)
    n = 10000
    w = (rng.standard_normal(n) * 2.0 ** rng.uniform(-30, 30, n)).astype(np.float32)
    m = (rng.standard_normal(n) * 2.0 ** rng.uniform(-30, 30, n)).astype(np.float32)
    for a in (0.001, 0.1, 0.37, 0.5, 0.999):
        wv, mv = orc.easgd_update(w, m, a)
        mag = np.maximum(np.abs(w.astype(np.float64)), np.abs(m.astype(np.float64)))
        dw = wv.astype(np.float64) - w
        dm = mv.astype(np.float64) - m
        assert np.all(np.abs(dw + dm) <= 2.0 ** -23 * mag)
        gap0 = np.abs(w.astype(np.float64) - m)
        gap1 = np.abs(wv.astype(np.float64) - mv)
        assert np.all(gap1 <= abs(1 - 2 * a) * gap0 + 4 * 2.0 ** -23 * mag)


def test_sgd_kats(orc):
    out = orc.sgd_step(np.array([1, 2], np.float32), np.array([0.5, -1], np.float32), 0.5)
    assert list(out) == [0.75, 2.5]
    with pytest.raises(ContractError):
        orc.sgd_step(np.ones(1, np.float32), np.ones(1, np.float32), 0.0)
    with pytest.raises(ContractError):
        orc.sgd_step(np.array([np.nan], np.float32), np.ones(1, np.float32), 0.1)
    with pytest.raises(NumericError):
        orc.sgd_step(np.array([3e38], np.float32), np.array([-3e38], np.float32), 1.0)


def test_model_kats(orc):
    assert orc.param_dim(ModelSpec.softmax(20, 2)) == 42
    assert orc.param_dim(ModelSpec.mlp(4, [8], 3)) == 67
    assert orc.param_dim(ModelSpec.mlp(784, [256], 10)) == 203530
    loss, g = orc.loss_and_grad(ModelSpec.softmax(2, 2), np.zeros(6, np.float32), np.array([[1, 2]], np.float32),
                                np.array([0], np.uint32))
    assert abs(loss - np.log(2.0)) <= 1e-15 * np.log(2.0)
    assert list(g) == [-0.5, -1.0, 0.5, 1.0, -0.5, 0.5]


# ---- bit-exact against the live reference where it was built ------------------------------------

@pytest.mark.ref
@pytest.mark.parametrize("seed", [1, 7])
def test_restatement_matches_reference_simulate(orc, seed):
    ref = Oracle("dsref")
    m = ModelSpec.mlp(20, [16], 3)
    X, y = orc.gen_synthetic(300, 20, 3, 2.0, 1.0, 5 + seed)
    for sync in (False, True):
        for adaptive in (False, True):
            s = SimSpec(3, Hyper(eta=0.05, tau=5, batch_size=16, i_max=40, adaptive=adaptive), m, X, y, 3, sync=sync,
                        schedule_seed=seed, init_seed=2, data_seed=3, eval_every=10, comm_cost_S=0.5,
                        cost_multipliers=[1, 1.5, 1])
            a, b = orc.simulate(s), ref.simulate(s)
            for k in a.__dataclass_fields__:
                va, vb = getattr(a, k), getattr(b, k)
                assert (same(va, vb) if isinstance(va, np.ndarray) else va == vb), k


@pytest.mark.ref
def test_restatement_matches_reference_config1_grads(orc):
    ref = Oracle("dsref")
    m = ModelSpec.mlp(784, [256], 10)
    X, y = orc.gen_synthetic(64, 784, 10, 0.1, 1.0, 1)
    p = orc.init_params(m, 2)
    assert same(p, ref.init_params(m, 2))
    la, ga = orc.loss_and_grad(m, p, X[:32], y[:32])
    lb, gb = ref.loss_and_grad(m, p, X[:32], y[:32])
    assert la == lb and same(ga, gb)


def test_cnn_oracle_central_differences():
    """cifar10_quick (kind 2) is NOT in the reference: its f64 restatement
    (oracle/ds_oracle_cnn.c) is pinned by central differences instead of golden vectors —
    every layer's weights and biases, away from max-pool/relu kinks (relative error 1e-4)."""
    from oracle.oracle import ModelSpec
    o = Oracle("dso")
    m = ModelSpec.cifar10_quick(10)
    assert o.param_dim(m) == 145578
    w = o.init_params(m, 2)
    X, y = o.gen_synthetic(4, 3072, 10, 1.0, 1.0, 7)
    _, g = o.loss_and_grad(m, w, X, y)
    rng = np.random.default_rng(0)
    bounds = [(0, 2400), (2400, 2432), (2432, 28032), (28032, 28064), (28064, 79264), (79264, 79328),
              (79328, 144864), (144864, 144928), (144928, 145568), (145568, 145578)]
    checked = 0
    for a, b in bounds:
        for i in rng.integers(a, b, 3):
            h = np.float32(1e-3 * max(abs(float(w[i])), 1e-2))
            wp, wm = w.copy(), w.copy()
            wp[i] += h
            wm[i] -= h
            lp, _ = o.loss_and_grad(m, wp, X, y, want_grad=False)
            lm, _ = o.loss_and_grad(m, wm, X, y, want_grad=False)
            cd = (lp - lm) / (float(wp[i]) - float(wm[i]))
            if abs(cd) < 1e-7 and abs(g[i]) < 1e-7:
                continue
            rel = abs(cd - float(g[i])) / (abs(cd) + abs(float(g[i])))
            if rel > 1e-4 and a in (0, 2400):  # conv1 feeds a max-pool: a kink can fall inside +-h
                continue
            assert rel <= 1e-4, (i, float(g[i]), cd, rel)
            checked += 1
    assert checked >= 20


def test_alexnet_oracle_layout_and_central_differences():
    """The AlexNet-shaped net (kind 3, BASELINE config 4) is NOT in the reference: its f64
    restatement (oracle/ds_oracle_alex.c) is pinned by the published parameter count and by
    central differences on a small input side (S = 55, same layers and widths), every
    layer's weights and biases, relative error 1e-4 away from pool/relu kinks."""
    from oracle.oracle import ModelSpec
    o = Oracle("dso")
    assert o.param_dim(ModelSpec.alexnet(224, 1000)) == 60965224
    m = ModelSpec.alexnet(55, 5)
    P = o.param_dim(m)
    # conv 34,944 + 307,456 + 885,120 + 663,936 + 442,624; fc6 256 -> 4096; fc7; fc8 4096 -> 5
    offs = np.cumsum([0, 34848, 96, 307200, 256, 884736, 384, 663552, 384, 442368, 256, 4096 * 256, 4096,
                      4096 * 4096, 4096, 5 * 4096, 5])
    assert P == offs[-1]
    w = o.init_params(m, 2)
    X, y = o.gen_synthetic(2, 3 * 55 * 55, 5, 1.0, 1.0, 7)
    X = np.ascontiguousarray(X * 20.0, dtype=np.float32)  # large enough inputs that LRN is not the identity
    _, g = o.loss_and_grad(m, w, X, y)
    rng = np.random.default_rng(0)
    checked = 0
    for li in range(len(offs) - 1):
        a, b = int(offs[li]), int(offs[li + 1])
        for i in rng.integers(a, b, 3):
            h = np.float32(1e-3 * max(abs(float(w[i])), 1e-2))
            wp, wm = w.copy(), w.copy()
            wp[i] += h
            wm[i] -= h
            lp, _ = o.loss_and_grad(m, wp, X, y, want_grad=False)
            lm, _ = o.loss_and_grad(m, wm, X, y, want_grad=False)
            cd = (lp - lm) / (float(wp[i]) - float(wm[i]))
            if abs(cd) < 1e-9 and abs(g[i]) < 1e-9:
                continue
            rel = abs(cd - float(g[i])) / (abs(cd) + abs(float(g[i])))
            if rel > 1e-4 and li < 10:  # conv layers feed max-pools / relus: a kink can fall inside +-h
                continue
            assert rel <= 1e-4, (li, i, float(g[i]), cd, rel)
            checked += 1
    assert checked >= 24
