"""Parity of the reference-compatible API (libdeepspark_b200.so via deepspark_c.h) with the
CPU oracle on identical inputs and seeds.

Host-side pieces (Rng streams, data generation, splits, sweep orders, init, layout) are
bit-exact. Device numerics (loss_and_grad, engine, simulate) follow the reference's f64
operation order; the only non-reproduced operations are CUDA's double tanh/exp/log vs
glibc's, so the stated tolerance is: batch losses to 1e-13 relative, f32 parameters and
master snapshots within 1 ulp per element (observed: bit-identical), identical exchange
decisions, identical eval-curve accuracies."""
import numpy as np
import pytest

from oracle.oracle import Hyper, ModelSpec, Oracle, SimSpec


@pytest.fixture(scope="module")
def orc():
    return Oracle("dso")


@pytest.fixture(scope="module")
def dev():
    from paper_1602_08191_b200.deepspark import DeepSpark
    return DeepSpark()


def ulps(a, b):
    a = np.asarray(a, np.float32).view(np.int32).astype(np.int64)
    b = np.asarray(b, np.float32).view(np.int32).astype(np.int64)
    ka = np.where(a < 0, np.int64(-2**31) - a, a)
    kb = np.where(b < 0, np.int64(-2**31) - b, b)
    return np.abs(ka - kb)


# ---- host-only (no GPU needed) --------------------------------------------------------

def test_rng_streams_bit_exact(orc, dev):
    for seed in (0, 1, 2026, 2**63 + 5):
        for a, b in zip(orc.rng_draws(seed, 2000, 97), dev.rng_draws(seed, 2000, 97)):
            assert np.array_equal(a.view(np.uint64), b.view(np.uint64))
    assert orc.mix_seed(7, 9) == dev.mix_seed(7, 9)


@pytest.mark.parametrize("spec", [(300, 20, 2, 10.0, 0.5, 31), (2000, 16, 8, 2.0, 2.0, 99), (500, 784, 10, 0.1, 1.0, 1)])
def test_gen_synthetic_bit_exact(orc, dev, spec):
    Xa, ya = orc.gen_synthetic(*spec)
    Xb, yb = dev.gen_synthetic(*spec)
    assert np.array_equal(Xa.view(np.uint32), Xb.view(np.uint32)) and np.array_equal(ya, yb)


def test_orders_bit_exact(orc, dev):
    for n, frac, seed in ((300, 0.2, 9), (2000, 0.25, 4), (7, 0.5, 1)):
        a, ha = orc.split_holdout_order(n, frac, seed)
        b, hb = dev.split_holdout_order(n, frac, seed)
        assert ha == hb and np.array_equal(a, b)
    for n, k, seed in ((300, 7, 9), (48000, 8, 3)):
        assert np.array_equal(orc.partition_order(n, k, seed), dev.partition_order(n, k, seed))
    for n, b, seed in ((100, 32, 4), (10, 4, 77), (48000, 32, 5)):
        ia, sa = orc.sweep_batches(n, b, seed, 40)
        ib, sb = dev.sweep_batches(n, b, seed, 40)
        assert np.array_equal(sa, sb)
        for j in range(40):
            assert np.array_equal(ia[j, :sa[j]], ib[j, :sb[j]])


@pytest.mark.parametrize("m", [ModelSpec.softmax(20, 2), ModelSpec.mlp(4, [8], 3), ModelSpec.mlp(784, [256], 10),
                               ModelSpec.mlp(5, [6, 7], 4), ModelSpec.cifar10_quick(10), ModelSpec.alexnet(55, 5),
                               ModelSpec.alexnet(224, 1000)])
def test_layout_init_fingerprint(orc, dev, m):
    assert orc.param_dim(m) == dev.param_dim(m)
    assert orc.fingerprint(m) == dev.fingerprint(m)
    assert np.array_equal(orc.init_params(m, 42).view(np.uint32), dev.init_params(m, 42).view(np.uint32))


# ---- device numerics ----------------------------------------------------------------------

@pytest.mark.gpu
def test_sgd_and_elastic_bit_exact(orc, dev):
    rng = np.random.default_rng(3)
    x = rng.standard_normal(5000).astype(np.float32)
    g = rng.standard_normal(5000).astype(np.float32)
    assert np.array_equal(orc.sgd_step(x, g, 0.05).view(np.uint32), dev.sgd_step(x, g, 0.05).view(np.uint32))
    for a, b in zip(orc.easgd_update(x, g, 0.3), dev.easgd_update(x, g, 0.3)):
        assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


@pytest.mark.gpu
def test_loss_grad_predict_accuracy(orc, dev):
    m = ModelSpec.mlp(20, [16], 3)
    X, y = orc.gen_synthetic(200, 20, 3, 2.0, 1.5, 5)
    p = orc.init_params(m, 1)
    la, ga = orc.loss_and_grad(m, p, X[:32], y[:32])
    lb, gb = dev.loss_and_grad(m, p, X[:32], y[:32])
    assert abs(la - lb) <= 1e-13 * abs(la) and ulps(ga, gb).max() <= 1
    assert np.array_equal(orc.predict(m, p, X), dev.predict(m, p, X))
    assert orc.accuracy(m, p, X, y, 3) == dev.accuracy(m, p, X, y, 3)


@pytest.mark.gpu
@pytest.mark.parametrize("mode", [0, 1, 2])
def test_run_training_loop(orc, dev, mode):
    m = ModelSpec.mlp(20, [16], 3)
    X, y = orc.gen_synthetic(300, 20, 3, 2.0, 1.5, 3)
    init = orc.init_params(m, 9)
    master = orc.init_params(m, 10)
    hp = Hyper(eta=0.05, tau=5, batch_size=16, i_max=40)
    a = orc.run_training_loop(m, X, y, 3, hp, 31, init, mode, master)
    b = dev.run_training_loop(m, X, y, 3, hp, 31, init, mode, master)
    np.testing.assert_allclose(a["batch_loss"], b["batch_loss"], rtol=1e-13)
    assert np.array_equal(a["exchanged"], b["exchanged"]) and np.array_equal(a["period_len"], b["period_len"])
    assert ulps(a["final_params"], b["final_params"]).max() <= 1
    if mode == 2:
        assert ulps(a["master"], b["master"]).max() <= 1


def sim_spec(orc, n=3, sync=False, adaptive=False, model=None, i_max=40, tau=5, S=0.0, mults=None, rep=False,
             wd=0.0, nsamp=300):
    m = model or ModelSpec.mlp(20, [16], 3)
    X, y = orc.gen_synthetic(nsamp, m.n_features, m.n_classes, 2.0, 1.0, 5)
    return SimSpec(n, Hyper(eta=0.05, tau=tau, batch_size=16, i_max=i_max, adaptive=adaptive, weight_decay=wd), m,
                   X, y, m.n_classes, sync=sync, schedule_seed=1, init_seed=2, data_seed=3, eval_every=10,
                   comm_cost_S=S, cost_multipliers=mults, replicate_shards=rep)


SIMS = {
    "async3": dict(),
    "async-costs": dict(S=0.5, mults=[1, 1.5, 1]),
    "async-adaptive": dict(adaptive=True, i_max=60),
    "async-softmax": dict(model=ModelSpec.softmax(20, 3)),
    "async-2layer": dict(model=ModelSpec.mlp(20, [12, 8], 3), n=2),
    "sync": dict(sync=True),
    "sync-replicated-wd": dict(sync=True, rep=True, wd=0.01),
}


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(SIMS))
def test_simulate_matches_oracle(orc, dev, name):
    s = sim_spec(orc, **SIMS[name])
    a = orc.simulate(s)
    b = dev.simulate(s)
    np.testing.assert_allclose(a.batch_loss, b["batch_loss"], rtol=1e-13)
    np.testing.assert_allclose(a.cumulated, b["cumulated"], rtol=1e-12, atol=1e-300)
    assert np.array_equal(a.exchanged, b["exchanged"])
    assert np.array_equal(a.period_len, b["period_len"])
    assert np.array_equal(a.wall_ms, b["wall_ms"])
    assert a.n_snaps == b["n_snaps"]
    assert np.array_equal(a.snap_worker, b["snap_worker"]) and np.array_equal(a.snap_time, b["snap_time"])
    assert ulps(a.snap_params, b["snap_params"]).max(initial=0) <= 1
    assert ulps(a.final_master, b["final_master"]).max() <= 1
    assert ulps(a.worker_final, b["worker_final"]).max() <= 1
    assert np.array_equal(a.eval_iter, b["eval_iter"]) and np.array_equal(a.eval_time, b["eval_time"])
    assert np.array_equal(a.eval_acc, b["eval_acc"])
    assert a.virtual_total == b["virtual_total"]
    same = np.mean(ulps(a.final_master, b["final_master"]) == 0)
    print(f"{name}: final master bit-identical fraction {same:.6f}")


@pytest.mark.gpu
def test_config1_two_worker_deterministic(orc, dev):
    """BASELINE config 1: MLP 784-256-10, 2 workers, tau=10, alpha=0.1, deterministic
    schedule (simulate_async's seeded event order) — per-exchange master snapshots."""
    m = ModelSpec.mlp(784, [256], 10)
    X, y = orc.gen_synthetic(6000, 784, 10, 0.1, 1.0, 1)
    s = SimSpec(2, Hyper(eta=0.05, alpha=0.1, tau=10, batch_size=32, i_max=150), m, X, y, 10, schedule_seed=1,
                init_seed=2, data_seed=3, eval_every=50)
    a = orc.simulate(s)
    b = dev.simulate(s)
    np.testing.assert_allclose(a.batch_loss, b["batch_loss"], rtol=1e-13)
    assert np.array_equal(a.snap_worker, b["snap_worker"])
    d = ulps(a.snap_params, b["snap_params"])
    assert d.max() <= 1
    assert np.array_equal(a.eval_acc, b["eval_acc"])
    print(f"config1: {a.n_snaps} exchanges, snapshots bit-identical fraction {np.mean(d == 0):.7f}, "
          f"final acc {b['eval_acc'][-1]:.4f}")


# ---- run_worker over the device path (worker.cpp:52-98; test_worker.cpp:122-260) ---------

def _worker_fixture(orc, tmp_path, sep=10.0, sigma=0.5, name="shard_0.dshd"):
    """test_worker.cpp's Fixture: standard_benchmark(12) with 120 samples, softmax model,
    the shard spilled to DSHD (seed 7)."""
    from test_shard import write_dshd
    X, y = orc.gen_synthetic(120, 20, 2, sep, sigma, 12)
    path = str(tmp_path / name)
    write_dshd(path, X, y, seed=7, c=2)
    return X, y, path


@pytest.mark.gpu
def test_run_worker_equals_in_process_loop(orc, dev, tmp_path):
    """test_worker.cpp:122-147: the worker through the device exchanger equals the
    in-process training loop with exchanges applied to a local master copy."""
    X, y, path = _worker_fixture(orc, tmp_path)
    m = ModelSpec.softmax(20, 2)
    init = orc.init_params(m, 55)
    hp = Hyper(eta=0.05, alpha=0.1, tau=5, batch_size=16, i_max=20)
    got = dev.run_worker(m, 0.1, init, path, hp, rng_seed=3, metrics_path=str(tmp_path / "w.csv"))
    ref = orc.run_training_loop(m, X, y, 2, hp, 3, init, 2, init)  # ExchangeFn on a host master
    np.testing.assert_allclose(got["batch_loss"], ref["batch_loss"], rtol=1e-13)
    assert np.array_equal(got["exchanged"], ref["exchanged"]) and np.array_equal(got["period_len"],
                                                                                 ref["period_len"])
    assert ulps(got["final_params"], ref["final_params"]).max() <= 1
    assert ulps(got["master"], ref["master"]).max() <= 1
    assert got["exchanges"] == 4  # iterations 5, 10, 15, 20


@pytest.mark.gpu
def test_run_worker_writes_metrics_and_params(orc, dev, tmp_path):
    """test_worker.cpp:149-165 + the byte-identical-logs case (167-182)."""
    import csv
    X, y, path = _worker_fixture(orc, tmp_path)
    m = ModelSpec.softmax(20, 2)
    init = orc.init_params(m, 55)
    hp = Hyper(eta=0.05, alpha=0.1, tau=5, batch_size=16, i_max=20)
    res = dev.run_worker(m, 0.1, init, path, hp, rng_seed=3, metrics_path=str(tmp_path / "run.csv"))
    rows = list(csv.DictReader(open(tmp_path / "run.csv")))
    assert len(rows) == 20
    for i, r in enumerate(rows):
        assert int(r["exchanged"]) == ((i + 1) % 5 == 0)
        assert float(r["batch_loss"]) == res["batch_loss"][i]  # shortest round-trip text
        assert float(r["cumulated_loss"]) == res["cumulated"][i]
    params = np.array([float(v) for v in open(tmp_path / "run.params").read().split()], np.float32)
    assert np.array_equal(params.view(np.uint32), res["final_params"].view(np.uint32))
    dev.run_worker(m, 0.1, init, path, hp, rng_seed=3, metrics_path=str(tmp_path / "run2.csv"))
    strip = lambda p: [",".join(l.split(",")[:1] + l.split(",")[2:]) for l in open(p).read().splitlines()]
    assert strip(tmp_path / "run.csv") == strip(tmp_path / "run2.csv")  # wall_ms column aside


@pytest.mark.gpu
def test_run_worker_adaptive_resolves_cut(orc, dev, tmp_path):
    """test_worker.cpp:184-214: a hard shard, loss_cut resolved from the first batch."""
    X, y, path = _worker_fixture(orc, tmp_path, sep=0.5, sigma=3.0, name="shard_9.dshd")
    m = ModelSpec.softmax(20, 2)
    init = orc.init_params(m, 55)
    hp = Hyper(eta=0.05, alpha=0.1, tau=5, batch_size=16, i_max=100, adaptive=True, loss_cut=0.0)
    res = dev.run_worker(m, 0.1, init, path, hp, rng_seed=3)
    ref = orc.run_training_loop(m, X, y, 2, Hyper(eta=0.05, alpha=0.1, tau=5, batch_size=16, i_max=100,
                                                   adaptive=True,
                                                   loss_cut=orc.resolve_loss_cut(m, X, y, 2, hp, 3, init)),
                                3, init, 2, init)
    assert int(res["exchanged"].sum()) == res["exchanges"] >= 1
    assert np.array_equal(res["exchanged"], ref["exchanged"])
    np.testing.assert_allclose(res["batch_loss"], ref["batch_loss"], rtol=1e-13)


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["alpha", "model", "shard", "no_master_dim"])
def test_run_worker_handshake_errors(orc, dev, tmp_path, case):
    """test_worker.cpp:216-242: disagreement with the exchanger is fatal before training
    (the center is untouched, no exchange happened)."""
    from paper_1602_08191_b200.deepspark import ContractError
    X, y, path = _worker_fixture(orc, tmp_path)
    m = ModelSpec.softmax(20, 2)
    init = orc.init_params(m, 55)
    hp = Hyper(eta=0.05, alpha=0.1, tau=5, batch_size=16, i_max=20)
    kw = {}
    served = m
    if case == "alpha":
        hp = Hyper(eta=0.05, alpha=0.2, tau=5, batch_size=16, i_max=20)  # server says 0.1
    elif case == "model":
        kw["worker_model"] = ModelSpec.mlp(20, [4], 2)  # different fingerprint (and dim)
    elif case == "shard":
        kw["worker_model"] = ModelSpec.softmax(21, 2)
    else:  # same fingerprint family, different dim served: softmax(20, 3)
        served = ModelSpec.softmax(20, 3)
        init = orc.init_params(served, 55)
        kw["worker_model"] = m
    with pytest.raises(ContractError):
        dev.run_worker(served, 0.1, init, path, hp, rng_seed=3, **kw)
