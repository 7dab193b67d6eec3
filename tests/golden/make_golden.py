"""Generates tests/golden/golden.npz from the UNMODIFIED reference (oracle/_ref, built from
/root/reference/proj/src by `make -C oracle ref`). Run in the build container:

    python tests/golden/make_golden.py

The fixtures pin the C restatement (oracle/ds_oracle.c) and the product without needing
/root/reference at test time. Sizes are small so the file stays light.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import Hyper, ModelSpec, Oracle, SimSpec  # noqa: E402


def main():
    ref = Oracle("dsref")
    g = {}
    # Rng streams (rng.hpp:11-68)
    for seed in (0, 2026, 12345678901234):
        u, uni, nrm, bel = ref.rng_draws(seed, 64, 97)
        g[f"rng_{seed}_u64"], g[f"rng_{seed}_uni"], g[f"rng_{seed}_nrm"], g[f"rng_{seed}_below97"] = u, uni, nrm, bel
    g["mix_seed"] = np.array([ref.mix_seed(s, t) for s in (0, 1, 99) for t in (0, 1, 0x1e17)], np.uint64)
    # data (dataset.cpp)
    X, y = ref.gen_synthetic(200, 12, 3, 2.0, 1.0, 7)
    g["syn_X"], g["syn_y"] = X, y
    o, nh = ref.split_holdout_order(200, 0.2, 5)
    g["holdout_order"], g["holdout_n"] = o, np.array([nh])
    g["partition_order"] = ref.partition_order(160, 3, 5)
    idx, sizes = ref.sweep_batches(50, 16, 9, 10)
    g["sweep_idx"], g["sweep_sizes"] = idx, sizes
    # model (model.cpp)
    specs = {"softmax": ModelSpec.softmax(12, 3), "mlp": ModelSpec.mlp(12, [10], 3), "mlp2": ModelSpec.mlp(12, [8, 6], 3)}
    for name, m in specs.items():
        p = ref.init_params(m, 11)
        g[f"{name}_init"] = p
        g[f"{name}_fp"] = np.array([ref.fingerprint(m)], np.uint64)
        loss, grad = ref.loss_and_grad(m, p, X[:16], y[:16])
        g[f"{name}_loss"], g[f"{name}_grad"] = np.array([loss]), grad
        lo, _ = ref.loss_and_grad(m, p, X[:16], y[:16], want_grad=False)
        g[f"{name}_loss_only"] = np.array([lo])
        g[f"{name}_pred"] = ref.predict(m, p, X)
    # updates (param_vector.cpp)
    rng = np.random.default_rng(1)
    w = rng.standard_normal(257).astype(np.float32)
    mm = rng.standard_normal(257).astype(np.float32)
    g["upd_w"], g["upd_m"] = w, mm
    g["easgd_w"], g["easgd_m"] = ref.easgd_update(w, mm, 0.1)
    g["sgd_out"] = ref.sgd_step(w, mm, 0.05)
    # run_training_loop with a local master (engine.cpp:84-113, test_worker.cpp:131-137)
    m = specs["mlp"]
    hp = Hyper(eta=0.05, tau=4, batch_size=16, i_max=24)
    init = ref.init_params(m, 3)
    master = ref.init_params(m, 4)
    r = ref.run_training_loop(m, X, y, 3, hp, 21, init, 2, master)
    for k in ("final_params", "batch_loss", "cumulated", "exchanged", "period_len", "master"):
        g[f"loop_{k}"] = r[k]
    # simulate (simulator.cpp) — async with costs, and sync
    for name, sync in (("async", False), ("sync", True)):
        s = SimSpec(3, Hyper(eta=0.05, tau=4, batch_size=16, i_max=20), m, X, y, 3, sync=sync, schedule_seed=1,
                    init_seed=2, data_seed=3, eval_every=5, comm_cost_S=0.5, cost_multipliers=[1.0, 1.5, 1.0])
        o = ref.simulate(s)
        for k in ("final_master", "worker_final", "batch_loss", "cumulated", "exchanged", "period_len", "wall_ms",
                  "snap_worker", "snap_time", "snap_params", "eval_time", "eval_iter", "eval_acc"):
            g[f"sim_{name}_{k}"] = getattr(o, k)
        g[f"sim_{name}_virtual_total"] = np.array([o.virtual_total])
    out = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")
    np.savez_compressed(out, **g)
    # a DSHD shard written by the reference's write_shard (shard.cpp:40-73): pins the
    # device ingestion (ds_shard_load) and the header checks
    import ctypes as C
    Xs, ys = ref.gen_synthetic(37, 9, 4, 2.0, 1.0, 17)
    fn = ref.lib.dsref_write_shard
    fn.argtypes = [C.c_char_p, C.c_void_p, C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint64]
    fn.restype = C.c_int
    path = os.path.join(os.path.dirname(out), "ref_small.dshd")
    assert fn(path.encode(), Xs.ctypes.data, ys.ctypes.data, len(ys), 9, 4, 0xFEED) == 0
    np.savez_compressed(os.path.join(os.path.dirname(out), "ref_small_dshd.npz"), X=Xs, y=ys)
    print(f"wrote {out}: {len(g)} arrays, {os.path.getsize(out)} bytes")


if __name__ == "__main__":
    main()
