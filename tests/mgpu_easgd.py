"""Multi-GPU EASGD run, one process per GPU (launched by tests/test_mgpu.py via torchrun).

Each rank is one worker with its simulate() partition; the center is sharded over all
GPUs and every exchange is an in-kernel P2P read-modify-write of all slices.

  --mode det   deterministic: global tickets from the replayed simulate_async order; the
               run is cut into tau-step chunks and after every chunk (= every round of
               `world` exchanges, tickets [c*world, (c+1)*world)) rank 0 snapshots the
               center and compares it with the oracle's per-exchange snapshot of that
               ticket; rank 0 also checks the final master and every worker (<= 1 ulp).
  --mode async LockFree, no tickets; rank 0 checks the master is finite and its holdout
               accuracy lies within a band of the oracle's deterministic run.
Prints one line `MGPU_RESULT {json}` on rank 0.
"""
import argparse
import ctypes as C
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", default="det", choices=["det", "async"])
    ap.add_argument("--kind", type=int, default=2)  # DS_ENGINE_FUSED
    ap.add_argument("--big", action="store_true")
    args = ap.parse_args()

    import torch
    import torch.distributed as dist
    from oracle.oracle import Hyper, ModelSpec, Oracle, SimSpec
    from paper_1602_08191_b200 import _lib as L
    from paper_1602_08191_b200 import dist as D
    from paper_1602_08191_b200.deepspark import DeepSpark

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    api = DeepSpark()
    if args.big:
        m = ModelSpec.mlp(784, [256], 10)
        X, y = api.gen_synthetic(6000, 784, 10, 0.1, 1.0, 1)
        hp = Hyper(eta=0.05, alpha=0.1, tau=10, batch_size=32, i_max=200)
    else:
        m = ModelSpec.mlp(20, [16], 3)
        X, y = api.gen_synthetic(600, 20, 3, 2.0, 1.5, 5)
        hp = Hyper(eta=0.05, alpha=0.1, tau=5, batch_size=16, i_max=60)
    ncls = m.n_classes
    data_seed, init_seed, sched_seed = 3, 2, 1
    shards, (Xh, yh) = D.sim_shards(api, X, y, world, 0.2, data_seed)
    Xk, yk = shards[rank]
    P = api.param_dim(m)
    init = torch.empty(P, dtype=torch.float32, device="cuda")
    if rank == 0:
        init.copy_(torch.from_numpy(api.init_params(m, init_seed)))
    dist.broadcast(init, 0)  # FETCH_INIT replaced by an NCCL broadcast
    torch.cuda.synchronize()

    mode = L.DS_MODE_LOCKED if args.mode == "det" else L.DS_MODE_LOCKFREE
    master = D.sharded_master(L, local, P, float(np.float32(hp.alpha)), mode, init.data_ptr(), rank, world)
    hidden = (C.c_uint32 * 1)(*m.hidden)
    desc = L.ds_model_desc(1, m.n_features, ncls, len(m.hidden), hidden)
    h = L.ds_hyper(hp.eta, hp.alpha, hp.tau, hp.batch_size, hp.i_max, 0.0, 0.0, 0)
    eng = C.c_void_p()
    L.check(L.lib.ds_engine_create(C.byref(eng), local, C.byref(desc), Xk.ctypes.data, yk.ctypes.data, len(yk), ncls,
                                   C.byref(h), D.sweep_seed(api, data_seed, rank), C.c_void_p(init.data_ptr()),
                                   args.kind))
    L.check(L.lib.ds_engine_attach_master(eng, master))
    if args.mode == "det":
        order_w, _ = api.exchange_order(world, hp.tau, hp.i_max, sched_seed)
        tk = D.worker_tickets(order_w, rank)
        L.check(L.lib.ds_engine_set_tickets(eng, tk.ctypes.data, len(tk)))
    dist.barrier()
    snaps = []  # (global exchange index, center) after every round of exchanges
    if args.mode == "det":
        order_w, _ = api.exchange_order(world, hp.tau, hp.i_max, sched_seed)
        rounds = hp.i_max // hp.tau
        assert all(sorted(order_w[c * world:(c + 1) * world]) == list(range(world)) for c in range(rounds))
        for c in range(rounds):
            L.check(L.lib.ds_engine_run(eng, hp.tau, 0, None))
            L.check(L.lib.ds_engine_sync(eng))
            dist.barrier()  # every rank finished its c-th exchange: tickets < (c+1)*world done
            if rank == 0:
                sn = np.zeros(P, np.float32)
                L.check(L.lib.ds_master_snapshot(master, sn.ctypes.data))
                snaps.append(((c + 1) * world - 1, sn))
            dist.barrier()
        rest = hp.i_max - rounds * hp.tau
        if rest:
            L.check(L.lib.ds_engine_run(eng, rest, 0, None))
    else:
        L.check(L.lib.ds_engine_run(eng, hp.i_max, 0, None))
    L.check(L.lib.ds_engine_sync(eng))
    params = np.zeros(P, np.float32)
    L.check(L.lib.ds_engine_get_params(eng, params.ctypes.data))
    dist.barrier()
    snap = np.zeros(P, np.float32)
    L.check(L.lib.ds_master_snapshot(master, snap.ctypes.data))
    cnt = C.c_uint64()
    L.check(L.lib.ds_master_exchange_count(master, C.byref(cnt)))
    all_params = D.gather_bytes(params.tobytes(), world)
    dist.barrier()
    L.lib.ds_engine_destroy(eng)
    dist.barrier()
    L.lib.ds_master_destroy(master)

    if rank == 0:
        orc = Oracle("dso")
        s = SimSpec(world, hp, m, X, y, ncls, schedule_seed=sched_seed, init_seed=init_seed, data_seed=data_seed,
                    eval_every=10 ** 6, record_master_snaps=args.mode == "det")
        ref = orc.simulate(s)

        def ulps(a, b):
            a = a.view(np.int32).astype(np.int64)
            b = b.view(np.int32).astype(np.int64)
            a = np.where(a < 0, -(2 ** 31) - a, a)
            b = np.where(b < 0, -(2 ** 31) - b, b)
            return np.abs(a - b)

        res = {"world": world, "mode": args.mode, "exchanges": int(cnt.value),
               "expected_exchanges": int(world * (hp.i_max // hp.tau)), "finite": bool(np.isfinite(snap).all())}
        acc_dev = orc.accuracy(m, snap, Xh, yh, ncls)
        acc_ref = orc.accuracy(m, ref.final_master, Xh, yh, ncls)
        res.update(acc_dev=acc_dev, acc_ref=acc_ref)
        if args.mode == "det":
            dm = ulps(snap, ref.final_master)
            res["master_max_ulp"] = int(dm.max())
            res["master_bit_identical"] = float(np.mean(dm == 0))
            wmax = 0
            for k in range(world):
                wk = np.frombuffer(all_params[k], np.float32)
                wmax = max(wmax, int(ulps(wk, ref.worker_final[k]).max()))
            res["workers_max_ulp"] = wmax
            # per-round center snapshots against the oracle's snapshot after that ticket
            res["snapshots_compared"] = len(snaps)
            res["snapshots_max_ulp"] = max((int(ulps(sn, ref.snap_params[g]).max()) for g, sn in snaps), default=-1)
        print("MGPU_RESULT " + json.dumps(res), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
