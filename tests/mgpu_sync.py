"""Multi-GPU synchronous SGD (simulate_sync semantics), one process per GPU, launched by
tests/test_mgpu.py via torchrun. Every round each rank's gradient is read by every other
rank over NVLink and summed in worker order inside one kernel (ds_sync_reduce_update).
Rank 0 checks the final master (all replicas) and every worker's per-round batch loss
against the CPU oracle's simulate(sync=True): the master bit-identical, the f64 losses
within 1e-14 relative (libm exp/log last-bit differences). Prints `MGPU_RESULT {json}`.
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
    ap.add_argument("--big", action="store_true")
    ap.add_argument("--wd", type=float, default=0.0)
    ap.add_argument("--engine", action="store_true", help="through ds_engine_attach_sync (device sweeper)")
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
        hp = Hyper(eta=0.05, tau=10, batch_size=32, i_max=100, weight_decay=args.wd)
    else:
        m = ModelSpec.mlp(20, [16], 3)
        X, y = api.gen_synthetic(600, 20, 3, 2.0, 1.5, 5)
        hp = Hyper(eta=0.05, tau=5, batch_size=16, i_max=60, weight_decay=args.wd)
    data_seed, init_seed, sched_seed = 3, 2, 1
    shards, (Xh, yh) = D.sim_shards(api, X, y, world, 0.2, data_seed)
    Xk, yk = shards[rank]
    P = api.param_dim(m)
    params = torch.empty(P, dtype=torch.float32, device="cuda")
    if rank == 0:
        params.copy_(torch.from_numpy(api.init_params(m, init_seed)))
    dist.broadcast(params, 0)  # FETCH_INIT replaced by an NCCL broadcast
    torch.cuda.synchronize()
    sg = D.sync_group(L, local, P, rank, world)
    hidden = (C.c_uint32 * 1)(*m.hidden)
    desc = L.ds_model_desc(1, m.n_features, m.n_classes, len(m.hidden), hidden)
    dist.barrier()
    if args.engine:  # the engine's own ShardSweeper + layered kernels, sync group attached
        h = L.ds_hyper(hp.eta, hp.alpha, hp.tau, hp.batch_size, hp.i_max, 0.0, hp.weight_decay, 0)
        eng = C.c_void_p()
        init_host = params.cpu().numpy()
        yk32 = np.ascontiguousarray(yk, dtype=np.uint32)  # kept alive across the create call
        Xk32 = np.ascontiguousarray(Xk, dtype=np.float32)
        L.check(L.lib.ds_engine_create(C.byref(eng), local, C.byref(desc), Xk32.ctypes.data,
                                       yk32.ctypes.data, len(yk), m.n_classes, C.byref(h),
                                       D.sweep_seed(api, data_seed, rank), init_host.ctypes.data, L.DS_ENGINE_LAYERED))
        L.check(L.lib.ds_engine_attach_sync(eng, sg))
        L.check(L.lib.ds_engine_run(eng, hp.i_max, 0, None))
        L.check(L.lib.ds_engine_sync(eng))
        losses = np.zeros(hp.i_max)
        L.check(L.lib.ds_engine_log(eng, 0, hp.i_max, losses.ctypes.data, None, None, None))
        out = np.zeros(P, np.float32)
        L.check(L.lib.ds_engine_get_params(eng, out.ctypes.data))
        params.copy_(torch.from_numpy(out))
        L.lib.ds_engine_destroy(eng)
    else:
        losses = D.run_sync_worker(L, api, desc, Xk, yk, m.n_classes, hp, D.sweep_seed(api, data_seed, rank), params,
                                   sg, local)
    final = params.cpu().numpy()
    finals = D.gather_bytes(final.tobytes(), world)
    all_losses = D.gather_bytes(losses.tobytes(), world)
    rounds = C.c_uint64()
    L.check(L.lib.ds_sync_rounds(sg, C.byref(rounds)))
    dist.barrier()
    L.lib.ds_sync_destroy(sg)
    if rank == 0:
        orc = Oracle("dso")
        s = SimSpec(world, hp, m, X, y, m.n_classes, sync=True, schedule_seed=sched_seed, init_seed=init_seed,
                    data_seed=data_seed, eval_every=10 ** 6, record_master_snaps=False)
        ref = orc.simulate(s)
        ref_loss = np.asarray(ref.batch_loss).reshape(world, -1)

        def ulps(a, b):
            a = a.view(np.int32).astype(np.int64)
            b = b.view(np.int32).astype(np.int64)
            a = np.where(a < 0, -(2 ** 31) - a, a)
            b = np.where(b < 0, -(2 ** 31) - b, b)
            return np.abs(a - b)
        res = {"world": world, "rounds": int(rounds.value), "i_max": hp.i_max,
               "replicas_identical": all(f == finals[0] for f in finals),
               "master_equal": bool(np.array_equal(np.frombuffer(finals[0], np.float32).view(np.uint32),
                                                   ref.final_master.view(np.uint32))),
               "master_max_ulp": int(ulps(np.frombuffer(finals[0], np.float32), ref.final_master).max()),
               "master_bit_identical": float(np.mean(ulps(np.frombuffer(finals[0], np.float32),
                                                          ref.final_master) == 0)),
               # losses go through exp/log (CUDA's vs glibc's: either may differ in the last
               # bit); the f32 master is bit-identical
               "loss_close": all(np.allclose(np.frombuffer(all_losses[k], np.float64), ref_loss[k], rtol=1e-14,
                                             atol=0.0) for k in range(world)),
               "loss_max_abs_diff": max(float(np.max(np.abs(np.frombuffer(all_losses[k], np.float64) - ref_loss[k])))
                                        for k in range(world)),
               "loss_first": [float(np.frombuffer(all_losses[0], np.float64)[0]), float(ref_loss[0][0])],
               "acc_dev": orc.accuracy(m, np.frombuffer(finals[0], np.float32).copy(), Xh, yh, m.n_classes),
               "acc_ref": orc.accuracy(m, ref.final_master, Xh, yh, m.n_classes)}
        print("MGPU_RESULT " + json.dumps(res), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
