"""Config 5: EASGD exchange sweep. P in {1M, 4M, 16M, 64M, 256M, 500M} f32
params; single GPU: the fused in-place elastic kernel (16 B/param vs measured HBM peak);
N GPUs (torchrun): every rank exchanges its own worker vector against the center sharded
over all GPUs, concurrently (LockFree), device-timed max over ranks; NVLink bytes per GPU
per direction = 8P(G-1)/G. Prints one JSON object per P (rank 0). Tool only.
  python tools/exchange_sweep.py
  torchrun --nproc-per-node N tools/exchange_sweep.py"""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import torch.distributed as dist
    from paper_1602_08191_b200 import _lib as L
    from paper_1602_08191_b200 import dist as D
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    try:
        peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                           "MEASURED_PEAKS.json"))).get("hbm_gbs", 6552.3)
    except Exception:
        peak = 6552.3
    s = torch.cuda.current_stream()
    nvl = None
    if world > 1:  # in-run NVLink read peak (bench.py's probe: every rank reads its peers concurrently)
        import bench
        nvl = bench.nvlink_peak(L, torch, dist, world, rank, local)
        if rank == 0:
            print(json.dumps({"nvlink_peak": nvl}), flush=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for P in (1 << 20, 4 << 20, 16 << 20, 64 << 20, 256 << 20, 500 * (1 << 20)):
        g = torch.Generator(device="cuda").manual_seed(7 + rank)
        w = torch.rand(P, device="cuda", generator=g) * 2 - 1
        iters = max(5, min(200, (1 << 30) // P))
        if world == 1:
            m = torch.rand(P, device="cuda", generator=g) * 2 - 1
            call = lambda: L.check(L.lib.ds_elastic_update(C.c_void_p(w.data_ptr()), C.c_void_p(m.data_ptr()), P,
                                                            C.c_float(0.1), C.c_void_p(s.cuda_stream)))
        else:
            init = torch.zeros(P, device="cuda")
            mh = D.sharded_master(L, local, P, 0.1, L.DS_MODE_LOCKFREE, init.data_ptr(), rank, world)
            call = lambda: L.check(L.lib.ds_master_exchange(mh, C.c_void_p(w.data_ptr()), C.c_void_p(w.data_ptr()),
                                                             C.c_void_p(s.cuda_stream)))
        for _ in range(3):
            call()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0.record(s)
        for _ in range(iters):
            call()
        e1.record(s)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / iters], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = t.item()
        rec = {"gpus": world, "params": P, "ms": ms, "exchanges_per_s_per_gpu": 1e3 / ms,
               "gbs_per_gpu": 16.0 * P / (ms / 1e3) / 1e9, "frac_hbm": 16.0 * P / (ms / 1e3) / 1e9 / peak}
        # tau: one period = tau local SGD updates of the worker vector (ds_sgd_update in place,
        # 12 B/param, the update a worker applies between exchanges) + one exchange
        gbuf = torch.rand(P, device="cuda", generator=g) * 1e-3
        sgd = lambda: L.check(L.lib.ds_sgd_update(C.c_void_p(w.data_ptr()), C.c_void_p(w.data_ptr()),  # noqa: E731
                                                  C.c_void_p(gbuf.data_ptr()), P, C.c_float(1e-3), C.c_float(0.0),
                                                  None, C.c_void_p(s.cuda_stream)))
        for tau in (1, 4, 16):
            reps = max(2, iters // tau)
            torch.cuda.synchronize()
            if world > 1:
                dist.barrier()
            e0.record(s)
            for _ in range(reps):
                for _ in range(tau):
                    sgd()
                call()
            e1.record(s)
            torch.cuda.synchronize()
            tt = torch.tensor([e0.elapsed_time(e1) / reps], dtype=torch.float64, device="cuda")
            if world > 1:
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            rec[f"tau{tau}"] = {"ms_per_period": tt.item(), "exchanges_per_s_per_gpu": 1e3 / tt.item(),
                                "exchange_share": ms / tt.item()}
        del gbuf
        if world > 1:
            rec["nvlink_gbs_per_gpu_per_dir"] = 8.0 * P * (world - 1) / world / (ms / 1e3) / 1e9
            pk = nvl.get("gbs_per_gpu") if isinstance(nvl, dict) else nvl
            if pk:
                rec["frac_nvlink_peak"] = rec["nvlink_gbs_per_gpu_per_dir"] / pk
            dist.barrier()
            L.lib.ds_master_destroy(mh)
            del init
        else:
            del m
        del w
        torch.cuda.empty_cache()
        if rank == 0:
            print(json.dumps(rec), flush=True)
    if world == 1 and os.environ.get("SWEEP_CPU_REF", "1") == "1":
        # the reference's own exchange beside it: MasterState::exchange
        # of the UNMODIFIED reference (oracle/_ref) in-process on this host — 1 thread Locked,
        # and T threads LockFree; seconds per exchange and GB/s at 16 B/param
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from oracle.oracle import Oracle
        ref = Oracle("dsref")
        T = os.cpu_count() or 1
        for P in (1 << 20, 4 << 20, 16 << 20, 64 << 20, 256 << 20):
            it = max(1, (64 << 20) // P)
            for lockfree, threads in ((False, 1), (True, T)):
                if threads > 1 and P > (64 << 20):
                    continue  # T private worker vectors of 1 GB each
                sec = ref.master_exchange_time(P, lockfree, threads, it) / it
                print(json.dumps({"cpu_reference": True, "params": P, "mode": "LockFree" if lockfree else "Locked",
                                  "threads": threads, "ms_per_exchange_per_thread": sec * 1e3,
                                  "gbs_total": 16.0 * P * threads / sec / 1e9}), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
