#!/usr/bin/env python3
"""bench.py — throughput of the B200 EASGD hot path (BASELINE.json metric).

Workload (config 1 shapes, one worker per GPU): MLP 784-256-10 (tanh), batch 32 per
worker, async EASGD with tau=10, alpha=0.1, eta=0.05, on synthetic MNIST-shaped data
made by the reference's own generator (gen_synthetic N=60000, sep 0.1, sigma 1.0; each
GPU draws its own partition with seed 1+rank, the holdout split of the reference's
simulator is removed, 48,000 rows = 150 MB stay resident per GPU, larger than L2).

A "step" is one local SGD iteration on every GPU; every tau-th step also performs the
elastic exchange with the center, which is sharded over all GPUs (LockFree, in-kernel
P2P read-modify-write over NVLink). value = all samples processed / max-over-ranks
device time. e2e = the same loop through the C-ABI with host buffers: every step
copies its gathered batch from pinned host memory and reads the batch loss back.

  python bench.py [--gpus N --steps K --warmup W]          # our B200 arm
  python bench.py --impl reference [...]                   # the reference CPU arm
  torchrun --nproc-per-node N bench.py --gpus N ...        # N > 1
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "train samples/sec @1/2/4/8 B200; EASGD exchange GB/s vs HBM/NVLink peak"
F, H, NCLS = 784, 256, 10
N_SAMPLES, SEP, SIGMA = 60000, 0.1, 1.0
INIT_SEED, DATA_SEED = 2, 3
FLOP_PER_SAMPLE = 818_176  # fwd 203,264 MAC + dW 203,264 MAC + dX 2,560 MAC, x2


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3000)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=32)
    ap.add_argument("--tau", type=int, default=10)
    ap.add_argument("--e2e-steps", type=int, default=2000)
    ap.add_argument("--exchange-params", type=int, default=256 * 1024 * 1024)
    ap.add_argument("--no-extras", action="store_true", help="skip e2e / exchange sweep / cpu baseline (profiling)")
    ap.add_argument("--cifar-steps", type=int, default=200, help="timed steps of the cifar10_quick leg (0 = skip)")
    ap.add_argument("--alexnet-steps", type=int, default=20, help="timed steps of the AlexNet leg (0 = skip)")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p.get("hbm_gbs", 6552.3), p.get("bf16_tflops", 1646.8), p.get("bf16_tflops_sustained", 1400.2), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


def worker_data(rank, api):
    """Rank's synthetic partition: gen_synthetic (seed 1+rank) minus the simulator's holdout."""
    X, y = api.gen_synthetic(N_SAMPLES, F, NCLS, SEP, SIGMA, 1 + rank)
    order, nh = api.split_holdout_order(N_SAMPLES, 0.2, api.mix_seed(DATA_SEED, 0x484f4c44))
    tr = order[nh:]
    return np.ascontiguousarray(X[tr]), np.ascontiguousarray(y[tr])


class ClockSampler:
    """nvidia-smi clocks + throttle reasons while the timed region runs."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.rows = []

    def __enter__(self):
        if os.environ.get("DS_BENCH_NO_CLOCKS"):
            return self
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi's start-up (NVML init) stalls the device for a moment: let it
            # finish before the caller records its start event
            t0 = time.time()
            while not self.rows and time.time() - t0 < 5.0:
                time.sleep(0.01)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit())
        mx = max(float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit())
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = [n for i, n in enumerate(names) if any(r[3 + i].lower() == "active" for r in self.rows)]
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(self.rows)}


def run_reference(args):
    """The reference's own CPU path: n worker threads (SgdEngine + ExchangePolicy +
    in-process MasterState), timed on the host cores of this box."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle.oracle import Oracle, ModelSpec, Hyper, available
    kind = "reference" if available("dsref") else "port"
    orc = Oracle("dsref" if kind == "reference" else "dso")
    n = max(1, args.gpus)
    m = ModelSpec.mlp(F, [H], NCLS)
    hp = Hyper(eta=0.05, alpha=0.1, tau=args.tau, batch_size=args.batch, i_max=10 ** 9)
    shards = [worker_data(k, orc) for k in range(n)]
    init = orc.init_params(m, INIT_SEED)
    if kind == "reference":
        probe = orc.workers_time(m, shards, NCLS, hp, init, True, 1, 5)  # calibrate: ~5 steps
        per = max(probe / 5, 1e-4)
        steps = int(min(args.steps, max(20, 60.0 / per)))  # bounded: <= ~1 min of CPU
        warm = int(min(args.warmup, max(3, 5.0 / per)))
        secs = orc.workers_time(m, shards, NCLS, hp, init, True, warm, steps)
    else:  # C restatement, single worker only
        t0 = time.perf_counter()
        orc.engine_steps(m, shards[0][0], shards[0][1], NCLS, hp, 7, init, 5)
        per = (time.perf_counter() - t0) / 5
        steps = int(min(args.steps, max(20, 60.0 / per)))
        warm = 0
        t0 = time.perf_counter()
        orc.engine_steps(m, shards[0][0], shards[0][1], NCLS, hp, 7, init, steps)
        secs = time.perf_counter() - t0
        n = 1
    value = n * args.batch * steps / secs
    all_cores = None
    if kind == "reference":
        # The same loop with one worker thread per host core (up to 64), for scale: the
        # reference parallelises only across workers (each SgdEngine step is one thread),
        # so this is its whole-box throughput; `value` stays on this arm's config.
        W = max(1, min(os.cpu_count() or 1, 64))
        if W > n:
            small = (shards[0][0][:4800], shards[0][1][:4800])  # batch cost does not depend on shard size
            steps_w = int(min(args.steps, max(10, 20.0 / per)))
            secs_w = orc.workers_time(m, [small] * W, NCLS, hp, init, True, 3, steps_w)
            all_cores = {"workers": W, "value": W * args.batch * steps_w / secs_w, "unit": "samples/s",
                         "steps": steps_w,
                         "note": "reference n-worker loop, one thread per host core, LockFree in-process "
                                 "MasterState; not this arm's config (one worker per GPU)"}
    line = {"metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": args.gpus, "steps": steps,
            "warmup": warm, "ms_per_step": 1000.0 * secs / steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference gen_synthetic, per-worker seeds)",
            "impl": "reference",
            "config": config_block(args, n),
            "cpu_baseline": {"value": value, "unit": "samples/s", "cores": n, "kind": kind,
                             "sample": f"{steps} timed iterations per worker x {n} worker thread(s) "
                                       f"(+{warm} warmup), LockFree in-process MasterState, tau={args.tau}"},
            "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if all_cores:
        line["all_cores"] = all_cores
    print(json.dumps(line), flush=True)
    return 0


def config_block(args, n):
    return {"workload": "mlp784-256-10 async EASGD (BASELINE config 1 shapes, one worker per GPU)",
            "model": "mlp:784:256:10 (tanh hidden, softmax CE)", "global_batch": args.batch * n,
            "batch_per_worker": args.batch, "seq_len": None, "tau": args.tau, "alpha": 0.1, "eta": 0.05,
            "workers": n, "parallelism": f"easgd-dp{n}",
            "exchange": "LockFree, center sharded over the GPUs, in-kernel P2P RMW" if n > 1 else
                        "LockFree, center on the same GPU, in-kernel",
            "l2_policy": "inputs larger than L2: 48,000-row (150 MB) shard per GPU, random batches",
            "numerics": "f64 accumulation in the reference's summation order, f32 params"}


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist
    from paper_1602_08191_b200 import _lib as L
    from paper_1602_08191_b200.deepspark import DeepSpark

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    api = DeepSpark()
    n = world
    hbm, bf16, bf16_sus, peak_kind = peaks()

    # ---- data, init (NCCL broadcast), master, engine --------------------------------
    X, y = worker_data(rank, api)
    P = (H * F + H) + (NCLS * H + NCLS)
    init = torch.empty(P, dtype=torch.float32, device="cuda")
    if rank == 0:
        from paper_1602_08191_b200.deepspark import Model
        init.copy_(torch.from_numpy(api.init_params(Model.mlp(F, [H], NCLS), INIT_SEED)))
    if world > 1:
        dist.broadcast(init, 0)  # replaces FETCH_INIT (exchanger.cpp:266-270)
    torch.cuda.synchronize()

    master = C.c_void_p()
    if world == 1:
        L.check(L.lib.ds_master_create(C.byref(master), local, P, C.c_float(0.1), L.DS_MODE_LOCKFREE,
                                       C.c_void_p(init.data_ptr())))
    else:
        L.check(L.lib.ds_master_create_sharded(C.byref(master), local, P, C.c_float(0.1), L.DS_MODE_LOCKFREE,
                                               rank, world, C.c_void_p(init.data_ptr())))
        rec = (C.c_uint8 * L.DS_IPC_RECORD_BYTES)()
        L.check(L.lib.ds_master_export(master, rec))
        recs = [None] * world
        dist.all_gather_object(recs, bytes(rec))
        allrec = (C.c_uint8 * (L.DS_IPC_RECORD_BYTES * world)).from_buffer_copy(b"".join(recs))
        L.check(L.lib.ds_master_attach(master, allrec))
        dist.barrier()

    hidden = (C.c_uint32 * 1)(H)
    desc = L.ds_model_desc(1, F, NCLS, 1, hidden)
    hp = L.ds_hyper(0.05, 0.1, args.tau, args.batch, 10 ** 9, 0.0, 0.0, 0)
    sweep_seed = api.mix_seed(api.mix_seed(DATA_SEED, 0x53574550), rank)
    eng = C.c_void_p()
    L.check(L.lib.ds_engine_create(C.byref(eng), local, C.byref(desc), X.ctypes.data, y.ctypes.data, len(y), NCLS,
                                   C.byref(hp), sweep_seed, C.c_void_p(init.data_ptr()), L.DS_ENGINE_AUTO))
    L.check(L.lib.ds_engine_attach_master(eng, master))
    sptr = C.c_void_p()
    L.check(L.lib.ds_engine_stream(eng, C.byref(sptr)))
    stream = torch.cuda.ExternalStream(sptr.value)

    # ---- warmup, then K timed steps in one device run -----------------------------------
    W, K = max(3, args.warmup), args.steps
    L.check(L.lib.ds_engine_reserve(eng, W + K))  # no allocation inside the timed region
    L.check(L.lib.ds_engine_run(eng, W, 0, None))
    L.check(L.lib.ds_engine_sync(eng))
    launches0 = C.c_uint64()
    L.check(L.lib.ds_engine_launches(eng, C.byref(launches0)))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        L.check(L.lib.ds_engine_run(eng, K, 0, None))
        ev1.record(stream)
        L.check(L.lib.ds_engine_sync(eng))
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    launches1 = C.c_uint64()
    L.check(L.lib.ds_engine_launches(eng, C.byref(launches1)))
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = t.item()
    value = n * args.batch * K / (ms_max / 1e3)

    # roofline of the dominant (and only) kernel of the timed region: the fused step
    flop_launch = FLOP_PER_SAMPLE * args.batch * K
    achieved = flop_launch / (ms / 1e3) / 1e12
    # The launch is the only kernel of the timed region. Its contract bound is reported
    # against the tensor peak (FLOPs), but the path is exact-order f64 on CUDA cores, so
    # the binding roofline is the FP64 pipe: 148 SMs x 64 DADD/DMUL lanes per clock.
    sm_clk = (clk.summary().get("sm_mhz") or 1965.0) * 1e6
    fp64_peak = 148 * 64 * sm_clk / 1e12  # TFLOP/s (one op per DADD/DMUL lane)
    traffic = 32 * 3136 * K  # ncu dram bytes per launch = the X rows (profiles/r01_fused_kernel_ncu.md)
    roof = {"bound": "tensor", "achieved": achieved, "peak": bf16_sus, "unit": "TFLOP/s", "frac": achieved / bf16_sus,
            "traffic": traffic, "peak_kind": f"{peak_kind} bf16 dense, sustained",
            "kernel": "mlp_kernel (persistent: forward, softmax-CE, backward, SGD, policy, exchange)",
            "algorithmic": f"{FLOP_PER_SAMPLE} FLOP/sample x {args.batch} x {K} steps per launch",
            "fp64_pipe": {"achieved_tflops": achieved, "peak_tflops": fp64_peak, "frac": achieved / fp64_peak,
                          "note": "the reference's sequential f64 order (bit parity) keeps every FLOP on the FP64 "
                                  "pipe; ncu: FP64 pipe active 12.5% of elapsed, 1 grid barrier per step"},
            "note": "latency-bound f64 CUDA-core chains (784-long dependent DADD chains per hidden unit), "
                    "not a tensor-core kernel; traffic = X rows only (22.5 MB DRAM read per 200-step launch)"}

    line = {"metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": n, "steps": K, "warmup": W,
            "ms_per_step": ms_max / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic (reference gen_synthetic, per-GPU seeds)",
            "config": config_block(args, n), "roofline": roof, "clocks": clk.summary(),
            "gpu_launches": int(launches1.value - launches0.value)}

    if not args.no_extras:
        line["e2e"] = e2e_leg(args, L, api, eng, X, y, rank, world, sweep_seed, n)
        line["exchange"] = exchange_leg(args, L, torch, dist, world, rank, local, hbm, peak_kind)
    if args.cifar_steps > 0:
        line["cifar10_quick"] = cifar_leg(args, L, api, torch, dist, world, rank, local)
        line["cifar10_quick_config3"] = {k: cifar_leg(args, L, api, torch, dist, world, rank, local, k)
                                         for k in ("sync", "adaptive")}
    if args.alexnet_steps > 0:
        line["alexnet"] = alexnet_leg(args, L, api, torch, dist, world, rank, local)
    if not args.no_extras:
        if rank == 0 and world == 1:
            line["cpu_baseline"] = cpu_baseline(args, X, y)
    L.lib.ds_engine_destroy(eng)
    if world > 1:
        dist.barrier()
    L.lib.ds_master_destroy(master)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def e2e_leg(args, L, api, eng, X, y, rank, world, sweep_seed, n):
    """Same training through the C-ABI with HOST buffers (stream mode): one persistent
    launch consumes batches the host gathers (the reference's ShardSweeper order) into
    pinned memory and pushes as H2D copies while the device trains; the kernel writes
    every step's batch loss to mapped pinned host memory (D2H). Host gather, H2D and
    the device step overlap. Timed by wall clock from stream_begin to stream_end."""
    import torch
    import torch.distributed as dist
    K = min(args.e2e_steps, args.steps)
    B = args.batch
    idx, sizes = api.sweep_batches(len(y), B, sweep_seed + 1, K)
    idx = np.ascontiguousarray(idx, dtype=np.uint32)
    Xh = np.ascontiguousarray(X, dtype=np.float32)
    yh = np.ascontiguousarray(y, dtype=np.uint32)
    losses = torch.zeros(K, dtype=torch.float64, pin_memory=True)
    push = L.lib.ds_engine_stream_push_rows
    xp, yp = C.c_void_p(Xh.ctypes.data), C.c_void_p(yh.ctypes.data)
    row_ptr = [C.c_void_p(idx[s].ctypes.data) for s in range(K)]

    def stream_run(steps):
        # the host side of the reference worker loop: ShardSweeper order (precomputed above),
        # gather_batch into the engine's pinned ring slot and push (ds_engine_stream_push_rows)
        L.check(L.lib.ds_engine_stream_begin(eng, steps, C.c_void_p(losses.data_ptr())))
        for s in range(steps):
            L.check(push(eng, xp, yp, row_ptr[s], int(sizes[s])))
        L.check(L.lib.ds_engine_stream_end(eng))

    L.check(L.lib.ds_engine_reserve(eng, min(K, 100) + K))  # TrainLog room: no allocation while timed
    stream_run(min(K, 100))  # warm-up session: first-touch of the pinned ring, host caches
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    stream_run(K)
    secs = time.perf_counter() - t0
    ok = bool(np.isfinite(losses.numpy()).all())
    t = torch.tensor([secs], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return {"value": n * B * K / t.item(), "unit": "samples/s", "h2d_bytes_per_step": B * F * 4 + B * 4 + 4,
            "d2h_bytes_per_step": 8, "steps": K, "losses_finite": ok,
            "path": "ds_engine_stream_*: per step ds_engine_stream_push_rows gathers the batch rows from the "
                    "host shard into a pinned ring slot and copies it H2D into an 8-slot device ring; one "
                    "persistent fused launch (step + exchange every tau) consumes it and writes each step's "
                    "loss to mapped host memory; wall clock from stream_begin to stream_end"}


def exchange_leg(args, L, torch, dist, world, rank, local, hbm, peak_kind):
    """Standalone elastic exchange (config 5 shape): fused in-place update streaming w and
    the center once, 16 B/param; with N>1 the center is sharded and the RMW crosses NVLink."""
    Pn = args.exchange_params
    g = torch.Generator(device="cuda").manual_seed(11 + rank)
    w = torch.rand(Pn, device="cuda", generator=g) * 2 - 1
    m = torch.rand(Pn, device="cuda", generator=g) * 2 - 1
    s = torch.cuda.current_stream()
    for _ in range(3):
        L.check(L.lib.ds_elastic_update(C.c_void_p(w.data_ptr()), C.c_void_p(m.data_ptr()), Pn, C.c_float(0.1),
                                        C.c_void_p(s.cuda_stream)))
    iters = 10
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(iters):
        L.check(L.lib.ds_elastic_update(C.c_void_p(w.data_ptr()), C.c_void_p(m.data_ptr()), Pn, C.c_float(0.1),
                                        C.c_void_p(s.cuda_stream)))
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    gbs = 16.0 * Pn / (ms / 1e3) / 1e9
    out = {"params": Pn, "bytes_per_param": 16, "local_gbs": gbs, "local_frac_hbm": gbs / hbm,
           "hbm_peak_gbs": hbm, "peak_kind": peak_kind, "ms": ms}
    del w, m
    if world > 1:
        # sharded center: every rank exchanges its own worker vector concurrently (LockFree)
        Ps = min(Pn, 64 * 1024 * 1024)
        init = torch.zeros(Ps, device="cuda")
        mh = C.c_void_p()
        L.check(L.lib.ds_master_create_sharded(C.byref(mh), local, Ps, C.c_float(0.1), L.DS_MODE_LOCKFREE, rank,
                                               world, C.c_void_p(init.data_ptr())))
        rec = (C.c_uint8 * L.DS_IPC_RECORD_BYTES)()
        L.check(L.lib.ds_master_export(mh, rec))
        recs = [None] * world
        dist.all_gather_object(recs, bytes(rec))
        allrec = (C.c_uint8 * (L.DS_IPC_RECORD_BYTES * world)).from_buffer_copy(b"".join(recs))
        L.check(L.lib.ds_master_attach(mh, allrec))
        wv = torch.rand(Ps, device="cuda", generator=g)
        for _ in range(2):
            L.check(L.lib.ds_master_exchange(mh, C.c_void_p(wv.data_ptr()), C.c_void_p(wv.data_ptr()),
                                             C.c_void_p(s.cuda_stream)))
        torch.cuda.synchronize()
        dist.barrier()
        e0.record(s)
        for _ in range(iters):
            L.check(L.lib.ds_master_exchange(mh, C.c_void_p(wv.data_ptr()), C.c_void_p(wv.data_ptr()),
                                             C.c_void_p(s.cuda_stream)))
        e1.record(s)
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1) / iters], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        sms = t.item()
        remote = 8.0 * Ps * (world - 1) / world  # bytes each rank moves over NVLink per exchange, per direction x2
        out.update({"sharded_params": Ps, "sharded_ms": sms, "sharded_gbs_per_gpu": 16.0 * Ps / (sms / 1e3) / 1e9,
                    "nvlink_gbs_per_gpu": remote / (sms / 1e3) / 1e9,
                    "nvlink_note": "(G-1)/G x 8 B/param over NVLink per exchange, all ranks concurrent"})
        dist.barrier()
        L.lib.ds_master_destroy(mh)
    return out


def cifar_leg(args, L, api, torch, dist, world, rank, local, mode="async"):
    """BASELINE config 2 shape (mode "async"): Caffe cifar10_quick on synthetic 3x32x32
    CIFAR-10-shaped data, async EASGD tau=10, batch 100 per worker, one worker per GPU,
    center sharded over the GPUs (LockFree). Config 3 adds mode "adaptive" (async, the
    Adaptive policy with resolve_loss_cut's cut = 20 x the first batch's loss,
    worker.cpp:18-30) and mode "sync" (simulate_sync semantics, simulator.cpp:156-223:
    every iteration the gradients of all GPUs are summed over NVLink and applied to the
    replicated center, ds_engine_attach_sync). NOT IN THE REFERENCE (no conv layers): tf32
    tensor-core layered kernels (csrc/conv_tc.cu, csrc/convnet.cu), no CPU reference arm.
    Device-timed, max over ranks."""
    from paper_1602_08191_b200 import dist as D
    B, K, N = 100, args.cifar_steps, 10000
    Xc, yc = api.gen_synthetic(N, 3072, 10, 1.0, 1.0, 101 + rank)
    Pc = 145578
    init = torch.empty(Pc, dtype=torch.float32, device="cuda")
    if rank == 0:
        from paper_1602_08191_b200.deepspark import Model
        init.copy_(torch.from_numpy(api.init_params(Model.cifar10_quick(10), INIT_SEED)))
    if world > 1:
        dist.broadcast(init, 0)
    torch.cuda.synchronize()
    hidden = (C.c_uint32 * 1)(0)
    desc = L.ds_model_desc(2, 3072, 10, 0, hidden)
    sweep = api.mix_seed(5, rank)

    def make(hp):
        e = C.c_void_p()
        L.check(L.lib.ds_engine_create(C.byref(e), local, C.byref(desc), Xc.ctypes.data, yc.ctypes.data, len(yc),
                                       10, C.byref(hp), sweep, C.c_void_p(init.data_ptr()), L.DS_ENGINE_AUTO))
        return e

    cut = 0.0
    if mode == "adaptive":  # resolve_loss_cut: 20 x loss_only(first batch of a fresh sweeper, initial params)
        probe = make(L.ds_hyper(0.01, 0.1, 10, B, 10 ** 9, 0.0, 0.0, 0))
        L.check(L.lib.ds_engine_run(probe, 1, 0, None))
        L.check(L.lib.ds_engine_sync(probe))
        first = np.zeros(1)
        L.check(L.lib.ds_engine_log(probe, 0, 1, first.ctypes.data, None, None, None))
        L.lib.ds_engine_destroy(probe)
        cut = 20.0 * float(first[0])
    eng = make(L.ds_hyper(0.01, 0.1, 10, B, 10 ** 9, cut, 0.0, 1 if mode == "adaptive" else 0))
    m = sg = None
    if mode == "sync":
        sg = D.sync_group(L, local, Pc, rank, world)
        L.check(L.lib.ds_engine_attach_sync(eng, sg))
    elif world == 1:
        m = C.c_void_p()
        L.check(L.lib.ds_master_create(C.byref(m), local, Pc, C.c_float(0.1), L.DS_MODE_LOCKFREE,
                                       C.c_void_p(init.data_ptr())))
    else:
        m = D.sharded_master(L, local, Pc, 0.1, L.DS_MODE_LOCKFREE, init.data_ptr(), rank, world)
    if m is not None:
        L.check(L.lib.ds_engine_attach_master(eng, m))
    L.check(L.lib.ds_engine_reserve(eng, K + 5))
    L.check(L.lib.ds_engine_run(eng, 5, 0, None))
    L.check(L.lib.ds_engine_sync(eng))
    sp = C.c_void_p()
    L.check(L.lib.ds_engine_stream(eng, C.byref(sp)))
    st = torch.cuda.ExternalStream(sp.value)
    n0 = C.c_uint64()
    L.check(L.lib.ds_engine_launches(eng, C.byref(n0)))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    L.check(L.lib.ds_engine_run(eng, K, 0, None))
    e1.record(st)
    L.check(L.lib.ds_engine_sync(eng))
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    n1 = C.c_uint64()
    L.check(L.lib.ds_engine_launches(eng, C.byref(n1)))
    loss = np.zeros(K + 5)
    L.check(L.lib.ds_engine_log(eng, 0, K + 5, loss.ctypes.data, None, None, None))
    exch = np.zeros(K + 5, np.uint8)
    L.check(L.lib.ds_engine_log(eng, 0, K + 5, None, None, exch.ctypes.data, None))
    L.lib.ds_engine_destroy(eng)
    if world > 1:
        dist.barrier()
    if m is not None:
        L.lib.ds_master_destroy(m)
    if sg is not None:
        L.lib.ds_sync_destroy(sg)
    ms = t.item()
    flop = 3 * 2 * 12_350_000 * B * K  # ~3x forward (fwd + dgrad + wgrad), 2 FLOP/MAC
    out = {"metric": "train samples/s (cifar10_quick, BASELINE config %d shape)" % (2 if mode == "async" else 3),
           "value": world * B * K / (ms / 1e3), "unit": "samples/s", "ms_per_step": ms / K, "steps": K,
           "batch_per_worker": B, "eta": 0.01, "workers": world, "mode": mode,
           "dtype": "tf32 tensor cores (tcgen05 implicit-GEMM convolutions, f32 accumulation in TMEM), f32 elsewhere",
           "data": "synthetic gen_synthetic 3072 features (3x32x32 CHW), 10 classes, 10,000 rows per GPU",
           "achieved_tflops": flop / (ms / 1e3) / 1e12, "gpu_launches": int(n1.value - n0.value),
           "loss_first_last": [float(loss[0]), float(loss[-1])],
           "reference_arm": "none: the reference has no conv layers (SURVEY §8 a20)"}
    if mode == "sync":
        out["exchange"] = "synchronous: f64 worker-ordered gradient sum over NVLink peers + SGD on every replica"
    else:
        out.update(tau=10, alpha=0.1, exchange="LockFree, center sharded over the GPUs" if world > 1 else
                   "LockFree, center on the same GPU", exchanges_in_timed_steps=int(exch[5:].astype(bool).sum()))
        if mode == "adaptive":
            out["loss_cut"] = cut
    return out


# multiply-adds per sample of the AlexNet-shaped net at S = 224 (oracle/ds_oracle_alex.h):
# (MACs per output pixel x output pixels) per layer; training = forward + data gradient
# (all but conv1) + weight gradient
ALEX_FWD_MAC = [96 * 363 * 54 * 54, 256 * 1200 * 27 * 27, 384 * 2304 * 13 * 13, 384 * 1728 * 13 * 13,
                256 * 1728 * 13 * 13, 4096 * 9216, 4096 * 4096, 1000 * 4096]
ALEX_TRAIN_FLOP = 2 * (3 * sum(ALEX_FWD_MAC) - ALEX_FWD_MAC[0])


def alexnet_leg(args, L, api, torch, dist, world, rank, local):
    """BASELINE config 4: AlexNet-shaped CNN on synthetic 224x224x3 ImageNet-shaped rows,
    1000 classes, batch 128 per worker, async EASGD tau=10 alpha=0.1 with the center sharded
    over the GPUs (LockFree), one worker per GPU. NOT IN THE REFERENCE (no conv layers):
    every convolution and FC contraction on the tcgen05 tensor cores (tf32, csrc/gemm_tc.cu),
    NHWC layer kernels in csrc/alexnet.cu. Rows are N(0,1) generated on the device (the
    reference's gen_synthetic is O(classes^2 x features) for 1000 x 150,528 and takes minutes);
    labels uniform. Device-timed, max over ranks."""
    from paper_1602_08191_b200 import dist as D
    from paper_1602_08191_b200.deepspark import Model
    B, K, N, S, Cls = 128, args.alexnet_steps, 512, 224, 1000
    F = 3 * S * S
    g = torch.Generator(device="cuda").manual_seed(1000 + rank)
    Xd = torch.randn(N, F, device="cuda", generator=g)  # 308 MB per GPU: larger than L2
    yk = np.random.default_rng(2000 + rank).integers(0, Cls, N).astype(np.uint32)
    m = Model.alexnet(S, Cls)
    P = api.param_dim(m)
    init = torch.empty(P, dtype=torch.float32, device="cuda")
    if rank == 0:
        init.copy_(torch.from_numpy(api.init_params(m, INIT_SEED)))
    if world > 1:
        dist.broadcast(init, 0)
    torch.cuda.synchronize()
    hidden = (C.c_uint32 * 1)(0)
    desc = L.ds_model_desc(3, F, Cls, 0, hidden)
    hp = L.ds_hyper(0.01, 0.1, 10, B, 10 ** 9, 0.0, 0.0, 0)
    eng = C.c_void_p()
    L.check(L.lib.ds_engine_create(C.byref(eng), local, C.byref(desc), C.c_void_p(Xd.data_ptr()), yk.ctypes.data, N,
                                   Cls, C.byref(hp), api.mix_seed(7, rank), C.c_void_p(init.data_ptr()),
                                   L.DS_ENGINE_AUTO))
    del Xd
    if world == 1:
        mst = C.c_void_p()
        L.check(L.lib.ds_master_create(C.byref(mst), local, P, C.c_float(0.1), L.DS_MODE_LOCKFREE,
                                       C.c_void_p(init.data_ptr())))
    else:
        mst = D.sharded_master(L, local, P, 0.1, L.DS_MODE_LOCKFREE, init.data_ptr(), rank, world)
    L.check(L.lib.ds_engine_attach_master(eng, mst))
    W = 3
    L.check(L.lib.ds_engine_reserve(eng, K + W))
    L.check(L.lib.ds_engine_run(eng, W, 0, None))
    L.check(L.lib.ds_engine_sync(eng))
    sp = C.c_void_p()
    L.check(L.lib.ds_engine_stream(eng, C.byref(sp)))
    st = torch.cuda.ExternalStream(sp.value)
    n0 = C.c_uint64()
    L.check(L.lib.ds_engine_launches(eng, C.byref(n0)))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    L.check(L.lib.ds_engine_run(eng, K, 0, None))
    e1.record(st)
    L.check(L.lib.ds_engine_sync(eng))
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    n1 = C.c_uint64()
    L.check(L.lib.ds_engine_launches(eng, C.byref(n1)))
    loss = np.zeros(K + W)
    L.check(L.lib.ds_engine_log(eng, 0, K + W, loss.ctypes.data, None, None, None))
    L.lib.ds_engine_destroy(eng)
    if world > 1:
        dist.barrier()
    L.lib.ds_master_destroy(mst)
    ms = t.item()
    tflops = ALEX_TRAIN_FLOP * B * K / (ms / 1e3) / 1e12
    return {"metric": "train samples/s (AlexNet-shaped, BASELINE config 4 shape)", "value": world * B * K / (ms / 1e3),
            "unit": "samples/s", "ms_per_step": ms / K, "steps": K, "warmup": W, "batch_per_worker": B,
            "tau": 10, "alpha": 0.1, "eta": 0.01, "workers": world, "params": P,
            "exchange": "LockFree, center sharded over the GPUs" if world > 1 else "LockFree, center on the same GPU",
            "dtype": "tf32 tensor cores (tcgen05 GEMMs, f32 accumulation in TMEM), f32 elsewhere",
            "data": "synthetic N(0,1) rows 3x224x224 (CHW), uniform labels over 1000 classes, 512 rows per GPU "
                    "(308 MB, larger than L2)",
            "flop_per_sample": ALEX_TRAIN_FLOP, "achieved_tflops": tflops,
            "tf32_peak_tflops": 823.4, "tf32_peak_kind": "measured bf16 dense burst (MEASURED_PEAKS.json) / 2; "
            "nominal tf32 dense 1100", "tensor_frac": tflops / 823.4,
            "gpu_launches": int(n1.value - n0.value), "loss_first_last": [float(loss[0]), float(loss[-1])],
            "reference_arm": "none: the reference has no conv layers (SURVEY §8 a20)"}


def cpu_baseline(args, X, y):
    """The reference's own SgdEngine loop (oracle/_ref, unmodified) on this box's host,
    one worker thread, a bounded sample (~15 s) of the same workload."""
    try:
        from oracle.oracle import Oracle, ModelSpec, Hyper, available
    except Exception as e:  # pragma: no cover
        return {"value": None, "unavailable": str(e)}
    kind = "reference" if available("dsref") else "port"
    orc = Oracle("dsref" if kind == "reference" else "dso")
    m = ModelSpec.mlp(F, [H], NCLS)
    hp = Hyper(eta=0.05, alpha=0.1, tau=args.tau, batch_size=args.batch, i_max=10 ** 9)
    init = orc.init_params(m, INIT_SEED)
    if kind == "reference":
        probe = orc.workers_time(m, [(X, y)], NCLS, hp, init, True, 1, 5)
        steps = int(max(20, min(2000, 15.0 / max(probe / 5, 1e-4))))
        secs = orc.workers_time(m, [(X, y)], NCLS, hp, init, True, 3, steps)
    else:
        steps = 200
        t0 = time.perf_counter()
        orc.engine_steps(m, X, y, NCLS, hp, 7, init, steps)
        secs = time.perf_counter() - t0
    return {"value": args.batch * steps / secs, "unit": "samples/s", "cores": 1, "kind": kind,
            "sample": f"{steps} SgdEngine iterations (b={args.batch}, tau={args.tau} exchanges with an "
                      f"in-process MasterState) on 1 host core of {os.cpu_count()}"}


if __name__ == "__main__":
    sys.exit(main())
