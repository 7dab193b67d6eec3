#!/usr/bin/env python3
"""bench.py — throughput of the B200 EASGD hot path (BASELINE.json metric).

Workload (BASELINE config 1): MLP 784-256-10 (tanh), EASGD with tau=10, alpha=0.1,
eta=0.05, batch 32 per worker, TWO workers per GPU (config 1's worker count), async
LockFree exchanges with the center (sharded over the GPUs when N > 1), on synthetic
MNIST-shaped data made by the reference's own generator (gen_synthetic N=60000, sep 0.1,
sigma 1.0, seed 1+rank; the simulator's holdout split removed; the GPU's 48,000 rows are
partitioned between its workers: 150 MB f32 + 75 MB bf16 resident, larger than L2).

The headline step is the tensor-core fast step (DS_ENGINE_TC, csrc/mlp_tc.cu): both
workers of a GPU train in ONE launch, one thread-block cluster each; the FC contractions
run on tcgen05 (bf16 operands, tf32 logits, f32 accumulation) -- a stated-tolerance mode
(tests/test_gpu_tc.py). The reference's exact f64 order (DS_ENGINE_FUSED, one worker per
GPU) is measured beside it as "f64_exact".

A "step" is one local SGD iteration of every worker; every tau-th step also performs the
elastic exchange. value = all samples processed / max-over-ranks device time. The K-step
launch is repeated until the device window is >= 200 ms ("repeats"). e2e = the same
training through the C-ABI with HOST buffers (stream mode): every step of every worker
gathers its batch on the host, copies it H2D from pinned memory, and the kernel writes the
step's loss to mapped host memory (D2H).

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
    ap.add_argument("--workers", type=int, default=2, help="EASGD workers per GPU (BASELINE config 1: 2)")
    ap.add_argument("--min-window-ms", type=float, default=200.0, help="repeat the K-step launch up to this")
    ap.add_argument("--e2e-steps", type=int, default=60000, help="e2e steps per worker (a window of ~0.5 s: short host windows are noisy)")
    ap.add_argument("--det-steps", type=int, default=20000, help="timed steps of the deterministic config-1 leg")
    ap.add_argument("--exchange-params", type=int, default=256 * 1024 * 1024)
    ap.add_argument("--sync-params", type=int, default=62_378_344, help="synchronous round size (AlexNet's P)")
    ap.add_argument("--no-extras", action="store_true", help="skip e2e / exchange sweep / cpu baseline (profiling)")
    ap.add_argument("--cifar-steps", type=int, default=200, help="timed steps of the cifar10_quick leg (0 = skip)")
    ap.add_argument("--cifar-workers", type=int, default=8, help="workers on one GPU in the packed cifar10_quick leg")
    ap.add_argument("--alexnet-steps", type=int, default=20, help="timed steps of the AlexNet leg (0 = skip)")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p.get("hbm_gbs", 6552.3), p.get("bf16_tflops", 1646.8), p.get("bf16_tflops_sustained", 1400.2), "measured"
    except Exception:
        return 6650.0, 1590.0, 1400.0, "fallback"


def worker_data(rank, api, workers=1):
    """Rank's synthetic rows (gen_synthetic seed 1+rank, minus the simulator's holdout),
    partitioned between the GPU's `workers` workers (contiguous blocks)."""
    X, y = api.gen_synthetic(N_SAMPLES, F, NCLS, SEP, SIGMA, 1 + rank)
    order, nh = api.split_holdout_order(N_SAMPLES, 0.2, api.mix_seed(DATA_SEED, 0x484f4c44))
    tr = order[nh:]
    Xr, yr = X[tr], y[tr]
    n = len(yr) // workers
    return [(np.ascontiguousarray(Xr[k * n:(k + 1) * n]), np.ascontiguousarray(yr[k * n:(k + 1) * n]))
            for k in range(workers)]


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
    n = max(1, args.gpus) * args.workers  # this arm's workers: `workers` per GPU
    m = ModelSpec.mlp(F, [H], NCLS)
    hp = Hyper(eta=0.05, alpha=0.1, tau=args.tau, batch_size=args.batch, i_max=10 ** 9)
    shards = [sh for g in range(max(1, args.gpus)) for sh in worker_data(g, orc, args.workers)]
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
                                 "MasterState; not this arm's config (workers per GPU x GPUs)"}
    line = {"metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": args.gpus, "steps": steps,
            "warmup": warm, "ms_per_step": 1000.0 * secs / steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference gen_synthetic, per-worker seeds)",
            "impl": "reference",
            "config": config_block(args, max(1, args.gpus)),
            "cpu_baseline": {"value": value, "unit": "samples/s", "cores": n, "kind": kind,
                             "sample": f"{steps} timed iterations per worker x {n} worker thread(s) "
                                       f"(+{warm} warmup), LockFree in-process MasterState, tau={args.tau}"},
            "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    if all_cores:
        line["all_cores"] = all_cores
    print(json.dumps(line), flush=True)
    return 0


def config_block(args, n):
    w = args.workers * n
    return {"workload": f"mlp784-256-10 EASGD, BASELINE config 1 ({args.workers} workers per GPU, async LockFree)",
            "model": "mlp:784:256:10 (tanh hidden, softmax CE)", "global_batch": args.batch * w,
            "batch_per_worker": args.batch, "seq_len": None, "tau": args.tau, "alpha": 0.1, "eta": 0.05,
            "workers": w, "workers_per_gpu": args.workers, "parallelism": f"easgd-dp{w} ({args.workers} per GPU)",
            "exchange": "LockFree, center sharded over the GPUs, in-kernel P2P RMW" if n > 1 else
                        "LockFree, center on the same GPU, in-kernel",
            "l2_policy": "inputs larger than L2: 48,000 rows per GPU (150 MB f32 + 75 MB bf16 copy), random batches",
            "numerics": "tensor-core step: bf16 operands (forward, weight gradient), tf32 logits, f32 accumulation "
                        "and parameters (stated tolerance, tests/test_gpu_tc.py); f64_exact: the reference's f64 order"}


def make_master(L, dist, local, rank, world, P, init_ptr, mode):
    master = C.c_void_p()
    if world == 1:
        L.check(L.lib.ds_master_create(C.byref(master), local, P, C.c_float(0.1), mode, C.c_void_p(init_ptr)))
    else:
        L.check(L.lib.ds_master_create_sharded(C.byref(master), local, P, C.c_float(0.1), mode, rank, world,
                                               C.c_void_p(init_ptr)))
        rec = (C.c_uint8 * L.DS_IPC_RECORD_BYTES)()
        L.check(L.lib.ds_master_export(master, rec))
        recs = [None] * world
        dist.all_gather_object(recs, bytes(rec))
        allrec = (C.c_uint8 * (L.DS_IPC_RECORD_BYTES * world)).from_buffer_copy(b"".join(recs))
        L.check(L.lib.ds_master_attach(master, allrec))
        dist.barrier()
    return master


def timed_runs(L, run, engines, stream, K, min_ms, clk_index, world, dist, torch):
    """K-step launches, repeated until the device window reaches min_ms; CUDA events on the
    launching stream, max over ranks. Returns (ms, repeats, launches, clocks)."""
    e0 = engines[0]
    for e in engines:  # TrainLog / plan room for the probe and every repeat: nothing allocated while timed
        L.check(L.lib.ds_engine_reserve(e, K + 8))
    probe = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    probe[0].record(stream)
    run(K)
    probe[1].record(stream)
    for e in engines:
        L.check(L.lib.ds_engine_sync(e))
    torch.cuda.synchronize()
    per = max(probe[0].elapsed_time(probe[1]), 1e-3)
    reps = torch.tensor([max(1, min(4096, int(np.ceil(min_ms / per))))], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(reps, op=dist.ReduceOp.MAX)
    R = int(reps.item())
    for e in engines:
        L.check(L.lib.ds_engine_reserve(e, (R + 1) * K + 8))
    n0 = C.c_uint64()
    L.check(L.lib.ds_engine_launches(e0, C.byref(n0)))
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(clk_index) as clk:
        ev0.record(stream)
        for _ in range(R):
            run(K)
        ev1.record(stream)
        for e in engines:
            L.check(L.lib.ds_engine_sync(e))
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1)
    n1 = C.c_uint64()
    L.check(L.lib.ds_engine_launches(e0, C.byref(n1)))
    t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return t.item(), R, int(n1.value - n0.value), clk.summary()


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
    n, Wk = world, args.workers
    hbm, bf16, bf16_sus, peak_kind = peaks()

    # ---- data, init (NCCL broadcast), center, engines -------------------------------
    shards = worker_data(rank, api, Wk)
    P = (H * F + H) + (NCLS * H + NCLS)
    init = torch.empty(P, dtype=torch.float32, device="cuda")
    if rank == 0:
        from paper_1602_08191_b200.deepspark import Model
        init.copy_(torch.from_numpy(api.init_params(Model.mlp(F, [H], NCLS), INIT_SEED)))
    if world > 1:
        dist.broadcast(init, 0)  # replaces FETCH_INIT (exchanger.cpp:266-270)
    torch.cuda.synchronize()
    master = make_master(L, dist, local, rank, world, P, init.data_ptr(), L.DS_MODE_LOCKFREE)

    hidden = (C.c_uint32 * 1)(H)
    desc = L.ds_model_desc(1, F, NCLS, 1, hidden)
    hp = L.ds_hyper(0.05, 0.1, args.tau, args.batch, 10 ** 9, 0.0, 0.0, 0)
    seeds = [api.mix_seed(api.mix_seed(DATA_SEED, 0x53574550), rank * Wk + k) for k in range(Wk)]
    engines = []
    for k, (Xk, yk) in enumerate(shards):
        e = C.c_void_p()
        L.check(L.lib.ds_engine_create(C.byref(e), local, C.byref(desc), Xk.ctypes.data, yk.ctypes.data, len(yk),
                                       NCLS, C.byref(hp), seeds[k], C.c_void_p(init.data_ptr()), L.DS_ENGINE_TC))
        L.check(L.lib.ds_engine_attach_master(e, master))
        engines.append(e)
    arr = (C.c_void_p * Wk)(*[e.value for e in engines])
    sptr = C.c_void_p()
    L.check(L.lib.ds_engine_stream(engines[0], C.byref(sptr)))
    stream = torch.cuda.ExternalStream(sptr.value)

    def run_group(steps):
        L.check(L.lib.ds_engine_run_group(arr, Wk, steps))

    # ---- warmup, then the K-step group launch (repeated to a >= 200 ms window) ----------
    Wu, K = max(3, args.warmup), args.steps
    run_group(Wu)
    for e in engines:
        L.check(L.lib.ds_engine_sync(e))
    ms, R, launches, clocks = timed_runs(L, run_group, engines, stream, K, args.min_window_ms, local, world, dist,
                                         torch)
    steps_done = K * R
    value = n * Wk * args.batch * steps_done / (ms / 1e3)

    # roofline of the only kernel of the timed region: mlp_tc_kernel. Algorithmic FLOPs:
    # 818,176 per sample (fwd 203,264 MAC + dW 203,264 MAC + dX 2,560 MAC) x batch x workers x steps
    flop = FLOP_PER_SAMPLE * args.batch * Wk * steps_done
    achieved = flop / (ms / 1e3) / 1e12
    peak, pk = (bf16, "burst") if ms < 1000.0 else (bf16_sus, "sustained")
    # per worker and step the tensor pipe runs 49 forward MMAs (M64 N16 K16 bf16) + 2 logits MMAs
    # (M64 N16 K8 tf32) + 14 weight-gradient MMAs (M128 N16 K16 bf16) on each of the cluster's CTAs
    # traffic: DRAM bytes per launch of the dominant kernel, from the committed ncu --set full
    # capture (bytes per worker-step there) scaled to this run's launch (Wk workers x K steps)
    traffic, traffic_note = None, None
    dram_f = os.path.join(ROOT, "profiles", "r02_mlp_tc_dram.json")
    if os.path.exists(dram_f):
        with open(dram_f) as f:
            dj = json.load(f)
        traffic = dj["dram_bytes_per_worker_step"] * Wk * K
        traffic_note = (f"bytes per launch ({Wk} workers x {K} steps) from {dj['source']}: "
                        f"{dj['dram_bytes_per_worker_step']} B per worker-step vs "
                        f"{dj['algorithmic_bytes_per_worker_step']} B algorithmic ({dj['algorithmic']})")
    roof = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
            "traffic": traffic, "traffic_note": traffic_note, "peak_kind": f"{peak_kind} bf16 dense, {pk} (device window {ms:.0f} ms)",
            "kernel": "mlp_tc_kernel (one cluster of 16 CTAs per worker: TMA gather4 multicast batches, tcgen05 "
                      "forward / logits / weight gradient, SGD from TMEM, policy, in-kernel exchange)",
            "algorithmic": f"{FLOP_PER_SAMPLE} FLOP/sample x {args.batch} x {Wk} workers x {steps_done} steps",
            "mma_per_cta_step": {"forward_bf16_m64n16k16": 49, "logits_tf32_m64n16k8": 2,
                                 "weight_grad_bf16_m128n16k16": 14},
            "sms_used": 16 * Wk,
            "note": "latency-bound: 26 MFLOP per 32-sample step spread over 16 SMs per worker; each small "
                    "tcgen05.mma costs ~55 cycles regardless of N (profiles/r02_umma_timing.md), plus two "
                    "DSMEM phases per step"}

    line = {"metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": n, "steps": K, "warmup": Wu,
            "repeats": R, "ms_per_step": ms / steps_done, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (reference gen_synthetic, per-GPU seeds, partitioned between the GPU's workers)",
            "config": config_block(args, n), "roofline": roof, "clocks": clocks, "gpu_launches": launches}
    if not args.no_extras:
        line["e2e"] = e2e_group_leg(args, L, api, engines, shards, seeds, rank, world, n)
    for e in engines:
        L.lib.ds_engine_destroy(e)
    if world > 1:
        dist.barrier()
    L.lib.ds_master_destroy(master)
    if not args.no_extras:
        line["f64_exact"] = f64_leg(args, L, api, torch, dist, world, rank, local, shards, init)
        line["packed"] = packed_leg(args, L, api, torch, dist, world, rank, local, init)
        if world == 1:
            line["config1_deterministic"] = det_leg(args, L, api, torch, shards, seeds, init)
        nvl = nvlink_peak(L, torch, dist, world, rank, local) if world > 1 else None
        line["exchange"] = exchange_leg(args, L, torch, dist, world, rank, local, hbm, peak_kind, nvl)
        if world > 1:
            line["sync_round"] = sync_leg(args, L, torch, dist, world, rank, local, nvl)
    if args.cifar_steps > 0:
        line["cifar10_quick"] = cifar_leg(args, L, api, torch, dist, world, rank, local)
        line["cifar10_quick_packed"] = cifar_packed_leg(args, L, api, torch, dist, world, rank, local, args.cifar_workers)
        line["cifar10_quick_config3"] = {k: cifar_leg(args, L, api, torch, dist, world, rank, local, k)
                                         for k in ("sync", "adaptive")}
    if args.alexnet_steps > 0:
        line["alexnet"] = alexnet_leg(args, L, api, torch, dist, world, rank, local)
    if not args.no_extras and rank == 0 and world == 1:
        line["cpu_baseline"] = cpu_baseline(args, shards)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def f64_leg(args, L, api, torch, dist, world, rank, local, shards, init):
    """The reference's exact f64 order (DS_ENGINE_FUSED: one persistent cooperative launch
    per GPU, bit-identical to the reference), one worker per GPU (the GPU's first shard)."""
    P = init.numel()
    master = make_master(L, dist, local, rank, world, P, init.data_ptr(), L.DS_MODE_LOCKFREE)
    hidden = (C.c_uint32 * 1)(H)
    desc = L.ds_model_desc(1, F, NCLS, 1, hidden)
    hp = L.ds_hyper(0.05, 0.1, args.tau, args.batch, 10 ** 9, 0.0, 0.0, 0)
    Xk, yk = shards[0]
    e = C.c_void_p()
    L.check(L.lib.ds_engine_create(C.byref(e), local, C.byref(desc), Xk.ctypes.data, yk.ctypes.data, len(yk), NCLS,
                                   C.byref(hp), api.mix_seed(9, rank), C.c_void_p(init.data_ptr()), L.DS_ENGINE_FUSED))
    L.check(L.lib.ds_engine_attach_master(e, master))
    sp = C.c_void_p()
    L.check(L.lib.ds_engine_stream(e, C.byref(sp)))
    st = torch.cuda.ExternalStream(sp.value)
    L.check(L.lib.ds_engine_run(e, 10, 0, None))
    L.check(L.lib.ds_engine_sync(e))
    ms, R, launches, clocks = timed_runs(L, lambda k: L.check(L.lib.ds_engine_run(e, k, 0, None)), [e], st,
                                         args.steps, args.min_window_ms, local, world, dist, torch)
    L.lib.ds_engine_destroy(e)
    if world > 1:
        dist.barrier()
    L.lib.ds_master_destroy(master)
    steps = args.steps * R
    achieved = FLOP_PER_SAMPLE * args.batch * steps / (ms / 1e3) / 1e12
    sm_clk = (clocks.get("sm_mhz") or 1965.0) * 1e6
    fp64_peak = 148 * 64 * sm_clk / 1e12
    return {"metric": METRIC, "value": world * args.batch * steps / (ms / 1e3), "unit": "samples/s",
            "ms_per_step": ms / steps, "steps": args.steps, "repeats": R, "workers_per_gpu": 1, "dtype": "f64",
            "gpu_launches": launches, "clocks": clocks,
            "numerics": "the reference's f64 summation order: bit-identical trajectories (tests/test_gpu_engine.py)",
            "kernel": "mlp_kernel (persistent cooperative, 128 CTAs, one grid barrier per step)",
            "fp64_pipe": {"achieved_tflops": achieved, "peak_tflops": fp64_peak, "frac": achieved / fp64_peak}}


def packed_leg(args, L, api, torch, dist, world, rank, local, init):
    """As many concurrent workers as one launch holds (clusters of 16 CTAs co-resident on
    the GPU): the GPU's aggregate tensor-core throughput at config 1's shapes."""
    from paper_1602_08191_b200.deepspark import DeepSpark  # noqa: F401
    Wp = 7
    shards = worker_data(rank, api, Wp)
    P = init.numel()
    master = make_master(L, dist, local, rank, world, P, init.data_ptr(), L.DS_MODE_LOCKFREE)
    hidden = (C.c_uint32 * 1)(H)
    desc = L.ds_model_desc(1, F, NCLS, 1, hidden)
    hp = L.ds_hyper(0.05, 0.1, args.tau, args.batch, 10 ** 9, 0.0, 0.0, 0)
    engines = []
    for k, (Xk, yk) in enumerate(shards):
        e = C.c_void_p()
        L.check(L.lib.ds_engine_create(C.byref(e), local, C.byref(desc), Xk.ctypes.data, yk.ctypes.data, len(yk),
                                       NCLS, C.byref(hp), api.mix_seed(17, rank * Wp + k), C.c_void_p(init.data_ptr()),
                                       L.DS_ENGINE_TC))
        L.check(L.lib.ds_engine_attach_master(e, master))
        engines.append(e)
    arr = (C.c_void_p * Wp)(*[e.value for e in engines])
    sp = C.c_void_p()
    L.check(L.lib.ds_engine_stream(engines[0], C.byref(sp)))
    st = torch.cuda.ExternalStream(sp.value)
    out = {}
    try:
        L.check(L.lib.ds_engine_run_group(arr, Wp, 10))
        ms, R, launches, clocks = timed_runs(L, lambda k: L.check(L.lib.ds_engine_run_group(arr, Wp, k)), engines, st,
                                             args.steps, args.min_window_ms, local, world, dist, torch)
        steps = args.steps * R
        out = {"value": world * Wp * args.batch * steps / (ms / 1e3), "unit": "samples/s",
               "workers_per_gpu": Wp, "ms_per_step": ms / steps, "steps": args.steps, "repeats": R,
               "gpu_launches": launches, "clocks": clocks,
               "note": "not config 1's worker count: the most 16-CTA clusters one B200 co-schedules"}
    except Exception as ex:  # the GPU may not co-schedule 7 clusters of 16
        out = {"unavailable": str(ex)}
    for e in engines:
        L.lib.ds_engine_destroy(e)
    if world > 1:
        dist.barrier()
    L.lib.ds_master_destroy(master)
    return out


def det_leg(args, L, api, torch, shards, seeds, init):
    """BASELINE config 1 as the reference's simulator runs it: 2 workers, DETERMINISTIC
    exchange order (simulate_async's replayed global order, simulator.cpp:91-143) — both
    workers in ONE tensor-core launch, the center serialised by the replayed tickets in
    the kernel (bit-reproducible run to run; tests/test_gpu_tc.py)."""
    P = init.numel()
    Wd = 2
    warm, steps = 300, args.det_steps
    order_w, _ = api.exchange_order(Wd, args.tau, warm + steps, 1)
    mh = C.c_void_p()
    L.check(L.lib.ds_master_create(C.byref(mh), 0, P, C.c_float(0.1), L.DS_MODE_LOCKED,
                                   C.c_void_p(init.data_ptr())))
    hidden = (C.c_uint32 * 1)(H)
    desc = L.ds_model_desc(1, F, NCLS, 1, hidden)
    hp = L.ds_hyper(0.05, 0.1, args.tau, args.batch, warm + steps, 0.0, 0.0, 0)
    engines = []
    out = {}
    try:
        for k in range(Wd):
            Xk, yk = shards[k % len(shards)]
            e = C.c_void_p()
            L.check(L.lib.ds_engine_create(C.byref(e), 0, C.byref(desc), Xk.ctypes.data, yk.ctypes.data, len(yk),
                                           NCLS, C.byref(hp), seeds[k % len(seeds)], C.c_void_p(init.data_ptr()),
                                           L.DS_ENGINE_TC))
            engines.append(e)
            L.check(L.lib.ds_engine_attach_master(e, mh))
            tk = np.nonzero(np.asarray(order_w) == k)[0].astype(np.uint64)
            L.check(L.lib.ds_engine_set_tickets(e, tk.ctypes.data, len(tk)))
            L.check(L.lib.ds_engine_reserve(e, warm + steps + 8))
        arr = (C.c_void_p * Wd)(*[e.value for e in engines])
        sp = C.c_void_p()
        L.check(L.lib.ds_engine_stream(engines[0], C.byref(sp)))
        st = torch.cuda.ExternalStream(sp.value)
        L.check(L.lib.ds_engine_run_group(arr, Wd, warm))
        for e in engines:
            L.check(L.lib.ds_engine_sync(e))
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(0) as clk:
            e0.record(st)
            L.check(L.lib.ds_engine_run_group(arr, Wd, steps))
            e1.record(st)
            for e in engines:
                L.check(L.lib.ds_engine_sync(e))
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        cnt = C.c_uint64()
        L.check(L.lib.ds_master_exchange_count(mh, C.byref(cnt)))
        out = {"value": Wd * args.batch * steps / (ms / 1e3), "unit": "samples/s", "workers": Wd,
               "ms_per_step": ms / steps, "steps": steps, "exchanges": int(cnt.value),
               "expected_exchanges": Wd * ((warm + steps) // args.tau), "clocks": clk.summary(),
               "mode": "Locked center, deterministic tickets replayed from simulate_async's order"}
    finally:
        for e in engines:
            L.lib.ds_engine_destroy(e)
        L.lib.ds_master_destroy(mh)
    return out


def e2e_group_leg(args, L, api, engines, shards, seeds, rank, world, n):
    """The same training through the C-ABI with HOST buffers (stream mode): one launch
    trains the GPU's workers while the host, per worker, runs the reference worker's
    ShardSweeper (the epoch permutations are computed inside the timed window) and
    gather_batch: ds_engine_stream_push_rows_n gathers each step's rows from the host shard
    as bf16 into a pinned staging ring (labels in each slot's last row) and the copy engine
    moves groups of 4 steps per DMA into the kernel's HBM ring (H2D) -- one host thread per
    worker (plus helpers inside the call); the kernel writes every step's loss to mapped
    pinned host memory (D2H). Wall clock from stream_begin to the last stream_end, max over
    ranks."""
    import torch
    import torch.distributed as dist
    K, B, Wk = args.e2e_steps, args.batch, len(engines)
    # the host cores are shared by every rank's feeders: producer threads per worker
    local = int(os.environ.get("LOCAL_WORLD_SIZE", "1"))
    os.environ.setdefault("DS_STREAM_FEED_THREADS", str(max(1, min(4, (os.cpu_count() or 2) // (local * Wk)))))
    losses = [torch.zeros(K, dtype=torch.float64, pin_memory=True) for _ in range(Wk)]
    lp = (C.c_void_p * Wk)(*[lo.data_ptr() for lo in losses])
    arr = (C.c_void_p * Wk)(*[e.value for e in engines])
    host = [(np.ascontiguousarray(Xk, np.float32), np.ascontiguousarray(yk, np.uint32)) for Xk, yk in shards]
    errs = []

    def feed(k, steps, seed):
        try:
            Xh, yh = host[k]
            idx, sizes = api.sweep_batches(len(yh), B, seed, steps)  # ShardSweeper, inside the window
            idx = np.ascontiguousarray(idx, dtype=np.uint32)
            sizes = np.ascontiguousarray(sizes, dtype=np.uint32)
            L.check(L.lib.ds_engine_stream_push_rows_n(engines[k], C.c_void_p(Xh.ctypes.data),
                                                       C.c_void_p(yh.ctypes.data), C.c_void_p(idx.ctypes.data),
                                                       C.c_void_p(sizes.ctypes.data), steps))
            L.check(L.lib.ds_engine_stream_end(engines[k]))
            L.check(L.lib.ds_engine_stream_cache_host_shard(engines[k], None, 0))  # rebuilt next session
        except Exception as ex:  # reported below
            errs.append(str(ex))

    def cache(k):
        try:
            L.check(L.lib.ds_engine_stream_cache_host_shard(engines[k], C.c_void_p(host[k][0].ctypes.data),
                                                            len(host[k][1])))
        except Exception as ex:  # reported below
            errs.append(str(ex))

    def session(steps, seed_off):
        # each worker's host shard as bf16 once per session (inside the timed window): the
        # per-step gather_batch is then row copies (half the host memory traffic, no cast)
        th = [threading.Thread(target=cache, args=(k,)) for k in range(Wk)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        L.check(L.lib.ds_engine_stream_begin_group(arr, Wk, steps, lp))
        th = [threading.Thread(target=feed, args=(k, steps, seeds[k] + seed_off)) for k in range(Wk)]
        for t in th:
            t.start()
        for t in th:
            t.join()

    for e in engines:
        L.check(L.lib.ds_engine_reserve(e, min(K, 100) + K + 8))
    session(min(K, 100), 11)  # warm-up session: first touch of the pinned rings, host caches
    if errs:
        return {"value": None, "error": errs[0]}
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    session(K, 12)
    secs = time.perf_counter() - t0
    if errs:
        return {"value": None, "error": errs[0]}
    ok = all(bool(np.isfinite(lo.numpy()).all()) for lo in losses)
    t = torch.tensor([secs], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    pitch = (F + 7) // 8 * 8
    return {"value": n * Wk * B * K / t.item(), "unit": "samples/s",
            "h2d_bytes_per_step": Wk * ((B + 1) * pitch * 2 + 4), "d2h_bytes_per_step": Wk * 8, "steps": K,
            "wall_s": t.item(), "losses_finite": ok,
            "path": "ds_engine_stream_begin_group + per worker ds_engine_stream_cache_host_shard (the host shard "
                    "cast to bf16 once per session, inside the window) + ds_engine_stream_push_rows_n (host "
                    "ShardSweeper, gather_batch as bf16 row copies into a pinned staging ring, one H2D DMA per 4 steps into the "
                    "kernel's HBM ring) from one host thread per worker; one tensor-core launch trains all of the "
                    "GPU's workers; per-step losses written to mapped host memory; wall clock from the bf16 "
                    "shard copies (before stream_begin) to the last stream_end"}


def exchange_leg(args, L, torch, dist, world, rank, local, hbm, peak_kind, nvl=None):
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
        nv = remote / (sms / 1e3) / 1e9
        out.update({"sharded_params": Ps, "sharded_ms": sms, "sharded_gbs_per_gpu": 16.0 * Ps / (sms / 1e3) / 1e9,
                    "sharded_frac_hbm": 16.0 * Ps / (sms / 1e3) / 1e9 / hbm,
                    "exchanges_per_s_per_gpu": 1e3 / sms,
                    "nvlink_gbs_per_gpu": nv, "nvlink_peak_gbs": nvl["gbs_per_gpu"] if nvl else None,
                    "frac_nvlink_peak": nv / nvl["gbs_per_gpu"] if nvl else None,
                    "nvlink_note": "(G-1)/G x 8 B/param over NVLink per exchange, all ranks concurrent"})
        dist.barrier()
        L.lib.ds_master_destroy(mh)
    return out


def nvlink_peak(L, torch, dist, world, rank, local, n_floats=64 * 1024 * 1024):
    """In-run NVLink read peak with the all-gather's pattern: every rank concurrently copies
    n floats split over all peers' memory into its own HBM (ds_sync_peer_read); per-GPU
    GB/s = bytes read over NVLink / max-over-ranks device time."""
    from paper_1602_08191_b200 import dist as D
    dim = n_floats // 4 + 32
    sg = D.sync_group(L, local, dim, rank, world)
    dst = torch.empty(n_floats, device="cuda")
    s = torch.cuda.current_stream()
    st = C.c_void_p(s.cuda_stream)
    for _ in range(3):
        L.check(L.lib.ds_sync_peer_read(sg, C.c_void_p(dst.data_ptr()), n_floats, st))
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters = 20
    e0.record(s)
    for _ in range(iters):
        L.check(L.lib.ds_sync_peer_read(sg, C.c_void_p(dst.data_ptr()), n_floats, st))
    e1.record(s)
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / iters], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    per = (n_floats // (world - 1)) & ~3
    gbs = 4.0 * per * (world - 1) / (t.item() / 1e3) / 1e9
    dist.barrier()
    L.lib.ds_sync_destroy(sg)
    return {"gbs_per_gpu": gbs, "bytes": 4 * per * (world - 1), "ms": t.item(),
            "pattern": "every rank reads n/(G-1) floats from each peer concurrently (ds_sync_peer_read)"}


def sync_leg(args, L, torch, dist, world, rank, local, nvl):
    """Synchronous SGD round at AlexNet's parameter count over N GPUs: the worker-ordered
    reduce-scatter + all-gather fused with the update (ds_sync_reduce_update), against the
    in-run NVLink peak and against NCCL's all_reduce of the same vector (the library
    baseline; its ring/tree order is not the reference's worker order)."""
    from paper_1602_08191_b200 import dist as D
    P = args.sync_params
    sg = D.sync_group(L, local, P, rank, world)
    g = torch.Generator(device="cuda").manual_seed(5)
    params = torch.randn(P, device="cuda", generator=g)
    grad = torch.randn(P, device="cuda", generator=g) * 1e-3
    flags = torch.zeros(1, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream()
    st = C.c_void_p(s.cuda_stream)
    slot = C.c_void_p()

    def rnd():
        L.check(L.lib.ds_sync_begin(sg, C.byref(slot), st))
        L.check(L.lib.ds_sync_reduce_update(sg, C.c_void_p(params.data_ptr()), C.c_float(0.01), C.c_float(0.0),
                                            C.c_void_p(flags.data_ptr()), st))
    # the gradient is written once into both slot parities (the round's cost excludes the
    # backward pass that would produce it)
    for _ in range(2):
        L.check(L.lib.ds_sync_begin(sg, C.byref(slot), st))
        L.check(L.lib.ds_memcpy(slot, C.c_void_p(grad.data_ptr()), 4 * P, st))
        L.check(L.lib.ds_sync_reduce_update(sg, C.c_void_p(params.data_ptr()), C.c_float(0.01), C.c_float(0.0),
                                            C.c_void_p(flags.data_ptr()), st))
    for _ in range(3):
        rnd()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters = 20
    e0.record(s)
    for _ in range(iters):
        rnd()
    e1.record(s)
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / iters], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = t.item()
    ok = int(flags.item()) == 0
    dist.barrier()
    L.lib.ds_sync_destroy(sg)
    # NCCL all_reduce (sum) of the same f32 vector + the separate SGD update it would need
    buf = grad.clone()
    for _ in range(3):
        dist.all_reduce(buf)
    torch.cuda.synchronize()
    dist.barrier()
    e0.record(s)
    for _ in range(iters):
        dist.all_reduce(buf)
    e1.record(s)
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1) / iters], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    nccl_ms = t.item()
    nvl_bytes = 2.0 * (world - 1) / world * 4 * P
    gbs = nvl_bytes / (ms / 1e3) / 1e9
    return {"params": P, "round_ms": ms, "rounds_per_s": 1e3 / ms, "flags_clean": ok,
            "nvlink_bytes_per_gpu": nvl_bytes, "nvlink_gbs_per_gpu": gbs,
            "nvlink_peak_gbs": nvl["gbs_per_gpu"], "frac_nvlink_peak": gbs / nvl["gbs_per_gpu"],
            "nccl_allreduce_ms": nccl_ms, "vs_nccl_allreduce": nccl_ms / ms,
            "note": "ours = reduce-scatter (worker-ordered f64 sum) + SGD + all-gather, update included; "
                    "NCCL = all_reduce alone (no update, not worker-ordered)"}


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



def cifar_packed_leg(args, L, api, torch, dist, world, rank, local, workers=8):
    """BASELINE config 2 with its largest worker count on ONE GPU: `workers` cifar10_quick
    engines (batch 100 each, own stream and CUDA graphs, own data partition) training
    asynchronously against one LockFree center on the same GPU (tau = 10). The engines'
    launches overlap on the device. Device-timed: an event on engine 0's stream opens the
    window (every other stream waits on it), engine 0's stream waits on every stream's end
    event before the closing event. NOT IN THE REFERENCE (no conv layers)."""
    B, K, N = 100, args.cifar_steps, 10000
    Pc = 145578
    from paper_1602_08191_b200.deepspark import Model
    init_h = api.init_params(Model.cifar10_quick(10), INIT_SEED)
    init = torch.from_numpy(init_h).to("cuda")
    hidden = (C.c_uint32 * 1)(0)
    desc = L.ds_model_desc(2, 3072, 10, 0, hidden)
    m = C.c_void_p()
    L.check(L.lib.ds_master_create(C.byref(m), local, Pc, C.c_float(0.1), L.DS_MODE_LOCKFREE,
                                   C.c_void_p(init.data_ptr())))
    engines, data = [], []
    for w in range(workers):
        Xc, yc = api.gen_synthetic(N, 3072, 10, 1.0, 1.0, 101 + rank * workers + w)
        data.append((Xc, yc))
        e = C.c_void_p()
        hp = L.ds_hyper(0.01, 0.1, 10, B, 10 ** 9, 0.0, 0.0, 0)
        L.check(L.lib.ds_engine_create(C.byref(e), local, C.byref(desc), Xc.ctypes.data, yc.ctypes.data, len(yc),
                                       10, C.byref(hp), api.mix_seed(5, rank * workers + w),
                                       C.c_void_p(init.data_ptr()), L.DS_ENGINE_AUTO))
        L.check(L.lib.ds_engine_attach_master(e, m))
        L.check(L.lib.ds_engine_reserve(e, K + 5))
        engines.append(e)
    for e in engines:
        L.check(L.lib.ds_engine_run(e, 5, 0, None))
    for e in engines:
        L.check(L.lib.ds_engine_sync(e))
    streams = []
    for e in engines:
        sp = C.c_void_p()
        L.check(L.lib.ds_engine_stream(e, C.byref(sp)))
        streams.append(torch.cuda.ExternalStream(sp.value))
    n0 = []
    for e in engines:
        v = C.c_uint64()
        L.check(L.lib.ds_engine_launches(e, C.byref(v)))
        n0.append(v.value)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(streams[0])
    for st in streams[1:]:
        st.wait_event(e0)
    chunk = 10
    for k in range(0, K, chunk):  # interleaved enqueue keeps every stream fed
        for e in engines:
            L.check(L.lib.ds_engine_run(e, min(chunk, K - k), 0, None))
    for st in streams[1:]:
        ev = torch.cuda.Event()
        ev.record(st)
        streams[0].wait_event(ev)
    e1.record(streams[0])
    for e in engines:
        L.check(L.lib.ds_engine_sync(e))
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    launches = 0
    finite = True
    for e, a in zip(engines, n0):
        v = C.c_uint64()
        L.check(L.lib.ds_engine_launches(e, C.byref(v)))
        launches += int(v.value - a)
        loss = np.zeros(K + 5)
        L.check(L.lib.ds_engine_log(e, 0, K + 5, loss.ctypes.data, None, None, None))
        finite = finite and bool(np.isfinite(loss).all())
        L.lib.ds_engine_destroy(e)
    xcount = C.c_uint64()
    L.check(L.lib.ds_master_exchange_count(m, C.byref(xcount)))
    L.lib.ds_master_destroy(m)
    ms = t.item()
    flop = 3 * 2 * 12_350_000 * B * K * workers
    return {"metric": "train samples/s (cifar10_quick, BASELINE config 2: %d workers on one GPU)" % workers,
            "value": world * workers * B * K / (ms / 1e3), "unit": "samples/s", "ms_per_step": ms / K,
            "steps": K, "batch_per_worker": B, "workers_per_gpu": workers, "tau": 10, "alpha": 0.1, "eta": 0.01,
            "exchange": "LockFree, one center per GPU shared by its workers", "center_exchanges": int(xcount.value),
            "achieved_tflops": flop / (ms / 1e3) / 1e12, "gpu_launches": launches, "losses_finite": finite,
            "dtype": "tf32 tensor cores (tcgen05 implicit-GEMM convolutions), f32 elsewhere",
            "data": "synthetic gen_synthetic 3072 features, 10,000 rows per worker",
            "reference_arm": "none: the reference has no conv layers (SURVEY §8 a20)"}

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


def cpu_baseline(args, shards):
    """The reference's own n-worker loop (oracle/_ref, unmodified: SgdEngine + ExchangePolicy
    + an in-process LockFree MasterState, one thread per worker) on this box's host, this
    arm's workers, a bounded sample (~15 s) of the same workload."""
    try:
        from oracle.oracle import Oracle, ModelSpec, Hyper, available
    except Exception as e:  # pragma: no cover
        return {"value": None, "unavailable": str(e)}
    kind = "reference" if available("dsref") else "port"
    orc = Oracle("dsref" if kind == "reference" else "dso")
    m = ModelSpec.mlp(F, [H], NCLS)
    hp = Hyper(eta=0.05, alpha=0.1, tau=args.tau, batch_size=args.batch, i_max=10 ** 9)
    init = orc.init_params(m, INIT_SEED)
    Wk = len(shards)
    if kind == "reference":
        probe = orc.workers_time(m, shards, NCLS, hp, init, True, 1, 5)
        steps = int(max(20, min(2000, 15.0 / max(probe / 5, 1e-4))))
        secs = orc.workers_time(m, shards, NCLS, hp, init, True, 3, steps)
    else:
        Wk, steps = 1, 200
        t0 = time.perf_counter()
        orc.engine_steps(m, shards[0][0], shards[0][1], NCLS, hp, 7, init, steps)
        secs = time.perf_counter() - t0
    return {"value": Wk * args.batch * steps / secs, "unit": "samples/s", "cores": Wk, "kind": kind,
            "sample": f"{steps} iterations per worker x {Wk} worker thread(s) (b={args.batch}, tau={args.tau}, "
                      f"LockFree in-process MasterState) on {Wk} of {os.cpu_count()} host cores"}


if __name__ == "__main__":
    sys.exit(main())
