"""Host plumbing for one-process-per-GPU runs (torch.distributed is only the carrier).

* ``shard_bounds``     — the 128-byte-aligned slices of the center (mirrors master.cu);
* ``worker_tickets``   — this worker's global exchange numbers in deterministic mode, from
                         the replayed simulate_async order (deepspark.exchange_order);
* ``sharded_master``   — create this rank's slice, all-gather the 256-byte IPC records,
                         attach the peers (ds_master_export / ds_master_attach);
* ``sim_shards``       — the train/holdout split and per-worker partitions exactly as the
                         reference simulator builds them (simulator.cpp:227-240).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

HOLD_TAG, PART_TAG, SWEEP_TAG = 0x484F4C44, 0x50415254, 0x53574550


def shard_bounds(dim: int, world: int):
    slice_len = ((dim + world - 1) // world + 31) & ~31
    out = []
    for k in range(world):
        b = min(k * slice_len, dim)
        out.append((b, min(b + slice_len, dim)))
    return out


def worker_tickets(order_workers: np.ndarray, rank: int) -> np.ndarray:
    return np.nonzero(np.asarray(order_workers) == rank)[0].astype(np.uint64)


def gather_bytes(blob: bytes, world: int, group=None):
    import torch.distributed as dist
    out = [None] * world
    dist.all_gather_object(out, blob, group=group)
    return out


def sharded_master(L, device: int, dim: int, alpha: float, mode: int, init_ptr: int, rank: int, world: int,
                   group=None):
    """This rank's slice of a center sharded over `world` GPUs, attached to all peers."""
    m = C.c_void_p()
    L.check(L.lib.ds_master_create_sharded(C.byref(m), device, dim, C.c_float(alpha), mode, rank, world,
                                           C.c_void_p(init_ptr)))
    rec = (C.c_uint8 * L.DS_IPC_RECORD_BYTES)()
    L.check(L.lib.ds_master_export(m, rec))
    recs = gather_bytes(bytes(rec), world, group)
    allrec = (C.c_uint8 * (L.DS_IPC_RECORD_BYTES * world)).from_buffer_copy(b"".join(recs))
    L.check(L.lib.ds_master_attach(m, allrec))
    return m


def sim_shards(api, X, y, n_workers: int, holdout_frac: float, data_seed: int, replicate: bool = False):
    """(train shards, holdout) of simulate() for these seeds: split_holdout then partition."""
    n = len(y)
    order, nh = api.split_holdout_order(n, holdout_frac, api.mix_seed(data_seed, HOLD_TAG))
    hold, train = order[:nh], order[nh:]
    if replicate:
        shards = [train] * n_workers
    else:
        porder = api.partition_order(len(train), n_workers, api.mix_seed(data_seed, PART_TAG))
        base, extra = divmod(len(train), n_workers)
        shards, pos = [], 0
        for k in range(n_workers):
            cnt = base + (1 if k < extra else 0)
            shards.append(train[porder[pos:pos + cnt]])
            pos += cnt
    return ([(np.ascontiguousarray(X[s]), np.ascontiguousarray(y[s])) for s in shards],
            (np.ascontiguousarray(X[hold]), np.ascontiguousarray(y[hold])))


def sweep_seed(api, data_seed: int, worker: int, replicate: bool = False) -> int:
    return api.mix_seed(api.mix_seed(data_seed, SWEEP_TAG), 0 if replicate else worker)
