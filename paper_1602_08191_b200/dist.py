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
    if world == 1:  # a one-GPU group needs no process group
        return [blob]
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


def sync_group(L, device: int, dim: int, rank: int, world: int, group=None):
    """This rank's member of a synchronous-SGD group (ds_sync), attached to every peer."""
    s = C.c_void_p()
    L.check(L.lib.ds_sync_create(C.byref(s), device, dim, rank, world))
    rec = (C.c_uint8 * L.DS_IPC_RECORD_BYTES)()
    L.check(L.lib.ds_sync_export(s, rec))
    recs = gather_bytes(bytes(rec), world, group)
    allrec = (C.c_uint8 * (L.DS_IPC_RECORD_BYTES * world)).from_buffer_copy(b"".join(recs))
    L.check(L.lib.ds_sync_attach(s, allrec))
    return s


def local_sync_group(L, device: int, dim: int, world: int):
    """`world` members of one synchronous group living in THIS process on one device (the
    single-GPU form; drive them with ds_sync_*_group, one launch per round)."""
    syncs = []
    recs = []
    for k in range(world):
        s = C.c_void_p()
        L.check(L.lib.ds_sync_create(C.byref(s), device, dim, k, world))
        rec = (C.c_uint8 * L.DS_IPC_RECORD_BYTES)()
        L.check(L.lib.ds_sync_export(s, rec))
        syncs.append(s)
        recs.append(bytes(rec))
    allrec = (C.c_uint8 * (L.DS_IPC_RECORD_BYTES * world)).from_buffer_copy(b"".join(recs))
    for s in syncs:
        L.check(L.lib.ds_sync_attach(s, allrec))
    return syncs


def run_sync_group_local(L, api, model_desc, shards, n_classes: int, hp, sweep_seeds, params_devs, syncs,
                         device: int, stream=None):
    """simulate_sync (simulator.cpp:156-223) with all `world` ranks on ONE GPU: each round
    every rank's ShardSweeper batch gives its gradient at its replica of the master (its
    slot), then ONE ds_sync_reduce_update_group launch reduces every slice in worker order
    and writes every replica. Returns the per-rank per-round batch losses ([world, i_max])."""
    import torch
    world = len(syncs)
    B, i_max = hp.batch_size, hp.i_max
    dev = torch.device("cuda", device)
    ws_bytes = C.c_uint64()
    L.check(L.lib.ds_loss_and_grad_workspace(C.byref(model_desc), B, C.byref(ws_bytes)))
    per = []
    for k, (Xk, yk) in enumerate(shards):
        idx, rows = api.sweep_batches(len(yk), B, sweep_seeds[k], i_max)
        F = Xk.shape[1]
        per.append(dict(
            F=F, rows=rows,
            Xd=torch.from_numpy(np.ascontiguousarray(Xk)).to(dev),
            yd=torch.from_numpy(np.ascontiguousarray(yk).astype(np.uint32).view(np.int32)).to(dev),
            idx=torch.from_numpy(np.ascontiguousarray(idx).astype(np.uint32).view(np.int32)).to(dev),
            bX=torch.empty((B, F), dtype=torch.float32, device=dev),
            by=torch.empty(B, dtype=torch.int32, device=dev),
            ws=torch.empty(max(1, ws_bytes.value), dtype=torch.uint8, device=dev)))
    losses = torch.zeros((world, i_max), dtype=torch.float64, device=dev)
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    st = C.c_void_p(stream) if stream is not None else None
    group = (C.c_void_p * world)(*[s.value for s in syncs])
    preps = (C.c_void_p * world)(*[p.data_ptr() for p in params_devs])
    slot = C.c_void_p()
    for r in range(i_max):
        for k in range(world):
            w = per[k]
            nr = int(w["rows"][r])
            L.check(L.lib.ds_gather_rows(C.c_void_p(w["bX"].data_ptr()), C.c_void_p(w["by"].data_ptr()),
                                         C.c_void_p(w["Xd"].data_ptr()), C.c_void_p(w["yd"].data_ptr()),
                                         C.c_void_p(w["idx"][r, :nr].data_ptr()), nr, w["F"], st))
            L.check(L.lib.ds_sync_begin(syncs[k], C.byref(slot), st))
            L.check(L.lib.ds_loss_and_grad(C.byref(model_desc), C.c_void_p(params_devs[k].data_ptr()),
                                           C.c_void_p(w["bX"].data_ptr()), C.c_void_p(w["by"].data_ptr()), nr, slot,
                                           C.c_void_p(losses.data_ptr() + 8 * (k * i_max + r)),
                                           C.c_void_p(w["ws"].data_ptr()), C.c_void_p(flags.data_ptr()), st))
        L.check(L.lib.ds_sync_reduce_update_group(group, world, preps, C.c_float(hp.eta), C.c_float(hp.weight_decay),
                                                  C.c_void_p(flags.data_ptr()), st))
    torch.cuda.synchronize(dev)
    fl = int(flags.item())
    if fl:
        raise RuntimeError(f"simulate_sync: device flags 0x{fl:x} (non-finite loss/grad/update or label range)")
    return losses.cpu().numpy()


def run_sync_worker(L, api, model_desc, Xk, yk, n_classes: int, hp, sweep_seed_k: int, params_dev, sg,
                    device: int, stream=None):
    """One rank of simulate_sync (simulator.cpp:156-223) on its own GPU: every round the
    rank's ShardSweeper batch (gathered on the device from the resident shard) gives a
    gradient at the current master replica; ds_sync_reduce_update sums all ranks' gradients
    in worker order over NVLink and applies the SGD step. Returns this worker's per-round
    batch losses (f64). `params_dev` (device f32[P]) holds the replica in and out."""
    import torch
    B, i_max = hp.batch_size, hp.i_max
    idx, rows = api.sweep_batches(len(yk), B, sweep_seed_k, i_max)
    dev = torch.device("cuda", device)
    Xd = torch.from_numpy(np.ascontiguousarray(Xk)).to(dev)
    yd = torch.from_numpy(np.ascontiguousarray(yk).astype(np.uint32).view(np.int32)).to(dev)
    idx_d = torch.from_numpy(np.ascontiguousarray(idx).astype(np.uint32).view(np.int32)).to(dev)
    F = Xk.shape[1]
    bX = torch.empty((B, F), dtype=torch.float32, device=dev)
    by = torch.empty(B, dtype=torch.int32, device=dev)
    ws_bytes = C.c_uint64()
    L.check(L.lib.ds_loss_and_grad_workspace(C.byref(model_desc), B, C.byref(ws_bytes)))
    ws = torch.empty(max(1, ws_bytes.value), dtype=torch.uint8, device=dev)
    losses = torch.zeros(i_max, dtype=torch.float64, device=dev)
    flags = torch.zeros(1, dtype=torch.int32, device=dev)
    st = C.c_void_p(stream) if stream is not None else None
    slot = C.c_void_p()
    for r in range(i_max):
        nr = int(rows[r])
        src = idx_d[r, :nr]  # sweep_batches: [i_max, B] shard rows, `rows[r]` valid
        L.check(L.lib.ds_gather_rows(C.c_void_p(bX.data_ptr()), C.c_void_p(by.data_ptr()), C.c_void_p(Xd.data_ptr()),
                                     C.c_void_p(yd.data_ptr()), C.c_void_p(src.data_ptr()), nr, F, st))
        L.check(L.lib.ds_sync_begin(sg, C.byref(slot), st))
        L.check(L.lib.ds_loss_and_grad(C.byref(model_desc), C.c_void_p(params_dev.data_ptr()),
                                       C.c_void_p(bX.data_ptr()), C.c_void_p(by.data_ptr()), nr, slot,
                                       C.c_void_p(losses.data_ptr() + 8 * r), C.c_void_p(ws.data_ptr()),
                                       C.c_void_p(flags.data_ptr()), st))
        L.check(L.lib.ds_sync_reduce_update(sg, C.c_void_p(params_dev.data_ptr()), C.c_float(hp.eta),
                                            C.c_float(hp.weight_decay), C.c_void_p(flags.data_ptr()), st))
    torch.cuda.synchronize(dev)
    fl = int(flags.item())
    if fl:
        raise RuntimeError(f"simulate_sync: device flags 0x{fl:x} (non-finite loss/grad/update or label range)")
    return losses.cpu().numpy()
