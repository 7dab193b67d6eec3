"""World-size-2 gloo tests (CPU) of the N>1 host logic: slice bounds of the sharded center,
deterministic ticket assignment from the replayed event order, and record gathering."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1602_08191_b200 import dist as D
    from paper_1602_08191_b200.deepspark import DeepSpark
    api = DeepSpark()
    order_w, order_it = api.exchange_order(world, 5, 60, 1, comm_cost_S=0.5, cost_multipliers=[1.0, 1.3][:world])
    tk = D.worker_tickets(order_w, rank)
    recs = D.gather_bytes(bytes([rank]) * 256, world)
    all_tk = D.gather_bytes(tk.tobytes(), world)
    if rank == 0:
        q.put(dict(order_w=order_w, order_it=order_it, recs=recs,
                   tickets=[np.frombuffer(b, np.uint64) for b in all_tk]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_tickets_and_records_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    tickets = res["tickets"]
    allt = np.sort(np.concatenate(tickets))
    assert np.array_equal(allt, np.arange(len(res["order_w"])))  # every exchange owned exactly once
    for k, t in enumerate(tickets):
        assert np.all(np.diff(t.astype(np.int64)) > 0)
        its = res["order_it"][t.astype(np.int64)]
        assert np.array_equal(its, np.arange(1, len(its) + 1) * 5)  # worker k exchanges at 5, 10, ...
    assert [r[0] for r in res["recs"]] == list(range(world))


def test_exchange_order_matches_oracle_simulate():
    """The replayed order equals the order of the oracle's master snapshots."""
    from oracle.oracle import Hyper, ModelSpec, Oracle, SimSpec
    from paper_1602_08191_b200.deepspark import DeepSpark
    orc, api = Oracle("dso"), DeepSpark()
    m = ModelSpec.softmax(4, 2)
    X, y = orc.gen_synthetic(200, 4, 2, 3.0, 1.0, 1)
    for n, S, mults in ((2, 0.0, None), (3, 0.5, [1.0, 1.5, 1.0]), (4, 0.25, [1.0, 1.0, 2.0, 0.5])):
        s = SimSpec(n, Hyper(eta=0.05, tau=3, batch_size=8, i_max=21), m, X, y, 2, schedule_seed=7, data_seed=3,
                    comm_cost_S=S, cost_multipliers=mults, eval_every=1000)
        o = orc.simulate(s)
        w, it = api.exchange_order(n, 3, 21, 7, comm_cost_S=S, cost_multipliers=mults)
        assert np.array_equal(w, o.snap_worker)


@pytest.mark.parametrize("dim,world", [(203530, 2), (203530, 4), (1000, 8), (31, 3), (1 << 20, 8)])
def test_shard_bounds(dim, world):
    from paper_1602_08191_b200 import dist as D
    b = D.shard_bounds(dim, world)
    assert b[0][0] == 0 and b[-1][1] == dim
    for (a0, a1), (c0, c1) in zip(b, b[1:]):
        assert a1 == c0
    for a0, a1 in b:
        assert a1 == a0 or (a0 * 4) % 128 == 0  # non-empty slices start 128-byte aligned
