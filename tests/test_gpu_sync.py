"""Synchronous training over the ds_sync reduce-scatter + all-gather, on ONE GPU.

The world-N group runs in this process on cuda:0 through the *_group entry points (one
kernel per round for all ranks), so the single-GPU suite exercises the multi-worker
arithmetic the multi-GPU run uses (tests/test_mgpu.py covers the cross-process flags and
the NVLink all-gather):

* simulate_sync (simulator.cpp:156-223) end to end: the final master bit-identical to the
  oracle's simulate(sync=True) on every replica, per-round losses to 1e-14 relative;
* the reduction alone at large sizes (64M and 500M floats... the 500M case only when the
  GPU has room), bit-exact against the worker-ordered f64 numpy restatement
  (Oracle.sync_sgd_round), with slice boundaries that do not divide the vector;
* synchronous EASGD (EXTENSION — not in the reference) bit-exact against
  Oracle.sync_easgd_round over several rounds;
* error behaviour: non-finite gradients raise the device flags, mismatched groups refused.
"""
import ctypes as C

import numpy as np
import pytest

from oracle.oracle import Hyper, ModelSpec, Oracle, SimSpec

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1602_08191_b200 import _lib as L
    from paper_1602_08191_b200 import dist as D
    from paper_1602_08191_b200.deepspark import DeepSpark
    return torch, L, D, DeepSpark(), Oracle("dso")


def _destroy(L, syncs):
    for s in syncs:
        L.lib.ds_sync_destroy(s)


@pytest.mark.parametrize("world,wd,big", [(2, 0.0, False), (3, 1e-3, False), (2, 0.0, True), (4, 5e-4, True)])
def test_sync_group_matches_simulate_sync(env, world, wd, big):
    torch, L, D, api, orc = env
    if big:
        m = ModelSpec.mlp(784, [256], 10)
        X, y = api.gen_synthetic(4000, 784, 10, 0.1, 1.0, 1)
        hp = Hyper(eta=0.05, tau=10, batch_size=32, i_max=40, weight_decay=wd)
    else:
        m = ModelSpec.mlp(20, [16], 3)
        X, y = api.gen_synthetic(600, 20, 3, 2.0, 1.5, 5)
        hp = Hyper(eta=0.05, tau=5, batch_size=16, i_max=60, weight_decay=wd)
    data_seed, init_seed, sched_seed = 3, 2, 1
    shards, _ = D.sim_shards(api, X, y, world, 0.2, data_seed)
    P = api.param_dim(m)
    init = torch.from_numpy(api.init_params(m, init_seed)).cuda()
    reps = [init.clone() for _ in range(world)]
    syncs = D.local_sync_group(L, 0, P, world)
    desc = L.ds_model_desc(1, m.n_features, m.n_classes, 1, (C.c_uint32 * 1)(*m.hidden))
    try:
        losses = D.run_sync_group_local(L, api, desc, shards, m.n_classes, hp,
                                        [D.sweep_seed(api, data_seed, k) for k in range(world)], reps, syncs, 0)
        rounds = C.c_uint64()
        L.check(L.lib.ds_sync_rounds(syncs[0], C.byref(rounds)))
        assert rounds.value == hp.i_max
    finally:
        _destroy(L, syncs)
    finals = [r.cpu().numpy() for r in reps]
    ref = orc.simulate(SimSpec(world, hp, m, X, y, m.n_classes, sync=True, schedule_seed=sched_seed,
                               init_seed=init_seed, data_seed=data_seed, eval_every=10 ** 6,
                               record_master_snaps=False))
    for f in finals:  # every replica bit-identical to the oracle's master
        assert np.array_equal(f.view(np.uint32), ref.final_master.view(np.uint32))
    ref_loss = np.asarray(ref.batch_loss).reshape(world, -1)
    np.testing.assert_allclose(losses, ref_loss, rtol=1e-14, atol=0)


def _reduce_case(env, dim, world, eta, wd, seed, rounds=2):
    torch, L, D, api, orc = env
    g = torch.Generator(device="cuda").manual_seed(seed)
    x = torch.randn(dim, device="cuda", generator=g)
    reps = [x.clone() for _ in range(world)]
    syncs = D.local_sync_group(L, 0, dim, world)
    flags = torch.zeros(1, dtype=torch.int32, device="cuda")
    group = (C.c_void_p * world)(*[s.value for s in syncs])
    preps = (C.c_void_p * world)(*[r.data_ptr() for r in reps])
    xh = x.cpu().numpy()
    try:
        for _ in range(rounds):
            grads = []
            for k in range(world):
                slot = C.c_void_p()
                L.check(L.lib.ds_sync_begin(syncs[k], C.byref(slot), None))
                gk = torch.randn(dim, device="cuda", generator=g)
                L.check(L.lib.ds_memcpy(slot, C.c_void_p(gk.data_ptr()), dim * 4, None))
                grads.append(gk.cpu().numpy())
                del gk
            L.check(L.lib.ds_sync_reduce_update_group(group, world, preps, C.c_float(eta), C.c_float(wd),
                                                      C.c_void_p(flags.data_ptr()), None))
            torch.cuda.synchronize()
            xh = orc.sync_sgd_round(xh, grads, eta, wd)
            del grads
        assert int(flags.item()) == 0
        for r in reps:
            assert torch.equal(r.cpu().view(torch.int32), torch.from_numpy(xh.view(np.int32)))
    finally:
        _destroy(L, syncs)


@pytest.mark.parametrize("dim,world", [(1, 2), (33, 3), (1000003, 4), (64 << 20, 2)])
def test_sync_reduce_bit_exact(env, dim, world):
    _reduce_case(env, dim, world, 0.03, 1e-4 if world > 2 else 0.0, seed=dim % 1000 + world)


def test_sync_reduce_bit_exact_500m(env):
    torch = env[0]
    free, _ = torch.cuda.mem_get_info()
    dim = 500_000_000
    # 2 replicas + 2 ranks x (2 slot parities x 2 dim + 2 dim pubs) + temporaries
    if free < dim * 4 * 18:
        pytest.skip("not enough device memory for the 500M-element case")
    _reduce_case(env, dim, 2, 0.01, 0.0, seed=7, rounds=1)


@pytest.mark.parametrize("dim,world", [(17, 2), (1000003, 3), (1 << 22, 8)])
def test_sync_easgd_group_bit_exact(env, dim, world):
    torch, L, D, api, orc = env
    alpha = 0.9 / world
    g = torch.Generator(device="cuda").manual_seed(dim + world)
    c0 = torch.randn(dim, device="cuda", generator=g)
    centers = [c0.clone() for _ in range(world)]
    workers = [c0 + 0.1 * torch.randn(dim, device="cuda", generator=g) for _ in range(world)]
    syncs = D.local_sync_group(L, 0, dim, world)
    flags = torch.zeros(1, dtype=torch.int32, device="cuda")
    group = (C.c_void_p * world)(*[s.value for s in syncs])
    pw = (C.c_void_p * world)(*[w.data_ptr() for w in workers])
    pc = (C.c_void_p * world)(*[c.data_ptr() for c in centers])
    ch = c0.cpu().numpy()
    xh = [w.cpu().numpy() for w in workers]
    try:
        for rnd in range(3):
            L.check(L.lib.ds_sync_easgd_update_group(group, world, pw, pc, C.c_float(alpha),
                                                     C.c_void_p(flags.data_ptr()), None))
            xh, ch = orc.sync_easgd_round(xh, ch, alpha)
            # local progress between rounds: perturb every worker the same way on both sides
            for k in range(world):
                d = 0.01 * torch.randn(dim, device="cuda", generator=g)
                workers[k].add_(d)
                xh[k] = (xh[k] + d.cpu().numpy()).astype(np.float32)
        torch.cuda.synchronize()
        assert int(flags.item()) == 0
        for k in range(world):
            assert torch.equal(centers[k].cpu().view(torch.int32), torch.from_numpy(ch.view(np.int32)))
            assert torch.equal(workers[k].cpu().view(torch.int32), torch.from_numpy(xh[k].view(np.int32)))
    finally:
        _destroy(L, syncs)


def test_sync_errors(env):
    torch, L, D, api, orc = env
    syncs = D.local_sync_group(L, 0, 100, 2)
    flags = torch.zeros(1, dtype=torch.int32, device="cuda")
    reps = [torch.zeros(100, device="cuda") for _ in range(2)]
    group = (C.c_void_p * 2)(*[s.value for s in syncs])
    preps = (C.c_void_p * 2)(*[r.data_ptr() for r in reps])
    try:
        # no round begun on rank 1 -> state error
        slot = C.c_void_p()
        L.check(L.lib.ds_sync_begin(syncs[0], C.byref(slot), None))
        with pytest.raises(L.StateError):
            L.check(L.lib.ds_sync_reduce_update_group(group, 2, preps, C.c_float(0.1), C.c_float(0.0),
                                                      C.c_void_p(flags.data_ptr()), None))
        slot1 = C.c_void_p()
        L.check(L.lib.ds_sync_begin(syncs[1], C.byref(slot1), None))
        bad = torch.full((100,), float("nan"), device="cuda")
        L.check(L.lib.ds_memcpy(slot1, C.c_void_p(bad.data_ptr()), 400, None))
        L.check(L.lib.ds_memset(slot, 0, 400, None))
        L.check(L.lib.ds_sync_reduce_update_group(group, 2, preps, C.c_float(0.1), C.c_float(0.0),
                                                  C.c_void_p(flags.data_ptr()), None))
        torch.cuda.synchronize()
        assert int(flags.item()) & 2  # DS_FLAG_G_NONFINITE
        with pytest.raises(L.ContractError):
            L.check(L.lib.ds_sync_reduce_update_group(group, 2, preps, C.c_float(0.0), C.c_float(0.0),
                                                      C.c_void_p(flags.data_ptr()), None))
        with pytest.raises(L.ContractError):
            L.check(L.lib.ds_sync_easgd_update_group(group, 2, preps, preps, C.c_float(1.5),
                                                     C.c_void_p(flags.data_ptr()), None))
    finally:
        _destroy(L, syncs)
