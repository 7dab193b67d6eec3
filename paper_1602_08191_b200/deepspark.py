"""Python binding of the reference-compatible API (include/deepspark_c.h over
libdeepspark_b200.so). Every numerical call runs on the B200; host-side pieces (data
generation, splits, sweep orders, event replay) are the C++ library's.

The method names and argument meanings follow the reference's C++ functions
(/root/reference/proj/include/deepspark/*.hpp); arguments are duck-typed so a caller
can pass any object carrying the fields of Model / Hyperparams / SimConfig.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _lib  # loads libds_cuda.so first (fails loudly when missing)

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libdeepspark_b200.so")
if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build with `make -C paper_1602_08191_b200`")
lib = C.CDLL(LIB_PATH)

ContractError = _lib.ContractError
NumericError = _lib.NumericError
CudaError = _lib.CudaError


class dsx_model(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n_features", C.c_uint32), ("n_classes", C.c_uint32),
                ("n_hidden", C.c_uint32), ("hidden", C.POINTER(C.c_uint32))]


class dsx_hyper(C.Structure):
    _fields_ = [("eta", C.c_double), ("alpha", C.c_double), ("tau", C.c_uint32), ("batch_size", C.c_uint32),
                ("i_max", C.c_uint64), ("loss_cut", C.c_double), ("weight_decay", C.c_double),
                ("adaptive", C.c_int32)]


class dsx_data(C.Structure):
    _fields_ = [("X", C.POINTER(C.c_float)), ("y", C.POINTER(C.c_uint32)), ("n", C.c_uint64),
                ("n_features", C.c_uint32), ("n_classes", C.c_uint32)]


class dsx_sim_cfg(C.Structure):
    _fields_ = [("n_workers", C.c_uint32), ("hyper", dsx_hyper), ("model", dsx_model), ("data", dsx_data),
                ("sync_mode", C.c_int32), ("batch_cost_C", C.c_double), ("comm_cost_S", C.c_double),
                ("cost_multipliers", C.POINTER(C.c_double)), ("schedule_seed", C.c_uint64),
                ("init_seed", C.c_uint64), ("data_seed", C.c_uint64), ("eval_every", C.c_uint32),
                ("holdout_frac", C.c_double), ("replicate_shards", C.c_int32), ("record_master_snaps", C.c_int32)]


class dsx_sim_out(C.Structure):
    _fields_ = [("final_master", C.POINTER(C.c_float)), ("worker_final", C.POINTER(C.c_float)),
                ("batch_loss", C.POINTER(C.c_double)), ("cumulated", C.POINTER(C.c_double)),
                ("exchanged", C.POINTER(C.c_uint8)), ("period_len", C.POINTER(C.c_uint32)),
                ("wall_ms", C.POINTER(C.c_int64)), ("snap_cap", C.c_uint64), ("n_snaps", C.c_uint64),
                ("snap_worker", C.POINTER(C.c_uint32)), ("snap_time", C.POINTER(C.c_double)),
                ("snap_params", C.POINTER(C.c_float)), ("eval_cap", C.c_uint64), ("n_eval", C.c_uint64),
                ("eval_time", C.POINTER(C.c_double)), ("eval_iter", C.POINTER(C.c_uint64)),
                ("eval_acc", C.POINTER(C.c_double)), ("virtual_total", C.c_double)]


class dsx_loop_out(C.Structure):
    _fields_ = [("final_params", C.POINTER(C.c_float)), ("batch_loss", C.POINTER(C.c_double)),
                ("cumulated", C.POINTER(C.c_double)), ("exchanged", C.POINTER(C.c_uint8)),
                ("period_len", C.POINTER(C.c_uint32))]


def _p(a, ct):
    if a is None:
        return C.cast(None, C.POINTER(ct))
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.POINTER(ct))


P = C.POINTER
_SIGS = {
    "dsx_last_error": (C.c_char_p, []),
    "dsx_mix_seed": (C.c_uint64, [C.c_uint64, C.c_uint64]),
    "dsx_rng_draws": (None, [C.c_uint64, C.c_uint64, P(C.c_uint64), P(C.c_double), P(C.c_double), C.c_uint64,
                             P(C.c_uint64)]),
    "dsx_param_dim": (C.c_uint64, [P(dsx_model)]),
    "dsx_fingerprint": (C.c_uint64, [P(dsx_model)]),
    "dsx_init_params": (C.c_int, [P(dsx_model), C.c_uint64, P(C.c_float)]),
    "dsx_loss_and_grad": (C.c_int, [P(dsx_model), P(C.c_float), P(C.c_float), P(C.c_uint32), C.c_uint32,
                                    P(C.c_float), P(C.c_double)]),
    "dsx_predict": (C.c_int, [P(dsx_model), P(C.c_float), P(C.c_float), C.c_uint64, P(C.c_uint32)]),
    "dsx_accuracy": (C.c_int, [P(dsx_model), P(C.c_float), P(dsx_data), P(C.c_double)]),
    "dsx_sgd_step": (C.c_int, [P(C.c_float), P(C.c_float), C.c_uint64, C.c_double, P(C.c_float)]),
    "dsx_easgd_update": (C.c_int, [P(C.c_float), P(C.c_float), C.c_uint64, C.c_double, P(C.c_float),
                                   P(C.c_float)]),
    "dsx_gen_synthetic": (C.c_int, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_double, C.c_double, C.c_uint64,
                                    P(C.c_float), P(C.c_uint32)]),
    "dsx_split_holdout_order": (C.c_int, [C.c_uint64, C.c_double, C.c_uint64, P(C.c_uint32), P(C.c_uint64)]),
    "dsx_partition_order": (C.c_int, [C.c_uint64, C.c_uint32, C.c_uint64, P(C.c_uint32)]),
    "dsx_sweep_batches": (C.c_int, [C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, P(C.c_uint32),
                                    P(C.c_uint32)]),
    "dsx_engine_steps": (C.c_int, [P(dsx_model), P(dsx_data), P(dsx_hyper), C.c_uint64, P(C.c_float),
                                   C.c_uint64, P(C.c_float), P(C.c_double)]),
    "dsx_run_training_loop": (C.c_int, [P(dsx_model), P(dsx_data), P(dsx_hyper), C.c_uint64, P(C.c_float),
                                        C.c_int, P(C.c_float), P(dsx_loop_out)]),
    "dsx_run_worker": (C.c_int, [P(dsx_model), C.c_double, C.c_int, P(C.c_float), P(dsx_model), C.c_char_p,
                                 P(dsx_hyper), C.c_uint32, C.c_uint64, C.c_char_p, P(C.c_float), P(C.c_uint64),
                                 P(dsx_loop_out)]),
    "dsx_resolve_loss_cut": (C.c_int, [P(dsx_model), P(dsx_data), P(dsx_hyper), C.c_uint64, P(C.c_float),
                                       P(C.c_double)]),
    "dsx_simulate": (C.c_int, [P(dsx_sim_cfg), P(dsx_sim_out)]),
    "dsx_exchange_order": (C.c_int, [C.c_uint32, C.c_double, C.c_double, P(C.c_double), C.c_uint32, C.c_uint64,
                                     C.c_uint64, P(C.c_uint32), P(C.c_uint64), C.c_uint64, P(C.c_uint64)]),
}
for _n, (_r, _a) in _SIGS.items():
    _f = getattr(lib, _n)
    _f.restype = _r
    _f.argtypes = _a
EXPORTED = sorted(_SIGS)

_ERRS = {1: ContractError, 2: NumericError, 3: CudaError}


def _check(rc: int):
    if rc:
        raise _ERRS.get(rc, _lib.DsError)(lib.dsx_last_error().decode(errors="replace"))


@dataclass
class Model:
    """deepspark::Model (model.hpp:32-56): kind 'softmax' | 'mlp' | 'cifar10_quick' |
    'alexnet' (the last two extensions, not in the reference)."""
    kind: str
    n_features: int
    n_classes: int
    hidden: Sequence[int] = ()

    @staticmethod
    def softmax(f, c):
        return Model("softmax", f, c, ())

    @staticmethod
    def mlp(f, hidden, c):
        return Model("mlp", f, c, tuple(hidden))

    @staticmethod
    def cifar10_quick(c=10):
        return Model("cifar10_quick", 3072, c, ())

    @staticmethod
    def alexnet(side=224, c=1000):
        return Model("alexnet", 3 * side * side, c, ())


@dataclass
class Hyperparams:
    """deepspark::Hyperparams (hyperparams.hpp:10-21)."""
    eta: float = 0.05
    alpha: float = 0.1
    tau: int = 100
    batch_size: int = 32
    i_max: int = 1000
    loss_cut: float = 0.0
    weight_decay: float = 0.0
    adaptive: bool = False


def _model(m):
    h = np.ascontiguousarray(np.asarray(tuple(m.hidden), dtype=np.uint32))
    d = dsx_model({"softmax": 0, "mlp": 1, "cifar10_quick": 2, "alexnet": 3}[m.kind], m.n_features, m.n_classes, len(m.hidden),
                  _p(h if len(m.hidden) else None, C.c_uint32))
    return d, h


def _hyper(h):
    return dsx_hyper(h.eta, h.alpha, h.tau, h.batch_size, h.i_max, h.loss_cut, h.weight_decay,
                     1 if h.adaptive else 0)


def _data(X, y, n_classes):
    X = np.ascontiguousarray(X, np.float32)
    y = np.ascontiguousarray(y, np.uint32)
    return dsx_data(_p(X, C.c_float), _p(y, C.c_uint32), y.shape[0], X.shape[1], n_classes), (X, y)


class DeepSpark:
    """The reference's public functions, B200-backed (same method set as oracle.Oracle)."""

    prefix = "dsx"

    def mix_seed(self, seed, stream):
        return lib.dsx_mix_seed(seed, stream)

    def rng_draws(self, seed, n, bound=0):
        u = np.zeros(n, np.uint64)
        uni = np.zeros(n)
        nrm = np.zeros(n)
        bel = np.zeros(n, np.uint64)
        lib.dsx_rng_draws(seed, n, _p(u, C.c_uint64), _p(uni, C.c_double), _p(nrm, C.c_double), bound,
                          _p(bel, C.c_uint64) if bound else _p(None, C.c_uint64))
        return u, uni, nrm, bel

    def param_dim(self, m):
        d, _h = _model(m)
        return lib.dsx_param_dim(C.byref(d))

    def fingerprint(self, m):
        d, _h = _model(m)
        return lib.dsx_fingerprint(C.byref(d))

    def init_params(self, m, seed):
        d, _h = _model(m)
        out = np.zeros(lib.dsx_param_dim(C.byref(d)), np.float32)
        _check(lib.dsx_init_params(C.byref(d), seed, _p(out, C.c_float)))
        return out

    def loss_and_grad(self, m, params, X, y, want_grad=True):
        d, _h = _model(m)
        params = np.ascontiguousarray(params, np.float32)
        X = np.ascontiguousarray(X, np.float32)
        y = np.ascontiguousarray(y, np.uint32)
        g = np.zeros_like(params) if want_grad else None
        loss = C.c_double()
        _check(lib.dsx_loss_and_grad(C.byref(d), _p(params, C.c_float), _p(X, C.c_float), _p(y, C.c_uint32),
                                     y.shape[0], _p(g, C.c_float), C.byref(loss)))
        return loss.value, g

    def predict(self, m, params, X):
        d, _h = _model(m)
        params = np.ascontiguousarray(params, np.float32)
        X = np.ascontiguousarray(X, np.float32)
        out = np.zeros(X.shape[0], np.uint32)
        _check(lib.dsx_predict(C.byref(d), _p(params, C.c_float), _p(X, C.c_float), X.shape[0], _p(out, C.c_uint32)))
        return out

    def accuracy(self, m, params, X, y, n_classes):
        d, _h = _model(m)
        params = np.ascontiguousarray(params, np.float32)
        dd, keep = _data(X, y, n_classes)
        acc = C.c_double()
        _check(lib.dsx_accuracy(C.byref(d), _p(params, C.c_float), C.byref(dd), C.byref(acc)))
        return acc.value

    def sgd_step(self, x, g, eta):
        x = np.ascontiguousarray(x, np.float32)
        g = np.ascontiguousarray(g, np.float32)
        out = np.zeros_like(x)
        _check(lib.dsx_sgd_step(_p(x, C.c_float), _p(g, C.c_float), x.shape[0], eta, _p(out, C.c_float)))
        return out

    def easgd_update(self, w, m, alpha):
        w = np.ascontiguousarray(w, np.float32)
        m = np.ascontiguousarray(m, np.float32)
        wo, mo = np.zeros_like(w), np.zeros_like(m)
        _check(lib.dsx_easgd_update(_p(w, C.c_float), _p(m, C.c_float), w.shape[0], alpha, _p(wo, C.c_float),
                                    _p(mo, C.c_float)))
        return wo, mo

    def gen_synthetic(self, n, f, c, sep, sigma, seed):
        X = np.zeros((n, f), np.float32)
        y = np.zeros(n, np.uint32)
        _check(lib.dsx_gen_synthetic(n, f, c, sep, sigma, seed, _p(X, C.c_float), _p(y, C.c_uint32)))
        return X, y

    def split_holdout_order(self, n, frac, seed):
        order = np.zeros(n, np.uint32)
        nh = C.c_uint64()
        _check(lib.dsx_split_holdout_order(n, frac, seed, _p(order, C.c_uint32), C.byref(nh)))
        return order, nh.value

    def partition_order(self, n, k, seed):
        order = np.zeros(n, np.uint32)
        _check(lib.dsx_partition_order(n, k, seed, _p(order, C.c_uint32)))
        return order

    def sweep_batches(self, shard_n, batch, seed, n_batches):
        idx = np.zeros(n_batches * batch, np.uint32)
        sizes = np.zeros(n_batches, np.uint32)
        _check(lib.dsx_sweep_batches(shard_n, batch, seed, n_batches, _p(idx, C.c_uint32), _p(sizes, C.c_uint32)))
        return idx.reshape(n_batches, batch), sizes

    def engine_steps(self, m, X, y, n_classes, hp, sweep_seed, init, steps):
        d, _h = _model(m)
        dd, keep = _data(X, y, n_classes)
        ch = _hyper(hp)
        init = np.ascontiguousarray(init, np.float32)
        params = np.zeros_like(init)
        losses = np.zeros(steps)
        _check(lib.dsx_engine_steps(C.byref(d), C.byref(dd), C.byref(ch), sweep_seed, _p(init, C.c_float), steps,
                                    _p(params, C.c_float), _p(losses, C.c_double)))
        return params, losses

    def run_training_loop(self, m, X, y, n_classes, hp, sweep_seed, init, exchange_mode=0, master=None):
        d, _h = _model(m)
        dd, keep = _data(X, y, n_classes)
        ch = _hyper(hp)
        init = np.ascontiguousarray(init, np.float32)
        I = hp.i_max
        res = dict(final_params=np.zeros_like(init), batch_loss=np.zeros(I), cumulated=np.zeros(I),
                   exchanged=np.zeros(I, np.uint8), period_len=np.zeros(I, np.uint32))
        out = dsx_loop_out(_p(res["final_params"], C.c_float), _p(res["batch_loss"], C.c_double),
                           _p(res["cumulated"], C.c_double), _p(res["exchanged"], C.c_uint8),
                           _p(res["period_len"], C.c_uint32))
        if master is not None:
            master = np.ascontiguousarray(master, np.float32).copy()
        _check(lib.dsx_run_training_loop(C.byref(d), C.byref(dd), C.byref(ch), sweep_seed, _p(init, C.c_float),
                                         exchange_mode, _p(master, C.c_float), C.byref(out)))
        res["master"] = master
        return res

    def run_worker(self, master_model, master_alpha, master_init, shard_path, hp, rng_seed, worker_model=None,
                   worker_id=0, metrics_path=None, lockfree=False):
        """run_worker (worker.cpp:52-98) against a device center serving `master_model`.
        Returns the LocalRunResult fields plus the center's snapshot ("master") and
        exchange count ("exchanges"); on a handshake error raises ContractError."""
        d, _h = _model(master_model)
        wd = None
        if worker_model is not None:
            wd, _wh = _model(worker_model)
        ch = _hyper(hp)
        init = np.ascontiguousarray(master_init, np.float32)
        I = hp.i_max
        res = dict(final_params=np.zeros_like(init), batch_loss=np.zeros(I), cumulated=np.zeros(I),
                   exchanged=np.zeros(I, np.uint8), period_len=np.zeros(I, np.uint32),
                   master=np.zeros_like(init))
        if worker_model is not None:
            res["final_params"] = np.zeros(self.param_dim(worker_model), np.float32)
        out = dsx_loop_out(_p(res["final_params"], C.c_float), _p(res["batch_loss"], C.c_double),
                           _p(res["cumulated"], C.c_double), _p(res["exchanged"], C.c_uint8),
                           _p(res["period_len"], C.c_uint32))
        cnt = C.c_uint64()
        _check(lib.dsx_run_worker(C.byref(d), master_alpha, 1 if lockfree else 0, _p(init, C.c_float),
                                  C.byref(wd) if wd is not None else None, str(shard_path).encode(), C.byref(ch),
                                  worker_id, rng_seed, metrics_path.encode() if metrics_path else None,
                                  _p(res["master"], C.c_float), C.byref(cnt), C.byref(out)))
        res["exchanges"] = cnt.value
        return res

    def resolve_loss_cut(self, m, X, y, n_classes, hp, sweep_seed, init):
        d, _h = _model(m)
        dd, keep = _data(X, y, n_classes)
        ch = _hyper(hp)
        init = np.ascontiguousarray(init, np.float32)
        cut = C.c_double()
        _check(lib.dsx_resolve_loss_cut(C.byref(d), C.byref(dd), C.byref(ch), sweep_seed, _p(init, C.c_float),
                                        C.byref(cut)))
        return cut.value

    def exchange_order(self, n_workers, tau, i_max, schedule_seed, batch_cost_C=1.0, comm_cost_S=0.0,
                       cost_multipliers=None):
        """Global (worker, iteration) exchange order of simulate_async (Fixed period)."""
        cap = n_workers * (i_max // tau) + 1
        w = np.zeros(cap, np.uint32)
        it = np.zeros(cap, np.uint64)
        cnt = C.c_uint64()
        mults = None if cost_multipliers is None else np.ascontiguousarray(cost_multipliers, np.float64)
        _check(lib.dsx_exchange_order(n_workers, batch_cost_C, comm_cost_S, _p(mults, C.c_double), tau, i_max,
                                      schedule_seed, _p(w, C.c_uint32), _p(it, C.c_uint64), cap, C.byref(cnt)))
        return w[:cnt.value], it[:cnt.value]

    def simulate(self, s, snap_cap: Optional[int] = None, eval_cap: int = 100000):
        """simulate(SimConfig) — s carries SimConfig's fields (+ X, y, n_classes for the dataset)."""
        d, _h = _model(s.model)
        dd, keep = _data(s.X, s.y, s.n_classes)
        mults = None if s.cost_multipliers is None else np.ascontiguousarray(s.cost_multipliers, np.float64)
        cfg = dsx_sim_cfg(s.n_workers, _hyper(s.hyper), d, dd, 1 if s.sync else 0, s.batch_cost_C, s.comm_cost_S,
                          _p(mults, C.c_double), s.schedule_seed, s.init_seed, s.data_seed, s.eval_every,
                          s.holdout_frac, 1 if s.replicate_shards else 0, 1 if s.record_master_snaps else 0)
        Pd = lib.dsx_param_dim(C.byref(d))
        n, I = s.n_workers, s.hyper.i_max
        if snap_cap is None:
            snap_cap = (n * I) if s.record_master_snaps else 0
        o = dict(final_master=np.zeros(Pd, np.float32), worker_final=np.zeros((n, Pd), np.float32),
                 batch_loss=np.zeros((n, I)), cumulated=np.zeros((n, I)), exchanged=np.zeros((n, I), np.uint8),
                 period_len=np.zeros((n, I), np.uint32), wall_ms=np.zeros((n, I), np.int64),
                 snap_worker=np.zeros(snap_cap, np.uint32), snap_time=np.zeros(snap_cap),
                 snap_params=np.zeros((snap_cap, Pd), np.float32), eval_time=np.zeros(eval_cap),
                 eval_iter=np.zeros(eval_cap, np.uint64), eval_acc=np.zeros(eval_cap))
        co = dsx_sim_out(_p(o["final_master"], C.c_float), _p(o["worker_final"], C.c_float),
                         _p(o["batch_loss"], C.c_double), _p(o["cumulated"], C.c_double),
                         _p(o["exchanged"], C.c_uint8), _p(o["period_len"], C.c_uint32), _p(o["wall_ms"], C.c_int64),
                         snap_cap, 0, _p(o["snap_worker"], C.c_uint32), _p(o["snap_time"], C.c_double),
                         _p(o["snap_params"], C.c_float), eval_cap, 0, _p(o["eval_time"], C.c_double),
                         _p(o["eval_iter"], C.c_uint64), _p(o["eval_acc"], C.c_double), 0.0)
        _check(lib.dsx_simulate(C.byref(cfg), C.byref(co)))
        ns, ne = min(co.n_snaps, snap_cap), min(co.n_eval, eval_cap)
        for k in ("snap_worker", "snap_time", "snap_params"):
            o[k] = o[k][:ns]
        for k in ("eval_time", "eval_iter", "eval_acc"):
            o[k] = o[k][:ne]
        o["virtual_total"] = co.virtual_total
        o["n_snaps"] = co.n_snaps
        return o
