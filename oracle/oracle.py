"""oracle.py — TEST INFRASTRUCTURE ONLY.

ctypes access to the two CPU checkers declared in ``oracle/ds_oracle.h``:

* ``Oracle("dso")``   — the C restatement (``oracle/libds_oracle.so``), always available;
* ``Oracle("dsref")`` — the unmodified reference (``oracle/_ref/libdeepspark_ref.so``),
  available where it was built (this container, or a GPU box that received the
  prebuilt library in the gpurun snapshot).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs import this module. The product never does.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "dso": os.path.join(HERE, "libds_oracle.so"),
    "dsref": os.path.join(HERE, "_ref", "libdeepspark_ref.so"),
}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class ContractError(OracleError):
    pass


class NumericError(OracleError):
    pass


class dso_model(C.Structure):
    _fields_ = [("kind", C.c_int32), ("n_features", C.c_uint32), ("n_classes", C.c_uint32),
                ("n_hidden", C.c_uint32), ("hidden", C.POINTER(C.c_uint32))]


class dso_hyper(C.Structure):
    _fields_ = [("eta", C.c_double), ("alpha", C.c_double), ("tau", C.c_uint32),
                ("batch_size", C.c_uint32), ("i_max", C.c_uint64), ("loss_cut", C.c_double),
                ("weight_decay", C.c_double), ("adaptive", C.c_int32)]


class dso_data(C.Structure):
    _fields_ = [("X", C.POINTER(C.c_float)), ("y", C.POINTER(C.c_uint32)), ("n", C.c_uint64),
                ("n_features", C.c_uint32), ("n_classes", C.c_uint32)]


class dso_sim_cfg(C.Structure):
    _fields_ = [("n_workers", C.c_uint32), ("hyper", dso_hyper), ("model", dso_model),
                ("data", dso_data), ("sync_mode", C.c_int32), ("batch_cost_C", C.c_double),
                ("comm_cost_S", C.c_double), ("cost_multipliers", C.POINTER(C.c_double)),
                ("schedule_seed", C.c_uint64), ("init_seed", C.c_uint64), ("data_seed", C.c_uint64),
                ("eval_every", C.c_uint32), ("holdout_frac", C.c_double),
                ("replicate_shards", C.c_int32), ("record_master_snaps", C.c_int32)]


class dso_sim_out(C.Structure):
    _fields_ = [("final_master", C.POINTER(C.c_float)), ("worker_final", C.POINTER(C.c_float)),
                ("batch_loss", C.POINTER(C.c_double)), ("cumulated", C.POINTER(C.c_double)),
                ("exchanged", C.POINTER(C.c_uint8)), ("period_len", C.POINTER(C.c_uint32)),
                ("wall_ms", C.POINTER(C.c_int64)), ("snap_cap", C.c_uint64), ("n_snaps", C.c_uint64),
                ("snap_worker", C.POINTER(C.c_uint32)), ("snap_time", C.POINTER(C.c_double)),
                ("snap_params", C.POINTER(C.c_float)), ("eval_cap", C.c_uint64), ("n_eval", C.c_uint64),
                ("eval_time", C.POINTER(C.c_double)), ("eval_iter", C.POINTER(C.c_uint64)),
                ("eval_acc", C.POINTER(C.c_double)), ("virtual_total", C.c_double)]


class dso_loop_out(C.Structure):
    _fields_ = [("final_params", C.POINTER(C.c_float)), ("batch_loss", C.POINTER(C.c_double)),
                ("cumulated", C.POINTER(C.c_double)), ("exchanged", C.POINTER(C.c_uint8)),
                ("period_len", C.POINTER(C.c_uint32))]


def _p(a: Optional[np.ndarray], ct):
    if a is None:
        return C.cast(None, C.POINTER(ct))
    assert a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(C.POINTER(ct))


@dataclass
class ModelSpec:
    """Mirror of deepspark::Model (model.hpp:32-56): kind 'softmax' | 'mlp', plus
    'cifar10_quick' (kind 2) and 'alexnet' (kind 3), NOT IN THE REFERENCE
    (oracle/ds_oracle_cnn.h, oracle/ds_oracle_alex.h)."""
    kind: str
    n_features: int
    n_classes: int
    hidden: Sequence[int] = ()

    @staticmethod
    def softmax(f: int, c: int) -> "ModelSpec":
        return ModelSpec("softmax", f, c, ())

    @staticmethod
    def mlp(f: int, hidden: Sequence[int], c: int) -> "ModelSpec":
        return ModelSpec("mlp", f, c, tuple(hidden))

    @staticmethod
    def cifar10_quick(c: int = 10) -> "ModelSpec":
        return ModelSpec("cifar10_quick", 3072, c, ())

    @staticmethod
    def alexnet(side: int = 224, c: int = 1000) -> "ModelSpec":
        """AlexNet-shaped (kind 3, NOT IN THE REFERENCE; oracle/ds_oracle_alex.h)."""
        return ModelSpec("alexnet", 3 * side * side, c, ())

    def c(self):
        h = np.ascontiguousarray(np.asarray(self.hidden, dtype=np.uint32))
        m = dso_model({"softmax": 0, "mlp": 1, "cifar10_quick": 2, "alexnet": 3}[self.kind], self.n_features, self.n_classes,
                      len(self.hidden), _p(h if len(self.hidden) else None, C.c_uint32))
        return m, h  # keep h alive


@dataclass
class Hyper:
    """Mirror of deepspark::Hyperparams (hyperparams.hpp:10-21)."""
    eta: float = 0.05
    alpha: float = 0.1
    tau: int = 100
    batch_size: int = 32
    i_max: int = 1000
    loss_cut: float = 0.0
    weight_decay: float = 0.0
    adaptive: bool = False

    def c(self):
        return dso_hyper(self.eta, self.alpha, self.tau, self.batch_size, self.i_max,
                         self.loss_cut, self.weight_decay, 1 if self.adaptive else 0)


@dataclass
class SimSpec:
    """Mirror of deepspark::SimConfig (simulator.hpp:24-54)."""
    n_workers: int
    hyper: Hyper
    model: ModelSpec
    X: np.ndarray
    y: np.ndarray
    n_classes: int
    sync: bool = False
    batch_cost_C: float = 1.0
    comm_cost_S: float = 0.0
    cost_multipliers: Optional[Sequence[float]] = None
    schedule_seed: int = 0
    init_seed: int = 0
    data_seed: int = 0
    eval_every: int = 50
    holdout_frac: float = 0.2
    replicate_shards: bool = False
    record_master_snaps: bool = True


@dataclass
class SimOut:
    final_master: np.ndarray
    worker_final: np.ndarray
    batch_loss: np.ndarray
    cumulated: np.ndarray
    exchanged: np.ndarray
    period_len: np.ndarray
    wall_ms: np.ndarray
    snap_worker: np.ndarray
    snap_time: np.ndarray
    snap_params: np.ndarray
    eval_time: np.ndarray
    eval_iter: np.ndarray
    eval_acc: np.ndarray
    virtual_total: float
    n_snaps: int = 0


class Oracle:
    def __init__(self, prefix: str = "dso"):
        path = LIBS[prefix]
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle{' ref' if prefix == 'dsref' else ''}`")
        self.prefix = prefix
        self.lib = C.CDLL(path)
        L = self.lib

        def f(name, res, *args):
            fn = getattr(L, f"{prefix}_{name}")
            fn.restype = res
            fn.argtypes = list(args)
            setattr(self, "_" + name, fn)

        P = C.POINTER
        f("last_error", C.c_char_p)
        f("mix_seed", C.c_uint64, C.c_uint64, C.c_uint64)
        f("rng_draws", None, C.c_uint64, C.c_uint64, P(C.c_uint64), P(C.c_double), P(C.c_double),
          C.c_uint64, P(C.c_uint64))
        f("param_dim", C.c_uint64, P(dso_model))
        f("fingerprint", C.c_uint64, P(dso_model))
        f("init_params", C.c_int, P(dso_model), C.c_uint64, P(C.c_float))
        f("loss_and_grad", C.c_int, P(dso_model), P(C.c_float), P(C.c_float), P(C.c_uint32),
          C.c_uint32, P(C.c_float), P(C.c_double))
        f("predict", C.c_int, P(dso_model), P(C.c_float), P(C.c_float), C.c_uint64, P(C.c_uint32))
        f("accuracy", C.c_int, P(dso_model), P(C.c_float), P(dso_data), P(C.c_double))
        f("sgd_step", C.c_int, P(C.c_float), P(C.c_float), C.c_uint64, C.c_double, P(C.c_float))
        f("easgd_update", C.c_int, P(C.c_float), P(C.c_float), C.c_uint64, C.c_double,
          P(C.c_float), P(C.c_float))
        f("gen_synthetic", C.c_int, C.c_uint32, C.c_uint32, C.c_uint32, C.c_double, C.c_double,
          C.c_uint64, P(C.c_float), P(C.c_uint32))
        f("split_holdout_order", C.c_int, C.c_uint64, C.c_double, C.c_uint64, P(C.c_uint32),
          P(C.c_uint64))
        f("partition_order", C.c_int, C.c_uint64, C.c_uint32, C.c_uint64, P(C.c_uint32))
        f("sweep_batches", C.c_int, C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint64, P(C.c_uint32),
          P(C.c_uint32))
        f("engine_steps", C.c_int, P(dso_model), P(dso_data), P(dso_hyper), C.c_uint64,
          P(C.c_float), C.c_uint64, P(C.c_float), P(C.c_double))
        f("run_training_loop", C.c_int, P(dso_model), P(dso_data), P(dso_hyper), C.c_uint64,
          P(C.c_float), C.c_int, P(C.c_float), P(dso_loop_out))
        f("resolve_loss_cut", C.c_int, P(dso_model), P(dso_data), P(dso_hyper), C.c_uint64,
          P(C.c_float), P(C.c_double))
        f("simulate", C.c_int, P(dso_sim_cfg), P(dso_sim_out))
        if prefix == "dsref":
            L.dsref_master_exchange_time.restype = C.c_double
            L.dsref_master_exchange_time.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int]

    # -- helpers -----------------------------------------------------------------------
    def _check(self, rc: int):
        if rc == 0:
            return
        msg = self._last_error().decode(errors="replace")
        if rc == 1:
            raise ContractError(rc, msg)
        if rc == 2:
            raise NumericError(rc, msg)
        raise OracleError(rc, msg)

    @staticmethod
    def _data(X: np.ndarray, y: np.ndarray, n_classes: int):
        X = np.ascontiguousarray(X, dtype=np.float32)
        y = np.ascontiguousarray(y, dtype=np.uint32)
        d = dso_data(_p(X, C.c_float), _p(y, C.c_uint32), y.shape[0], X.shape[1] if X.ndim == 2 else 0,
                     n_classes)
        return d, (X, y)

    # -- API ---------------------------------------------------------------------------
    def mix_seed(self, seed: int, stream: int) -> int:
        return self._mix_seed(seed, stream)

    def rng_draws(self, seed: int, n: int, bound: int = 0):
        u = np.zeros(n, np.uint64)
        uni = np.zeros(n, np.float64)
        nrm = np.zeros(n, np.float64)
        bel = np.zeros(n, np.uint64)
        self._rng_draws(seed, n, _p(u, C.c_uint64), _p(uni, C.c_double), _p(nrm, C.c_double),
                        bound, _p(bel, C.c_uint64) if bound else _p(None, C.c_uint64))
        return u, uni, nrm, bel

    def param_dim(self, m: ModelSpec) -> int:
        cm, _h = m.c()
        return self._param_dim(C.byref(cm))

    def fingerprint(self, m: ModelSpec) -> int:
        cm, _h = m.c()
        return self._fingerprint(C.byref(cm))

    def init_params(self, m: ModelSpec, seed: int) -> np.ndarray:
        cm, _h = m.c()
        out = np.zeros(self._param_dim(C.byref(cm)), np.float32)
        self._check(self._init_params(C.byref(cm), seed, _p(out, C.c_float)))
        return out

    def loss_and_grad(self, m: ModelSpec, params, X, y, want_grad: bool = True):
        cm, _h = m.c()
        params = np.ascontiguousarray(params, np.float32)
        X = np.ascontiguousarray(X, np.float32)
        y = np.ascontiguousarray(y, np.uint32)
        g = np.zeros(params.shape[0], np.float32) if want_grad else None
        loss = C.c_double()
        self._check(self._loss_and_grad(C.byref(cm), _p(params, C.c_float), _p(X, C.c_float),
                                        _p(y, C.c_uint32), y.shape[0], _p(g, C.c_float), C.byref(loss)))
        return loss.value, g

    def predict(self, m: ModelSpec, params, X) -> np.ndarray:
        cm, _h = m.c()
        params = np.ascontiguousarray(params, np.float32)
        X = np.ascontiguousarray(X, np.float32)
        out = np.zeros(X.shape[0], np.uint32)
        self._check(self._predict(C.byref(cm), _p(params, C.c_float), _p(X, C.c_float), X.shape[0],
                                  _p(out, C.c_uint32)))
        return out

    def accuracy(self, m: ModelSpec, params, X, y, n_classes) -> float:
        cm, _h = m.c()
        params = np.ascontiguousarray(params, np.float32)
        d, keep = self._data(X, y, n_classes)
        acc = C.c_double()
        self._check(self._accuracy(C.byref(cm), _p(params, C.c_float), C.byref(d), C.byref(acc)))
        return acc.value

    def sgd_step(self, x, g, eta: float) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float32)
        g = np.ascontiguousarray(g, np.float32)
        out = np.zeros_like(x)
        self._check(self._sgd_step(_p(x, C.c_float), _p(g, C.c_float), x.shape[0], eta, _p(out, C.c_float)))
        return out

    def easgd_update(self, w, m, alpha: float):
        w = np.ascontiguousarray(w, np.float32)
        m = np.ascontiguousarray(m, np.float32)
        wo = np.zeros_like(w)
        mo = np.zeros_like(m)
        self._check(self._easgd_update(_p(w, C.c_float), _p(m, C.c_float), w.shape[0], alpha,
                                       _p(wo, C.c_float), _p(mo, C.c_float)))
        return wo, mo

    @staticmethod
    def sync_easgd_round(workers, center, alpha: float):
        """Synchronous EASGD round (EXTENSION, not in the reference: the EASGD paper's
        synchronous variant with the reference's elastic arithmetic, param_vector.cpp:41-61):
        e_k = f32(alpha * f32(x_k - c)); x_k' = x_k - e_k; c' = c + f32(sum_k e_k), the sum
        in f64 in worker order. numpy f32 operations round once each, like the C oracle."""
        a = np.float32(alpha)
        c = np.ascontiguousarray(center, np.float32)
        s = np.zeros(c.shape, np.float64)
        outs = []
        for x in workers:
            x = np.ascontiguousarray(x, np.float32)
            e = (a * (x - c)).astype(np.float32)
            s = s + e.astype(np.float64)
            outs.append((x - e).astype(np.float32))
        return outs, (c + s.astype(np.float32)).astype(np.float32)

    @staticmethod
    def sync_sgd_round(x, grads, eta: float, wd: float = 0.0):
        """One simulate_sync master update (simulator.cpp:192-210): gsum in f64 in worker
        order, gavg = f32(gsum / n), gavg += f32(wd) * x, sgd_step (param_vector.cpp:21-39)."""
        x = np.ascontiguousarray(x, np.float32)
        gs = np.zeros(x.shape, np.float64)
        for g in grads:
            gs = gs + np.asarray(g, np.float32).astype(np.float64)
        g = (gs / np.float64(len(grads))).astype(np.float32)
        if wd > 0:
            g = (g + (np.float32(wd) * x).astype(np.float32)).astype(np.float32)
        return (x - (np.float32(eta) * g).astype(np.float32)).astype(np.float32)

    def gen_synthetic(self, n, f, c, sep, sigma, seed):
        X = np.zeros((n, f), np.float32)
        y = np.zeros(n, np.uint32)
        self._check(self._gen_synthetic(n, f, c, sep, sigma, seed, _p(X, C.c_float), _p(y, C.c_uint32)))
        return X, y

    def split_holdout_order(self, n, frac, seed):
        order = np.zeros(n, np.uint32)
        nh = C.c_uint64()
        self._check(self._split_holdout_order(n, frac, seed, _p(order, C.c_uint32), C.byref(nh)))
        return order, nh.value

    def partition_order(self, n, k, seed):
        order = np.zeros(n, np.uint32)
        self._check(self._partition_order(n, k, seed, _p(order, C.c_uint32)))
        return order

    def sweep_batches(self, shard_n, batch, seed, n_batches):
        idx = np.zeros(n_batches * batch, np.uint32)
        sizes = np.zeros(n_batches, np.uint32)
        self._check(self._sweep_batches(shard_n, batch, seed, n_batches, _p(idx, C.c_uint32),
                                        _p(sizes, C.c_uint32)))
        return idx.reshape(n_batches, batch), sizes

    def engine_steps(self, m: ModelSpec, X, y, n_classes, hp: Hyper, sweep_seed, init, steps):
        cm, _h = m.c()
        d, keep = self._data(X, y, n_classes)
        ch = hp.c()
        init = np.ascontiguousarray(init, np.float32)
        params = np.zeros_like(init)
        losses = np.zeros(steps, np.float64)
        self._check(self._engine_steps(C.byref(cm), C.byref(d), C.byref(ch), sweep_seed,
                                       _p(init, C.c_float), steps, _p(params, C.c_float),
                                       _p(losses, C.c_double)))
        return params, losses

    def run_training_loop(self, m: ModelSpec, X, y, n_classes, hp: Hyper, sweep_seed, init,
                          exchange_mode=0, master=None):
        cm, _h = m.c()
        d, keep = self._data(X, y, n_classes)
        ch = hp.c()
        init = np.ascontiguousarray(init, np.float32)
        I = hp.i_max
        res = dict(final_params=np.zeros_like(init), batch_loss=np.zeros(I), cumulated=np.zeros(I),
                   exchanged=np.zeros(I, np.uint8), period_len=np.zeros(I, np.uint32))
        out = dso_loop_out(_p(res["final_params"], C.c_float), _p(res["batch_loss"], C.c_double),
                           _p(res["cumulated"], C.c_double), _p(res["exchanged"], C.c_uint8),
                           _p(res["period_len"], C.c_uint32))
        if master is not None:
            master = np.ascontiguousarray(master, np.float32).copy()
        self._check(self._run_training_loop(C.byref(cm), C.byref(d), C.byref(ch), sweep_seed,
                                            _p(init, C.c_float), exchange_mode, _p(master, C.c_float),
                                            C.byref(out)))
        res["master"] = master
        return res

    def resolve_loss_cut(self, m: ModelSpec, X, y, n_classes, hp: Hyper, sweep_seed, init) -> float:
        cm, _h = m.c()
        d, keep = self._data(X, y, n_classes)
        ch = hp.c()
        init = np.ascontiguousarray(init, np.float32)
        cut = C.c_double()
        self._check(self._resolve_loss_cut(C.byref(cm), C.byref(d), C.byref(ch), sweep_seed,
                                           _p(init, C.c_float), C.byref(cut)))
        return cut.value

    def simulate(self, s: SimSpec, snap_cap: Optional[int] = None, eval_cap: int = 100000) -> SimOut:
        cm, _h = s.model.c()
        d, keep = self._data(s.X, s.y, s.n_classes)
        mults = None if s.cost_multipliers is None else np.ascontiguousarray(s.cost_multipliers, np.float64)
        cfg = dso_sim_cfg(s.n_workers, s.hyper.c(), cm, d, 1 if s.sync else 0, s.batch_cost_C, s.comm_cost_S,
                          _p(mults, C.c_double), s.schedule_seed, s.init_seed, s.data_seed, s.eval_every,
                          s.holdout_frac, 1 if s.replicate_shards else 0, 1 if s.record_master_snaps else 0)
        P = self._param_dim(C.byref(cm))
        n, I = s.n_workers, s.hyper.i_max
        if snap_cap is None:
            snap_cap = (n * I) if s.record_master_snaps else 0
        o = SimOut(final_master=np.zeros(P, np.float32), worker_final=np.zeros((n, P), np.float32),
                   batch_loss=np.zeros((n, I)), cumulated=np.zeros((n, I)),
                   exchanged=np.zeros((n, I), np.uint8), period_len=np.zeros((n, I), np.uint32),
                   wall_ms=np.zeros((n, I), np.int64), snap_worker=np.zeros(snap_cap, np.uint32),
                   snap_time=np.zeros(snap_cap), snap_params=np.zeros((snap_cap, P), np.float32),
                   eval_time=np.zeros(eval_cap), eval_iter=np.zeros(eval_cap, np.uint64),
                   eval_acc=np.zeros(eval_cap), virtual_total=0.0)
        co = dso_sim_out(_p(o.final_master, C.c_float), _p(o.worker_final, C.c_float),
                         _p(o.batch_loss, C.c_double), _p(o.cumulated, C.c_double),
                         _p(o.exchanged, C.c_uint8), _p(o.period_len, C.c_uint32), _p(o.wall_ms, C.c_int64),
                         snap_cap, 0, _p(o.snap_worker, C.c_uint32), _p(o.snap_time, C.c_double),
                         _p(o.snap_params, C.c_float), eval_cap, 0, _p(o.eval_time, C.c_double),
                         _p(o.eval_iter, C.c_uint64), _p(o.eval_acc, C.c_double), 0.0)
        self._check(self._simulate(C.byref(cfg), C.byref(co)))
        ns = min(co.n_snaps, snap_cap)
        ne = min(co.n_eval, eval_cap)
        o.n_snaps = co.n_snaps
        o.snap_worker, o.snap_time, o.snap_params = o.snap_worker[:ns], o.snap_time[:ns], o.snap_params[:ns]
        o.eval_time, o.eval_iter, o.eval_acc = o.eval_time[:ne], o.eval_iter[:ne], o.eval_acc[:ne]
        o.virtual_total = co.virtual_total
        return o

    def master_exchange_time(self, P: int, lockfree: bool, threads: int, iters: int) -> float:
        assert self.prefix == "dsref"
        return self.lib.dsref_master_exchange_time(P, 1 if lockfree else 0, threads, iters)

    def workers_time(self, m: ModelSpec, shards, n_classes: int, hp: Hyper, init, lockfree: bool, warmup: int,
                     steps: int) -> float:
        """Reference n-worker loop (threads) — wall seconds of `steps` iterations per worker."""
        assert self.prefix == "dsref"
        L = self.lib
        L.dsref_workers_time.restype = C.c_double
        L.dsref_workers_time.argtypes = [C.POINTER(dso_model), C.POINTER(dso_data), C.c_uint32,
                                         C.POINTER(dso_hyper), C.POINTER(C.c_float), C.c_int, C.c_uint64,
                                         C.c_uint64, C.POINTER(C.c_double)]
        cm, _h = m.c()
        keep = []
        arr = (dso_data * len(shards))()
        for k, (X, y) in enumerate(shards):
            d, kk = self._data(X, y, n_classes)
            keep.append(kk)
            arr[k] = d
        ch = hp.c()
        init = np.ascontiguousarray(init, np.float32)
        losses = np.zeros(len(shards))
        s = L.dsref_workers_time(C.byref(cm), arr, len(shards), C.byref(ch), _p(init, C.c_float),
                                 1 if lockfree else 0, warmup, steps, _p(losses, C.c_double))
        if s < 0:
            raise OracleError(3, self._last_error().decode())
        return s


def available(prefix: str) -> bool:
    return os.path.exists(LIBS[prefix])
