// c_api.cpp — deepspark_c.h: flat-buffer entry points over the C++ API, for FFI hosts.
#include "deepspark_c.h"

#include <cstring>
#include <exception>
#include <numeric>
#include <string>

#include "deepspark/dataset.hpp"
#include "deepspark/engine.hpp"
#include "deepspark/errors.hpp"
#include "deepspark/exchanger.hpp"
#include "deepspark/model.hpp"
#include "deepspark/simulator.hpp"
#include "deepspark/worker.hpp"

using namespace deepspark;

namespace {

thread_local std::string g_err;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const ContractError& e) {
    g_err = e.what();
    return 1;
  } catch (const NumericError& e) {
    g_err = e.what();
    return 2;
  } catch (const CudaError& e) {
    g_err = e.what();
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 5;
  }
}

Model model_of(const dsx_model* m) {
  Model out;
  out.kind = m->kind == 0 ? ModelKind::SoftmaxRegression
             : m->kind == 1 ? ModelKind::Mlp
             : m->kind == 2 ? ModelKind::Cifar10Quick
                            : ModelKind::AlexNet;
  out.n_features = m->n_features;
  out.n_classes = m->n_classes;
  out.hidden.assign(m->hidden, m->hidden + m->n_hidden);
  return out;
}

Hyperparams hyper_of(const dsx_hyper* h) {
  Hyperparams hp;
  hp.eta = h->eta;
  hp.alpha = h->alpha;
  hp.tau = h->tau;
  hp.batch_size = h->batch_size;
  hp.i_max = h->i_max;
  hp.loss_cut = h->loss_cut;
  hp.weight_decay = h->weight_decay;
  hp.period_mode = h->adaptive ? PeriodMode::Adaptive : PeriodMode::Fixed;
  return hp;
}

Dataset data_of(const dsx_data* d) {
  Dataset ds;
  ds.n_features = d->n_features;
  ds.n_classes = d->n_classes;
  ds.features.assign(d->X, d->X + d->n * d->n_features);
  ds.labels.assign(d->y, d->y + d->n);
  return ds;
}

std::vector<uint32_t> shuffled_order(uint64_t n, uint64_t seed) {
  std::vector<uint32_t> v(n);
  std::iota(v.begin(), v.end(), 0u);
  Rng r(seed);
  r.shuffle(v);
  return v;
}

}  // namespace

extern "C" {

const char* dsx_last_error(void) { return g_err.c_str(); }

uint64_t dsx_mix_seed(uint64_t seed, uint64_t stream) { return mix_seed(seed, stream); }

void dsx_rng_draws(uint64_t seed, uint64_t n, uint64_t* u64, double* uni, double* nrm, uint64_t bound, uint64_t* below) {
  if (u64) { Rng r(seed); for (uint64_t i = 0; i < n; ++i) u64[i] = r.next_u64(); }
  if (uni) { Rng r(seed); for (uint64_t i = 0; i < n; ++i) uni[i] = r.uniform(); }
  if (nrm) { Rng r(seed); for (uint64_t i = 0; i < n; ++i) nrm[i] = r.normal(); }
  if (below && bound) { Rng r(seed); for (uint64_t i = 0; i < n; ++i) below[i] = r.below(bound); }
}

uint64_t dsx_param_dim(const dsx_model* m) { return model_of(m).param_dim(); }
uint64_t dsx_fingerprint(const dsx_model* m) { return model_of(m).fingerprint(); }

int dsx_init_params(const dsx_model* m, uint64_t seed, float* out) {
  return guard([&] {
    const ParamVector p = init_params(model_of(m), seed);
    std::memcpy(out, p.data(), p.size() * sizeof(float));
  });
}

int dsx_loss_and_grad(const dsx_model* m, const float* params, const float* X, const uint32_t* y, uint32_t rows,
                      float* grad, double* loss) {
  return guard([&] {
    const Model model = model_of(m);
    const size_t P = model.param_dim();
    Minibatch b;
    b.n_features = m->n_features;
    b.features.assign(X, X + static_cast<size_t>(rows) * m->n_features);
    b.labels.assign(y, y + rows);
    if (grad) *loss = loss_and_grad(model, {params, P}, b, {grad, P});
    else *loss = loss_only(model, {params, P}, b);
  });
}

int dsx_predict(const dsx_model* m, const float* params, const float* X, uint64_t rows, uint32_t* out) {
  return guard([&] {
    const Model model = model_of(m);
    for (uint64_t r = 0; r < rows; ++r)
      out[r] = predict(model, {params, model.param_dim()}, {X + r * m->n_features, m->n_features});
  });
}

int dsx_accuracy(const dsx_model* m, const float* params, const dsx_data* d, double* acc) {
  return guard([&] {
    const Model model = model_of(m);
    *acc = accuracy(model, {params, model.param_dim()}, data_of(d));
  });
}

int dsx_sgd_step(const float* x, const float* g, uint64_t n, double eta, float* out) {
  return guard([&] {
    const ParamVector r = sgd_step(ParamVector(x, x + n), ParamVector(g, g + n), eta);
    std::memcpy(out, r.data(), n * sizeof(float));
  });
}

int dsx_easgd_update(const float* w, const float* m, uint64_t n, double alpha, float* w_out, float* m_out) {
  return guard([&] {
    auto [a, b] = easgd_update(ParamVector(w, w + n), ParamVector(m, m + n), alpha);
    std::memcpy(w_out, a.data(), n * sizeof(float));
    std::memcpy(m_out, b.data(), n * sizeof(float));
  });
}

int dsx_gen_synthetic(uint32_t n, uint32_t f, uint32_t c, double sep, double sigma, uint64_t seed, float* X,
                      uint32_t* y) {
  return guard([&] {
    SyntheticSpec s;
    s.n_samples = n;
    s.n_features = f;
    s.n_classes = c;
    s.class_separation = sep;
    s.noise_sigma = sigma;
    s.seed = seed;
    const Dataset ds = gen_synthetic(s);
    std::memcpy(X, ds.features.data(), ds.features.size() * sizeof(float));
    std::memcpy(y, ds.labels.data(), ds.labels.size() * sizeof(uint32_t));
  });
}

// Index orders of split_holdout / partition (dataset.cpp), for hosts that keep the
// rows in their own buffers: holdout = order[0:n_hold), train = order[n_hold:).
int dsx_split_holdout_order(uint64_t n, double frac, uint64_t seed, uint32_t* order, uint64_t* n_hold) {
  return guard([&] {
    if (n == 0) throw ContractError("dataset: no samples");
    if (!(frac > 0.0 && frac < 1.0)) throw ContractError("split_holdout: fraction must lie in (0,1)");
    const auto v = shuffled_order(n, mix_seed(seed, 0x401d));
    const uint64_t h = std::max<uint64_t>(1, static_cast<uint64_t>(n * frac));
    if (h >= n) throw ContractError("split_holdout: nothing left for training");
    std::memcpy(order, v.data(), n * sizeof(uint32_t));
    *n_hold = h;
  });
}

int dsx_partition_order(uint64_t n, uint32_t k, uint64_t seed, uint32_t* order) {
  return guard([&] {
    if (n == 0) throw ContractError("dataset: no samples");
    if (k == 0) throw ContractError("partition: n must be positive");
    if (k > n) throw ContractError("partition: more shards than samples");
    const auto v = shuffled_order(n, mix_seed(seed, 0x5a4d));
    std::memcpy(order, v.data(), n * sizeof(uint32_t));
  });
}

int dsx_sweep_batches(uint64_t shard_n, uint32_t batch, uint64_t seed, uint64_t n_batches, uint32_t* idx,
                      uint32_t* sizes) {
  return guard([&] {
    Dataset ds;
    ds.n_features = 1;
    ds.n_classes = 1;
    ds.features.assign(shard_n, 0.0f);
    ds.labels.assign(shard_n, 0u);
    ShardSweeper sw(ds, batch, seed);
    for (uint64_t b = 0; b < n_batches; ++b) {
      const auto v = sw.next_indices();
      sizes[b] = static_cast<uint32_t>(v.size());
      std::memcpy(idx + b * batch, v.data(), v.size() * sizeof(uint32_t));
    }
  });
}

int dsx_engine_steps(const dsx_model* m, const dsx_data* shard, const dsx_hyper* hp, uint64_t sweep_seed,
                     const float* init, uint64_t steps, float* params, double* losses) {
  return guard([&] {
    const Model model = model_of(m);
    const Dataset ds = data_of(shard);
    SgdEngine eng(model, ds, hyper_of(hp), sweep_seed, ParamVector(init, init + model.param_dim()));
    eng.run(steps, false);
    eng.sync();
    if (losses) {
      const TrainLog log = eng.log(0, steps);
      for (uint64_t s = 0; s < steps; ++s) losses[s] = log[s].batch_loss;
    }
    if (params) std::memcpy(params, eng.params().data(), model.param_dim() * sizeof(float));
  });
}

int dsx_run_training_loop(const dsx_model* m, const dsx_data* shard, const dsx_hyper* hp, uint64_t sweep_seed,
                          const float* init, int exchange_mode, float* master_inout, dsx_loop_out* out) {
  return guard([&] {
    const Model model = model_of(m);
    const size_t P = model.param_dim();
    const Dataset ds = data_of(shard);
    const Hyperparams h = hyper_of(hp);
    LocalRunResult r;
    if (exchange_mode == 2) {
      MasterState master(static_cast<uint32_t>(P), static_cast<float>(h.alpha), UpdateMode::Locked,
                         ParamVector(master_inout, master_inout + P));
      r = run_training_loop(model, ds, h, sweep_seed, ParamVector(init, init + P), master);
      const ParamVector snap = master.snapshot();
      std::memcpy(master_inout, snap.data(), P * sizeof(float));
    } else if (exchange_mode == 1) {
      r = run_training_loop(model, ds, h, sweep_seed, ParamVector(init, init + P),
                            [](const ParamVector& w) { return w; });
    } else {
      r = run_training_loop(model, ds, h, sweep_seed, ParamVector(init, init + P), nullptr);
    }
    if (out->final_params) std::memcpy(out->final_params, r.final_params.data(), P * sizeof(float));
    for (size_t i = 0; i < r.log.size(); ++i) {
      if (out->batch_loss) out->batch_loss[i] = r.log[i].batch_loss;
      if (out->cumulated) out->cumulated[i] = r.log[i].cumulated_loss;
      if (out->exchanged) out->exchanged[i] = r.log[i].exchanged;
      if (out->period_len) out->period_len[i] = r.log[i].period_len;
    }
  });
}

int dsx_run_worker(const dsx_model* master_model, double master_alpha, int master_mode, const float* master_init,
                   const dsx_model* worker_model, const char* shard_path, const dsx_hyper* hp, uint32_t worker_id,
                   uint64_t rng_seed, const char* metrics_path, float* master_out, uint64_t* master_exchanges,
                   dsx_loop_out* out) {
  return guard([&] {
    if (!master_model || !master_init || !shard_path || !hp) throw ContractError("run_worker: null argument");
    const Model served = model_of(master_model);
    const size_t P = served.param_dim();
    MasterState master(static_cast<uint32_t>(P), static_cast<float>(master_alpha),
                       master_mode == 1 ? UpdateMode::LockFree : UpdateMode::Locked,
                       ParamVector(master_init, master_init + P));
    master.bind_model(served);
    WorkerConfig cfg;
    cfg.master = &master;
    cfg.shard_path = shard_path;
    cfg.hyper = hyper_of(hp);
    cfg.worker_id = worker_id;
    cfg.rng_seed = rng_seed;
    cfg.metrics_path = metrics_path ? metrics_path : "";
    if (worker_model) cfg.model = model_of(worker_model);
    auto publish = [&] {
      if (master_out) {
        const ParamVector snap = master.snapshot();
        std::memcpy(master_out, snap.data(), P * sizeof(float));
      }
      if (master_exchanges) *master_exchanges = master.exchange_count();
    };
    LocalRunResult r;
    try {
      r = run_worker(cfg);
    } catch (...) {
      publish();
      throw;
    }
    publish();
    if (out) {
      if (out->final_params) std::memcpy(out->final_params, r.final_params.data(), r.final_params.size() * sizeof(float));
      for (size_t i = 0; i < r.log.size(); ++i) {
        if (out->batch_loss) out->batch_loss[i] = r.log[i].batch_loss;
        if (out->cumulated) out->cumulated[i] = r.log[i].cumulated_loss;
        if (out->exchanged) out->exchanged[i] = r.log[i].exchanged;
        if (out->period_len) out->period_len[i] = r.log[i].period_len;
      }
    }
  });
}

int dsx_resolve_loss_cut(const dsx_model* m, const dsx_data* shard, const dsx_hyper* hp, uint64_t sweep_seed,
                         const float* init, double* cut) {
  return guard([&] {
    const Model model = model_of(m);
    *cut = resolve_loss_cut(hyper_of(hp), model, data_of(shard), sweep_seed,
                            ParamVector(init, init + model.param_dim()))
               .loss_cut;
  });
}

int dsx_simulate(const dsx_sim_cfg* c, dsx_sim_out* o) {
  return guard([&] {
    SimConfig cfg;
    cfg.n_workers = c->n_workers;
    cfg.hyper = hyper_of(&c->hyper);
    cfg.model = model_of(&c->model);
    cfg.dataset = data_of(&c->data);
    cfg.mode = c->sync_mode ? SimMode::Synchronous : SimMode::AsyncEASGD;
    cfg.batch_cost_C = c->batch_cost_C;
    cfg.comm_cost_S = c->comm_cost_S;
    if (c->cost_multipliers) cfg.cost_multipliers.assign(c->cost_multipliers, c->cost_multipliers + c->n_workers);
    cfg.schedule_seed = c->schedule_seed;
    cfg.init_seed = c->init_seed;
    cfg.data_seed = c->data_seed;
    cfg.eval_every = c->eval_every;
    cfg.holdout_frac = c->holdout_frac;
    cfg.replicate_shards = c->replicate_shards != 0;
    cfg.record_master_snaps = c->record_master_snaps != 0;
    const SimResult r = simulate(cfg);
    const size_t P = cfg.model.param_dim();
    const uint64_t I = cfg.hyper.i_max;
    if (o->final_master) std::memcpy(o->final_master, r.final_master.data(), P * sizeof(float));
    for (uint32_t k = 0; k < r.n_workers; ++k) {
      if (o->worker_final) std::memcpy(o->worker_final + k * P, r.worker_final_params[k].data(), P * sizeof(float));
      const TrainLog& log = r.worker_logs[k];
      for (size_t i = 0; i < log.size(); ++i) {
        const size_t at = k * I + i;
        if (o->batch_loss) o->batch_loss[at] = log[i].batch_loss;
        if (o->cumulated) o->cumulated[at] = log[i].cumulated_loss;
        if (o->exchanged) o->exchanged[at] = log[i].exchanged;
        if (o->period_len) o->period_len[at] = log[i].period_len;
        if (o->wall_ms) o->wall_ms[at] = log[i].wall_ms;
      }
    }
    o->n_snaps = r.master_snaps.size();
    for (size_t j = 0; j < r.master_snaps.size() && j < o->snap_cap; ++j) {
      if (o->snap_worker) o->snap_worker[j] = r.master_snaps[j].worker;
      if (o->snap_time) o->snap_time[j] = r.master_snaps[j].virtual_time;
      if (o->snap_params) std::memcpy(o->snap_params + j * P, r.master_snaps[j].params.data(), P * sizeof(float));
    }
    o->n_eval = r.eval_curve.size();
    for (size_t j = 0; j < r.eval_curve.size() && j < o->eval_cap; ++j) {
      if (o->eval_time) o->eval_time[j] = r.eval_curve[j].virtual_time;
      if (o->eval_iter) o->eval_iter[j] = r.eval_curve[j].per_worker_iter;
      if (o->eval_acc) o->eval_acc[j] = r.eval_curve[j].accuracy;
    }
    o->virtual_total = r.virtual_clock_total;
  });
}

int dsx_exchange_order(uint32_t n_workers, double batch_cost_C, double comm_cost_S, const double* mults, uint32_t tau,
                       uint64_t i_max, uint64_t schedule_seed, uint32_t* worker, uint64_t* iteration, uint64_t cap,
                       uint64_t* count) {
  return guard([&] {
    SimConfig cfg;
    cfg.n_workers = n_workers;
    cfg.batch_cost_C = batch_cost_C;
    cfg.comm_cost_S = comm_cost_S;
    if (mults) cfg.cost_multipliers.assign(mults, mults + n_workers);
    cfg.hyper.tau = tau;
    cfg.hyper.i_max = i_max;
    cfg.schedule_seed = schedule_seed;
    const auto ev = exchange_order(cfg);
    *count = ev.size();
    for (size_t j = 0; j < ev.size() && j < cap; ++j) {
      if (worker) worker[j] = ev[j].worker;
      if (iteration) iteration[j] = ev[j].iteration;
    }
  });
}

}  // extern "C"
