// ref_capi.cpp — TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrapper (prefix dsref_) over the UNMODIFIED DeepSpark reference library,
// compiled by oracle/Makefile from /root/reference/proj/src into oracle/_ref/. It calls
// only the reference's public API (proj/include/deepspark/*.hpp) so tests can pin the
// C restatement (ds_oracle.c, prefix dso_) and generate golden vectors, and bench.py's
// --impl reference arm can time the reference's own CPU path. Never used by the product.
#include <chrono>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "deepspark/dataset.hpp"
#include "deepspark/engine.hpp"
#include "deepspark/errors.hpp"
#include "deepspark/exchanger.hpp"
#include "deepspark/model.hpp"
#include "deepspark/param_vector.hpp"
#include "deepspark/rng.hpp"
#include "deepspark/shard.hpp"
#include "deepspark/simulator.hpp"
#include "deepspark/worker.hpp"

extern "C" {
#include "ds_oracle.h"
}

using namespace deepspark;

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const ContractError& e) {
    g_err = e.what();
    return 1;
  } catch (const NumericError& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

Model to_model(const dso_model* m) {
  Model out;
  out.kind = m->kind == 0 ? ModelKind::SoftmaxRegression : ModelKind::Mlp;
  out.n_features = m->n_features;
  out.n_classes = m->n_classes;
  out.hidden.assign(m->hidden, m->hidden + m->n_hidden);
  return out;
}

Hyperparams to_hyper(const dso_hyper* h) {
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

Dataset to_dataset(const dso_data* d) {
  Dataset ds;
  ds.n_features = d->n_features;
  ds.n_classes = d->n_classes;
  ds.features.assign(d->X, d->X + d->n * d->n_features);
  ds.labels.assign(d->y, d->y + d->n);
  return ds;
}

// A 1-feature dataset whose feature is the row index: the reference's shuffles and
// splits copy rows, so reading the feature back recovers the index order exactly.
Dataset index_dataset(uint64_t n) {
  Dataset ds;
  ds.n_features = 1;
  ds.n_classes = 1;
  ds.features.resize(n);
  ds.labels.assign(n, 0u);
  for (uint64_t i = 0; i < n; ++i) ds.features[i] = static_cast<float>(i);
  return ds;
}

Minibatch to_batch(const float* X, const uint32_t* y, uint32_t rows, uint32_t nf) {
  Minibatch b;
  b.n_features = nf;
  b.features.assign(X, X + static_cast<size_t>(rows) * nf);
  b.labels.assign(y, y + rows);
  return b;
}

}  // namespace

extern "C" {

const char* dsref_last_error(void) { return g_err.c_str(); }

uint64_t dsref_mix_seed(uint64_t seed, uint64_t stream) { return mix_seed(seed, stream); }

void dsref_rng_draws(uint64_t seed, uint64_t n, uint64_t* u64, double* uni, double* nrm,
                     uint64_t bound, uint64_t* below) {
  if (u64) { Rng r(seed); for (uint64_t i = 0; i < n; ++i) u64[i] = r.next_u64(); }
  if (uni) { Rng r(seed); for (uint64_t i = 0; i < n; ++i) uni[i] = r.uniform(); }
  if (nrm) { Rng r(seed); for (uint64_t i = 0; i < n; ++i) nrm[i] = r.normal(); }
  if (below && bound) { Rng r(seed); for (uint64_t i = 0; i < n; ++i) below[i] = r.below(bound); }
}

uint64_t dsref_param_dim(const dso_model* m) { return to_model(m).param_dim(); }

uint64_t dsref_fingerprint(const dso_model* m) { return to_model(m).fingerprint(); }

int dsref_init_params(const dso_model* m, uint64_t seed, float* out) {
  return guarded([&] {
    const ParamVector p = init_params(to_model(m), seed);
    std::memcpy(out, p.data(), p.size() * sizeof(float));
  });
}

int dsref_loss_and_grad(const dso_model* m, const float* params, const float* X, const uint32_t* y,
                        uint32_t rows, float* grad, double* loss) {
  return guarded([&] {
    const Model model = to_model(m);
    const size_t P = model.param_dim();
    const Minibatch b = to_batch(X, y, rows, m->n_features);
    if (grad) {
      std::vector<float> g(P);
      *loss = loss_and_grad(model, {params, P}, b, g);
      std::memcpy(grad, g.data(), P * sizeof(float));
    } else {
      *loss = loss_only(model, {params, P}, b);
    }
  });
}

int dsref_predict(const dso_model* m, const float* params, const float* X, uint64_t rows,
                  uint32_t* out) {
  return guarded([&] {
    const Model model = to_model(m);
    const size_t P = model.param_dim();
    for (uint64_t r = 0; r < rows; ++r) {
      out[r] = predict(model, {params, P}, {X + r * m->n_features, m->n_features});
    }
  });
}

int dsref_accuracy(const dso_model* m, const float* params, const dso_data* d, double* acc) {
  return guarded([&] {
    const Model model = to_model(m);
    *acc = accuracy(model, {params, model.param_dim()}, to_dataset(d));
  });
}

int dsref_sgd_step(const float* x, const float* g, uint64_t n, double eta, float* out) {
  return guarded([&] {
    const ParamVector r = sgd_step(ParamVector(x, x + n), ParamVector(g, g + n), eta);
    std::memcpy(out, r.data(), n * sizeof(float));
  });
}

int dsref_easgd_update(const float* w, const float* m, uint64_t n, double alpha, float* w_out,
                       float* m_out) {
  return guarded([&] {
    auto [a, b] = easgd_update(ParamVector(w, w + n), ParamVector(m, m + n), alpha);
    std::memcpy(w_out, a.data(), n * sizeof(float));
    std::memcpy(m_out, b.data(), n * sizeof(float));
  });
}

int dsref_gen_synthetic(uint32_t n, uint32_t f, uint32_t c, double sep, double sigma, uint64_t seed,
                        float* X, uint32_t* y) {
  return guarded([&] {
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

// write_shard (shard.cpp:40-73): golden DSHD files for the device ingestion tests
int dsref_write_shard(const char* path, const float* X, const uint32_t* y, uint64_t n, uint32_t f, uint32_t c,
                      uint64_t seed) {
  return guarded([&] {
    Dataset ds;
    ds.n_features = f;
    ds.n_classes = c;
    ds.features.assign(X, X + n * f);
    ds.labels.assign(y, y + n);
    write_shard(ds, path, seed);
  });
}

int dsref_split_holdout_order(uint64_t n, double frac, uint64_t seed, uint32_t* order,
                              uint64_t* n_hold) {
  return guarded([&] {
    auto [train, hold] = split_holdout(index_dataset(n), frac, seed);
    *n_hold = hold.size();
    size_t k = 0;
    for (float v : hold.features) order[k++] = static_cast<uint32_t>(v);
    for (float v : train.features) order[k++] = static_cast<uint32_t>(v);
  });
}

int dsref_partition_order(uint64_t n, uint32_t k, uint64_t seed, uint32_t* order) {
  return guarded([&] {
    const auto shards = partition(index_dataset(n), k, seed);
    size_t pos = 0;
    for (const auto& s : shards)
      for (float v : s.features) order[pos++] = static_cast<uint32_t>(v);
  });
}

int dsref_sweep_batches(uint64_t shard_n, uint32_t batch, uint64_t seed, uint64_t n_batches,
                        uint32_t* idx, uint32_t* sizes) {
  return guarded([&] {
    const Dataset ds = index_dataset(shard_n);
    ShardSweeper sw(ds, batch, seed);
    Minibatch mb;
    for (uint64_t b = 0; b < n_batches; ++b) {
      sw.next(mb);
      sizes[b] = static_cast<uint32_t>(mb.rows());
      for (size_t j = 0; j < mb.rows(); ++j) idx[b * batch + j] = static_cast<uint32_t>(mb.features[j]);
    }
  });
}

int dsref_engine_steps(const dso_model* m, const dso_data* shard, const dso_hyper* hp,
                       uint64_t sweep_seed, const float* init, uint64_t steps, float* params,
                       double* losses) {
  return guarded([&] {
    const Model model = to_model(m);
    const Dataset ds = to_dataset(shard);
    SgdEngine eng(model, ds, to_hyper(hp), sweep_seed,
                  ParamVector(init, init + model.param_dim()));
    for (uint64_t s = 0; s < steps; ++s) {
      const double l = eng.step();
      if (losses) losses[s] = l;
    }
    if (params) std::memcpy(params, eng.params().data(), eng.params().size() * sizeof(float));
  });
}

int dsref_run_training_loop(const dso_model* m, const dso_data* shard, const dso_hyper* hp,
                            uint64_t sweep_seed, const float* init, int exchange_mode,
                            float* master_inout, dso_loop_out* out) {
  return guarded([&] {
    const Model model = to_model(m);
    const size_t P = model.param_dim();
    const Dataset ds = to_dataset(shard);
    const Hyperparams h = to_hyper(hp);
    ExchangeFn fn = nullptr;
    const float af = static_cast<float>(h.alpha);
    if (exchange_mode == 1) {
      fn = [](const ParamVector& w) { return w; };
    } else if (exchange_mode == 2) {
      fn = [&](const ParamVector& w) {
        ParamVector o(w.size());
        for (size_t i = 0; i < w.size(); ++i) elastic_update_elem(w[i], master_inout[i], af, o[i], master_inout[i]);
        return o;
      };
    }
    const LocalRunResult r = run_training_loop(model, ds, h, sweep_seed, ParamVector(init, init + P), fn);
    if (out->final_params) std::memcpy(out->final_params, r.final_params.data(), P * sizeof(float));
    for (size_t i = 0; i < r.log.size(); ++i) {
      if (out->batch_loss) out->batch_loss[i] = r.log[i].batch_loss;
      if (out->cumulated) out->cumulated[i] = r.log[i].cumulated_loss;
      if (out->exchanged) out->exchanged[i] = r.log[i].exchanged;
      if (out->period_len) out->period_len[i] = r.log[i].period_len;
    }
  });
}

int dsref_resolve_loss_cut(const dso_model* m, const dso_data* shard, const dso_hyper* hp,
                           uint64_t sweep_seed, const float* init, double* cut) {
  return guarded([&] {
    const Model model = to_model(m);
    const Dataset ds = to_dataset(shard);
    const Hyperparams r = resolve_loss_cut(to_hyper(hp), model, ds, sweep_seed,
                                           ParamVector(init, init + model.param_dim()));
    *cut = r.loss_cut;
  });
}

int dsref_simulate(const dso_sim_cfg* c, dso_sim_out* o) {
  return guarded([&] {
    SimConfig cfg;
    cfg.n_workers = c->n_workers;
    cfg.hyper = to_hyper(&c->hyper);
    cfg.model = to_model(&c->model);
    cfg.dataset = to_dataset(&c->data);
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

double dsref_master_exchange_time(uint64_t P, int lockfree, int threads, int iters) {
  std::vector<float> init(P);
  Rng rng(7);
  for (auto& v : init) v = static_cast<float>(rng.uniform(-1.0, 1.0));
  MasterState ms(static_cast<uint32_t>(P), 0.1f, lockfree ? UpdateMode::LockFree : UpdateMode::Locked,
                 init);
  std::vector<std::vector<float>> w(threads, init), out(threads, std::vector<float>(P));
  for (int t = 0; t < threads; ++t)
    for (auto& v : w[t]) v = static_cast<float>(rng.uniform(-1.0, 1.0));
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) {
    pool.emplace_back([&, t] {
      for (int i = 0; i < iters; ++i) ms.exchange(w[t].data(), out[t].data());
    });
  }
  for (auto& th : pool) th.join();
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // extern "C"

// The reference's n-worker EASGD loop (the launch-local shape, main.cpp:443-570, minus
// the TCP wire): one std::thread per worker running SgdEngine::step + ExchangePolicy
// and MasterState::exchange against one in-process master (the exchanger's own
// update rule, exchanger.cpp:76-92). Used by bench.py --impl reference / cpu_baseline.
// Returns the wall seconds of the `steps` timed iterations (after `warmup`), all
// workers started and stopped together; losses_out[k] gets worker k's last loss.
#include <barrier>
extern "C" double dsref_workers_time(const dso_model* m, const dso_data* shards, uint32_t n_workers,
                                     const dso_hyper* hp, const float* init, int lockfree, uint64_t warmup,
                                     uint64_t steps, double* losses_out) {
  try {
    const Model model = to_model(m);
    const size_t P = model.param_dim();
    const Hyperparams h = to_hyper(hp);
    std::vector<Dataset> ds;
    for (uint32_t k = 0; k < n_workers; ++k) ds.push_back(to_dataset(&shards[k]));
    MasterState master(static_cast<uint32_t>(P), static_cast<float>(h.alpha),
                       lockfree ? UpdateMode::LockFree : UpdateMode::Locked, ParamVector(init, init + P));
    std::barrier sync(static_cast<std::ptrdiff_t>(n_workers) + 1);
    std::vector<std::thread> pool;
    for (uint32_t k = 0; k < n_workers; ++k) {
      pool.emplace_back([&, k] {
        SgdEngine eng(model, ds[k], h, mix_seed(1234, k), ParamVector(init, init + P));
        ExchangePolicy pol(h);
        ParamVector out(P);
        double loss = 0.0;
        auto iterate = [&](uint64_t n) {
          for (uint64_t i = 0; i < n; ++i) {
            loss = eng.step();
            if (pol.on_iteration(loss).exchange) {
              master.exchange(eng.params().data(), out.data());
              eng.set_params(out);
            }
          }
        };
        iterate(warmup);
        sync.arrive_and_wait();
        iterate(steps);
        sync.arrive_and_wait();
        if (losses_out) losses_out[k] = loss;
      });
    }
    sync.arrive_and_wait();
    const auto t0 = std::chrono::steady_clock::now();
    sync.arrive_and_wait();
    const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    for (auto& t : pool) t.join();
    return s;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1.0;
  }
}
