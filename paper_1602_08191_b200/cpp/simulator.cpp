// simulate() on a B200 — reference simulator.cpp:16-265.
//
// Async EASGD: every worker is a device-resident SgdEngine and the master is the device
// center. The host pops the reference's seeded virtual-clock event queue
// (simulator.cpp:91-143) and, per event, runs that worker's next iteration on the GPU;
// when the device policy fires, the elastic exchange runs as a device kernel against
// the center, in event order. Holdout evaluation is a device kernel on the center.
// Sync: per round every worker's gradient at the master is summed in f64 on the device,
// averaged, rounded to f32 and applied (simulator.cpp:156-223).
#include "deepspark/simulator.hpp"

#include <algorithm>
#include <cmath>
#include <queue>
#include <tuple>

#include "deepspark/errors.hpp"
#include "deepspark/exchanger.hpp"
#include "deepspark/rng.hpp"
#include "deepspark/worker.hpp"
#include "device_ctx.hpp"

namespace deepspark {

namespace {
constexpr uint64_t kSweepTag = 0x53574550;  // "SWEP"
constexpr uint64_t kPartTag = 0x50415254;   // "PART"
constexpr uint64_t kHoldTag = 0x484f4c44;   // "HOLD"

double mult(const SimConfig& cfg, uint32_t k) { return cfg.cost_multipliers.empty() ? 1.0 : cfg.cost_multipliers[k]; }

struct Event {
  double t;
  uint64_t tie;
  uint32_t worker;
  bool operator>(const Event& o) const { return std::tie(t, tie, worker) > std::tie(o.t, o.tie, o.worker); }
};

// The holdout, resident on the device, scored against device-resident parameters.
class DeviceHoldout {
 public:
  DeviceHoldout(const Model& m, const Dataset& ds)
      : n_(ds.size()), X_(ds.features.size() * sizeof(float)), y_(ds.size() * sizeof(uint32_t)), hits_(64) {
    auto& ctx = detail::DeviceCtx::get();
    ctx.upload(X_.as<void>(), ds.features.data(), ds.features.size() * sizeof(float));
    ctx.upload(y_.as<void>(), ds.labels.data(), ds.size() * sizeof(uint32_t));
    ctx.sync();
    hidden_ = m.hidden;
    d_ = ds_model_desc{model_kind_code(m.kind), m.n_features, m.n_classes,
                       static_cast<uint32_t>(hidden_.size()), hidden_.data()};
  }
  double accuracy_of(const float* dparams) {
    auto& ctx = detail::DeviceCtx::get();
    check_status(ds_memset(hits_.as<void>(), 0, sizeof(unsigned long long), ctx.stream()), "eval");
    check_status(ds_count_hits(&d_, dparams, X_.as<float>(), y_.as<uint32_t>(), n_, hits_.as<unsigned long long>(),
                               ctx.stream()),
                 "eval");
    unsigned long long h = 0;
    ctx.download(&h, hits_.as<void>(), sizeof(h));
    ctx.sync();
    return static_cast<double>(h) / static_cast<double>(n_);
  }

 private:
  size_t n_;
  detail::DeviceBuffer X_, y_, hits_;
  std::vector<uint32_t> hidden_;
  ds_model_desc d_{};
};

float* master_device_ptr(MasterState& m) {
  float* p = nullptr;
  check_status(ds_master_local_slice(m.handle(), &p, nullptr, nullptr), "simulate");
  return p;
}

SimResult simulate_async(const SimConfig& cfg, const std::vector<const Dataset*>& shards, const Dataset& holdout,
                         ParamVector master0) {
  const uint32_t n = cfg.n_workers;
  const float alpha_f = static_cast<float>(cfg.hyper.alpha);
  SimResult res;
  res.n_workers = n;
  res.worker_logs.resize(n);
  std::vector<SgdEngine> engines;
  engines.reserve(n);
  for (uint32_t k = 0; k < n; ++k) {
    const Hyperparams hp = resolve_loss_cut(cfg.hyper, cfg.model, *shards[k], sim_sweep_seed(cfg, k), master0);
    hp.validate();
    engines.emplace_back(cfg.model, *shards[k], hp, sim_sweep_seed(cfg, k), master0);
    res.worker_logs[k].reserve(hp.i_max);
  }
  MasterState master(static_cast<uint32_t>(master0.size()), alpha_f, UpdateMode::Locked, master0);
  float* dmaster = master_device_ptr(master);
  DeviceHoldout eval(cfg.model, holdout);

  Rng sched(cfg.schedule_seed);
  std::priority_queue<Event, std::vector<Event>, std::greater<Event>> pq;
  std::vector<uint64_t> done(n, 0);
  for (uint32_t k = 0; k < n; ++k) pq.push({cfg.batch_cost_C * mult(cfg, k), sched.next_u64(), k});
  res.eval_curve.push_back({0.0, 0, eval.accuracy_of(dmaster)});
  uint64_t next_eval = cfg.eval_every;
  double total = 0.0;
  while (!pq.empty()) {
    const Event ev = pq.top();
    pq.pop();
    const uint32_t k = ev.worker;
    engines[k].run(1, true);
    engines[k].sync();
    ++done[k];
    TrainRecord rec = engines[k].log(done[k] - 1, 1)[0];
    double next_t = ev.t + cfg.batch_cost_C * mult(cfg, k);
    if (rec.exchanged) {
      engines[k].exchange_with(master);  // device kernel, in event order
      engines[k].sync();
      if (cfg.record_master_snaps) res.master_snaps.push_back({ev.t, k, master.snapshot()});
      next_t += cfg.comm_cost_S;
      total = std::max(total, ev.t + cfg.comm_cost_S);
    } else {
      total = std::max(total, ev.t);
    }
    rec.iter = done[k];
    rec.wall_ms = std::llround(ev.t);
    res.worker_logs[k].push_back(rec);
    if (done[k] < cfg.hyper.i_max) pq.push({next_t, sched.next_u64(), k});
    const uint64_t min_iter = *std::min_element(done.begin(), done.end());
    while (next_eval <= min_iter) {
      res.eval_curve.push_back({ev.t, next_eval, eval.accuracy_of(dmaster)});
      next_eval += cfg.eval_every;
    }
  }
  if (res.eval_curve.back().per_worker_iter != cfg.hyper.i_max)
    res.eval_curve.push_back({total, cfg.hyper.i_max, eval.accuracy_of(dmaster)});
  for (uint32_t k = 0; k < n; ++k) res.worker_final_params.push_back(engines[k].params());
  res.final_master = master.snapshot();
  res.virtual_clock_total = total;
  res.iterations_per_worker = cfg.hyper.i_max;
  return res;
}

SimResult simulate_sync(const SimConfig& cfg, const std::vector<const Dataset*>& shards, const Dataset& holdout,
                        ParamVector master0) {
  const uint32_t n = cfg.n_workers;
  const size_t P = master0.size();
  const float wd = static_cast<float>(cfg.hyper.weight_decay);
  const uint32_t B = cfg.hyper.batch_size;
  std::vector<ShardSweeper> sweepers;
  sweepers.reserve(n);
  for (uint32_t k = 0; k < n; ++k) sweepers.emplace_back(*shards[k], B, sim_sweep_seed(cfg, k));

  SimResult res;
  res.n_workers = n;
  res.worker_logs.resize(n);
  double round_cost = 0.0;
  for (uint32_t k = 0; k < n; ++k) round_cost = std::max(round_cost, cfg.batch_cost_C * mult(cfg, k));
  round_cost += cfg.comm_cost_S;

  auto& ctx = detail::DeviceCtx::get();
  std::vector<uint32_t> hidden = cfg.model.hidden;
  const ds_model_desc d{model_kind_code(cfg.model.kind), cfg.model.n_features,
                        cfg.model.n_classes, static_cast<uint32_t>(hidden.size()), hidden.data()};
  uint64_t ws_bytes = 0;
  check_status(ds_loss_and_grad_workspace(&d, B, &ws_bytes), "simulate");
  detail::DeviceBuffer dm(P * sizeof(float)), gsum(P * sizeof(double)), gk(P * sizeof(float)), gavg(P * sizeof(float)),
      dX(static_cast<size_t>(B) * cfg.model.n_features * sizeof(float)), dy(B * sizeof(uint32_t)), ws(ws_bytes),
      losses(n * sizeof(double)), flags(64);
  ctx.upload(dm.as<void>(), master0.data(), P * sizeof(float));
  DeviceHoldout eval(cfg.model, holdout);
  res.eval_curve.push_back({0.0, 0, eval.accuracy_of(dm.as<float>())});
  uint64_t next_eval = cfg.eval_every;
  Minibatch batch;
  std::vector<double> hl(n);
  double t = 0.0;
  for (uint64_t r = 1; r <= cfg.hyper.i_max; ++r) {
    t += round_cost;
    check_status(ds_memset(gsum.as<void>(), 0, P * sizeof(double), ctx.stream()), "simulate");
    check_status(ds_memset(flags.as<void>(), 0, sizeof(uint32_t), ctx.stream()), "simulate");
    for (uint32_t k = 0; k < n; ++k) {
      sweepers[k].next(batch);
      for (uint32_t y : batch.labels)
        if (y >= cfg.model.n_classes) throw ContractError("loss_and_grad: label " + std::to_string(y) + " out of range");
      ctx.upload(dX.as<void>(), batch.features.data(), batch.features.size() * sizeof(float));
      ctx.upload(dy.as<void>(), batch.labels.data(), batch.labels.size() * sizeof(uint32_t));
      check_status(ds_loss_and_grad(&d, dm.as<float>(), dX.as<float>(), dy.as<uint32_t>(),
                                    static_cast<uint32_t>(batch.rows()), gk.as<float>(), losses.as<double>() + k,
                                    ws.as<void>(), flags.as<uint32_t>(), ctx.stream()),
                   "simulate");
      check_status(ds_grad_accumulate(gsum.as<double>(), gk.as<float>(), P, ctx.stream()), "simulate");
    }
    check_status(ds_grad_average(gavg.as<float>(), gsum.as<double>(), P, n, wd, dm.as<float>(), ctx.stream()), "simulate");
    check_status(ds_sgd_update(dm.as<float>(), dm.as<float>(), gavg.as<float>(), P, static_cast<float>(cfg.hyper.eta), 0.0f,
                               flags.as<uint32_t>(), ctx.stream()),
                 "simulate");
    uint32_t fl = 0;
    ctx.download(hl.data(), losses.as<void>(), n * sizeof(double));
    ctx.download(&fl, flags.as<void>(), sizeof(uint32_t));
    ctx.sync();
    if (fl & DS_FLAG_LOSS_NONFINITE) throw NumericError("loss_and_grad: non-finite loss");
    if (fl & DS_FLAG_GRAD_NONFINITE) throw NumericError("loss_and_grad: non-finite gradient");
    if (fl & DS_FLAG_X_NONFINITE) throw ContractError("sgd_step: x contains a non-finite value");
    if (fl & DS_FLAG_G_NONFINITE) throw ContractError("sgd_step: grad contains a non-finite value");
    if (fl & DS_FLAG_OUT_NONFINITE) throw NumericError("sgd_step: non-finite result");
    for (uint32_t k = 0; k < n; ++k) {
      TrainRecord rec;
      rec.iter = r;
      rec.wall_ms = std::llround(t);
      rec.batch_loss = hl[k];
      rec.cumulated_loss = 0.0;
      rec.exchanged = true;
      rec.period_len = 1;
      res.worker_logs[k].push_back(rec);
    }
    if (cfg.record_master_snaps) {
      ParamVector snap(P);
      ctx.download(snap.data(), dm.as<void>(), P * sizeof(float));
      ctx.sync();
      res.master_snaps.push_back({t, 0, std::move(snap)});
    }
    while (next_eval <= r) {
      res.eval_curve.push_back({t, next_eval, eval.accuracy_of(dm.as<float>())});
      next_eval += cfg.eval_every;
    }
  }
  if (res.eval_curve.back().per_worker_iter != cfg.hyper.i_max)
    res.eval_curve.push_back({t, cfg.hyper.i_max, eval.accuracy_of(dm.as<float>())});
  ParamVector master(P);
  ctx.download(master.data(), dm.as<void>(), P * sizeof(float));
  ctx.sync();
  res.worker_final_params.assign(n, master);
  res.final_master = std::move(master);
  res.virtual_clock_total = t;
  res.iterations_per_worker = cfg.hyper.i_max;
  return res;
}

}  // namespace

uint64_t sim_sweep_seed(const SimConfig& cfg, uint32_t worker) {
  return mix_seed(mix_seed(cfg.data_seed, kSweepTag), cfg.replicate_shards ? 0 : worker);
}
uint64_t sim_partition_seed(const SimConfig& cfg) { return mix_seed(cfg.data_seed, kPartTag); }
uint64_t sim_holdout_seed(const SimConfig& cfg) { return mix_seed(cfg.data_seed, kHoldTag); }

void SimConfig::validate() const {
  if (n_workers < 1) throw ContractError("sim: n_workers must be >= 1");
  if (!(batch_cost_C > 0.0)) throw ContractError("sim: batch_cost_C must be positive");
  if (!(comm_cost_S >= 0.0)) throw ContractError("sim: comm_cost_S must be nonnegative");
  if (eval_every < 1) throw ContractError("sim: eval_every must be >= 1");
  if (!(holdout_frac > 0.0 && holdout_frac < 1.0)) throw ContractError("sim: holdout_frac must be in (0,1)");
  if (!cost_multipliers.empty()) {
    if (cost_multipliers.size() != n_workers) throw ContractError("sim: cost_multipliers must have one entry per worker");
    for (double m : cost_multipliers)
      if (!(m > 0.0)) throw ContractError("sim: cost multipliers must be positive");
  }
  model.validate();
  dataset.validate();
  if (dataset.n_features != model.n_features || dataset.n_classes > model.n_classes)
    throw ContractError("sim: dataset dimensions do not fit the model");
}

SimResult simulate(const SimConfig& cfg) {
  cfg.validate();
  auto [train, holdout] = split_holdout(cfg.dataset, cfg.holdout_frac, sim_holdout_seed(cfg));
  std::vector<Dataset> owned;
  std::vector<const Dataset*> shards(cfg.n_workers);
  if (cfg.replicate_shards) {
    for (auto& s : shards) s = &train;
  } else {
    owned = partition(train, cfg.n_workers, sim_partition_seed(cfg));
    for (uint32_t k = 0; k < cfg.n_workers; ++k) shards[k] = &owned[k];
  }
  ParamVector master = init_params(cfg.model, cfg.init_seed);
  return cfg.mode == SimMode::AsyncEASGD ? simulate_async(cfg, shards, holdout, std::move(master))
                                         : simulate_sync(cfg, shards, holdout, std::move(master));
}

std::vector<ExchangeEvent> exchange_order(const SimConfig& cfg) {
  if (cfg.n_workers < 1) throw ContractError("sim: n_workers must be >= 1");
  if (cfg.hyper.period_mode != PeriodMode::Fixed || cfg.hyper.tau == 0)
    throw ContractError("exchange_order: needs a Fixed period (adaptive order is value-dependent)");
  if (!cfg.cost_multipliers.empty() && cfg.cost_multipliers.size() != cfg.n_workers)
    throw ContractError("sim: cost_multipliers must have one entry per worker");
  const uint32_t n = cfg.n_workers;
  Rng sched(cfg.schedule_seed);
  std::priority_queue<Event, std::vector<Event>, std::greater<Event>> pq;
  std::vector<uint64_t> done(n, 0);
  for (uint32_t k = 0; k < n; ++k) pq.push({cfg.batch_cost_C * mult(cfg, k), sched.next_u64(), k});
  std::vector<ExchangeEvent> out;
  while (!pq.empty()) {
    const Event ev = pq.top();
    pq.pop();
    const uint32_t k = ev.worker;
    const uint64_t it = ++done[k];
    double next_t = ev.t + cfg.batch_cost_C * mult(cfg, k);
    if (it % cfg.hyper.tau == 0) {  // ExchangePolicy Fixed: since == tau, reset on fire
      out.push_back({k, it, ev.t});
      next_t += cfg.comm_cost_S;
    }
    if (it < cfg.hyper.i_max) pq.push({next_t, sched.next_u64(), k});
  }
  return out;
}

std::optional<uint64_t> iterations_to_accuracy(const SimResult& result, double target) {
  for (const EvalPoint& p : result.eval_curve)
    if (p.accuracy >= target) return p.per_worker_iter;
  return std::nullopt;
}

double estimate_d(const SimResult& async_result, uint64_t baseline_N, double target) {
  if (baseline_N == 0) throw ContractError("estimate_d: baseline_N must be positive");
  const auto iters = iterations_to_accuracy(async_result, target);
  if (!iters) throw ContractError("estimate_d: run never reached the target accuracy");
  return static_cast<double>(async_result.n_workers) * static_cast<double>(*iters) / static_cast<double>(baseline_N);
}

}  // namespace deepspark
