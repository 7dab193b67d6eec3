// The worker loop — reference engine.cpp:10-113. ShardSweeper and ExchangePolicy are
// host objects with the reference's semantics (the simulator and reference-style
// callers use them directly); SgdEngine and run_training_loop drive the device engine
// (ds_engine_*), whose own sweep plan and policy reproduce the same order on the GPU.
#include "deepspark/engine.hpp"

#include <algorithm>
#include <chrono>
#include <numeric>

#include "deepspark/errors.hpp"
#include "deepspark/exchanger.hpp"
#include "device_ctx.hpp"

namespace deepspark {

ShardSweeper::ShardSweeper(const Dataset& shard, uint32_t batch_size, uint64_t seed)
    : shard_(&shard), batch_size_(batch_size), seed_(seed) {
  shard.validate();
  if (batch_size_ == 0) throw ContractError("sweeper: batch_size must be positive");
  order_.resize(shard.size());
  std::iota(order_.begin(), order_.end(), 0u);
  reshuffle();
}

void ShardSweeper::reshuffle() {
  Rng rng(mix_seed(seed_, epoch_));
  rng.shuffle(order_);
  pos_ = 0;
}

std::vector<uint32_t> ShardSweeper::next_indices() {
  if (pos_ >= order_.size()) {
    ++epoch_;
    reshuffle();
  }
  const size_t take = std::min<size_t>(batch_size_, order_.size() - pos_);
  std::vector<uint32_t> idx(order_.begin() + pos_, order_.begin() + pos_ + take);
  pos_ += take;
  return idx;
}

void ShardSweeper::next(Minibatch& out) {
  const std::vector<uint32_t> idx = next_indices();
  gather_batch(*shard_, idx, out);
}

ExchangePolicy::Decision ExchangePolicy::on_iteration(double batch_loss) {
  cumulated_ += batch_loss;
  ++since_exchange_;
  const bool fire = mode_ == PeriodMode::Fixed ? since_exchange_ == tau_ : should_exchange(cumulated_, loss_cut_);
  Decision d;
  if (fire) {
    d.exchange = true;
    d.period_len = since_exchange_;
    cumulated_ = 0.0;
    since_exchange_ = 0;
  }
  return d;
}

namespace {

ds_hyper to_ds(const Hyperparams& hp) {
  ds_hyper h{};
  h.eta = hp.eta;
  h.alpha = hp.alpha;
  h.tau = hp.tau;
  h.batch_size = hp.batch_size;
  h.i_max = hp.i_max;
  h.loss_cut = hp.loss_cut;
  h.weight_decay = hp.weight_decay;
  h.adaptive = hp.period_mode == PeriodMode::Adaptive ? 1 : 0;
  return h;
}

int engine_kind() {
  const char* env = std::getenv("DEEPSPARK_ENGINE");  // auto | layered | fused | tc
  if (!env) return DS_ENGINE_AUTO;
  const std::string v(env);
  if (v == "layered") return DS_ENGINE_LAYERED;
  if (v == "fused") return DS_ENGINE_FUSED;
  if (v == "tc") return DS_ENGINE_TC;  // the tensor-core step (stated tolerance, one hidden layer)
  return DS_ENGINE_AUTO;
}

}  // namespace

SgdEngine::SgdEngine(Model model, const Dataset& shard, const Hyperparams& hp, uint64_t sweep_seed, ParamVector initial)
    : model_(std::move(model)), shard_(&shard), hp_(hp) {
  hp_.validate();
  shard.validate();
  if (initial.size() != model_.param_dim()) throw ContractError("engine: initial params dim does not match model");
  if (shard.n_features != model_.n_features || shard.n_classes > model_.n_classes)
    throw ContractError("engine: shard dims do not match model");
  std::vector<uint32_t> hidden = model_.hidden;
  ds_model_desc d{model_kind_code(model_.kind), model_.n_features, model_.n_classes,
                  static_cast<uint32_t>(hidden.size()), hidden.data()};
  const ds_hyper h = to_ds(hp_);
  check_status(ds_engine_create(&h_, detail::default_device(), &d, shard.features.data(), shard.labels.data(),
                                shard.size(), shard.n_classes, &h, sweep_seed, initial.data(), engine_kind()),
               "SgdEngine");
  host_params_ = std::move(initial);
  host_valid_ = true;
}

SgdEngine::~SgdEngine() {
  if (h_) ds_engine_destroy(h_);
}

SgdEngine::SgdEngine(SgdEngine&& o) noexcept
    : model_(std::move(o.model_)),
      shard_(o.shard_),
      hp_(o.hp_),
      h_(o.h_),
      iter_(o.iter_),
      host_params_(std::move(o.host_params_)),
      host_valid_(o.host_valid_) {
  o.h_ = nullptr;
}

uint64_t SgdEngine::run(uint64_t steps, bool stop_at_exchange) {
  uint64_t ran = steps;
  check_status(ds_engine_run(h_, steps, stop_at_exchange ? 1 : 0, stop_at_exchange ? &ran : nullptr), "SgdEngine::run");
  iter_ += ran;
  host_valid_ = false;
  return ran;
}

void SgdEngine::sync() { check_status(ds_engine_sync(h_), "SgdEngine"); }

double SgdEngine::step() {
  run(1, false);
  sync();
  double loss = 0.0;
  check_status(ds_engine_log(h_, iter_ - 1, 1, &loss, nullptr, nullptr, nullptr), "SgdEngine::step");
  return loss;
}

const ParamVector& SgdEngine::params() const {
  if (!host_valid_) {
    check_status(ds_engine_sync(h_), "SgdEngine::params");
    host_params_.resize(model_.param_dim());
    check_status(ds_engine_get_params(h_, host_params_.data()), "SgdEngine::params");
    host_valid_ = true;
  }
  return host_params_;
}

void SgdEngine::set_params(ParamVector p) {
  if (p.size() != model_.param_dim()) throw ContractError("engine: params dim change");
  check_status(ds_engine_set_params(h_, p.data()), "SgdEngine::set_params");
  host_params_ = std::move(p);
  host_valid_ = true;
}

void SgdEngine::attach_master(MasterState* master) {
  check_status(ds_engine_attach_master(h_, master ? master->handle() : nullptr), "SgdEngine::attach_master");
}

void SgdEngine::exchange_with(MasterState& master) {
  float* p = nullptr;
  void* stream = nullptr;
  check_status(ds_engine_params_device(h_, &p), "SgdEngine::exchange_with");
  check_status(ds_engine_stream(h_, &stream), "SgdEngine::exchange_with");
  master.exchange_device(p, p, stream);
  host_valid_ = false;
}

TrainLog SgdEngine::log(uint64_t first, uint64_t count) const {
  std::vector<double> loss(count), cum(count);
  std::vector<uint8_t> ex(count);
  std::vector<uint32_t> period(count);
  check_status(ds_engine_log(h_, first, count, loss.data(), cum.data(), ex.data(), period.data()), "SgdEngine::log");
  TrainLog out(count);
  for (uint64_t i = 0; i < count; ++i) {
    out[i].iter = first + i + 1;
    out[i].batch_loss = loss[i];
    out[i].cumulated_loss = cum[i];
    out[i].exchanged = ex[i] != 0;
    out[i].period_len = period[i];
  }
  return out;
}

LocalRunResult run_training_loop(const Model& model, const Dataset& shard, const Hyperparams& hp, uint64_t sweep_seed,
                                 ParamVector initial, const ExchangeFn& exchange) {
  hp.validate();
  SgdEngine engine(model, shard, hp, sweep_seed, std::move(initial));
  // the TrainLog rows and sweep plan are allocated before the clock starts (wall_ms
  // measures training, as the reference's host loop does)
  check_status(ds_engine_reserve(engine.handle(), std::min<uint64_t>(hp.i_max, 1u << 16)), "run_training_loop");
  const auto t0 = std::chrono::steady_clock::now();
  std::vector<int64_t> wall(hp.i_max, 0);
  uint64_t done = 0;
  auto stamp = [&](uint64_t upto) {
    const int64_t ms =
        std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - t0).count();
    for (uint64_t i = done; i < upto; ++i) wall[i] = ms;
  };
  if (!exchange) {
    engine.run(hp.i_max, false);  // the whole loop in one device run
    engine.sync();
    stamp(hp.i_max);
    done = hp.i_max;
  } else {
    while (done < hp.i_max) {
      const uint64_t ran = engine.run(hp.i_max - done, true);
      engine.sync();
      uint8_t fired = 0;
      check_status(ds_engine_log(engine.handle(), done + ran - 1, 1, nullptr, nullptr, &fired, nullptr), "loop");
      stamp(done + ran);
      done += ran;
      if (fired) engine.set_params(exchange(engine.params()));  // the ExchangeFn seam (engine.cpp:97-99)
    }
  }
  LocalRunResult out;
  out.log = engine.log(0, hp.i_max);
  for (uint64_t i = 0; i < hp.i_max; ++i) out.log[i].wall_ms = wall[i];
  out.final_params = engine.params();
  return out;
}

LocalRunResult run_training_loop(const Model& model, const Dataset& shard, const Hyperparams& hp, uint64_t sweep_seed,
                                 ParamVector initial, MasterState& master) {
  hp.validate();
  if (master.dim() != model.param_dim()) throw ContractError("run_training_loop: master dim does not match model");
  SgdEngine engine(model, shard, hp, sweep_seed, std::move(initial));
  engine.attach_master(&master);
  check_status(ds_engine_reserve(engine.handle(), std::min<uint64_t>(hp.i_max, 1u << 16)), "run_training_loop");
  const auto t0 = std::chrono::steady_clock::now();
  engine.run(hp.i_max, false);
  engine.sync();
  const int64_t ms = std::chrono::duration_cast<std::chrono::milliseconds>(std::chrono::steady_clock::now() - t0).count();
  LocalRunResult out;
  out.log = engine.log(0, hp.i_max);
  for (auto& r : out.log) r.wall_ms = ms;
  out.final_params = engine.params();
  engine.attach_master(nullptr);
  return out;
}

}  // namespace deepspark
