// Built-in models — structure and init on the host (reference model.cpp:12-159),
// loss/gradient/prediction on the GPU through ds_loss_and_grad / ds_count_hits /
// ds_predict (reference model.cpp:163-328 semantics and error behaviour).
#include "deepspark/model.hpp"

#include <algorithm>
#include <cmath>
#include <sstream>

#include "deepspark/errors.hpp"
#include "deepspark/rng.hpp"
#include "device_ctx.hpp"

namespace deepspark {

namespace {

detail::ModelDesc desc_of(const Model& m) {
  detail::ModelDesc md;
  md.hidden = m.hidden;
  md.d.kind = model_kind_code(m.kind);
  md.d.n_features = m.n_features;
  md.d.n_classes = m.n_classes;
  md.d.n_hidden = static_cast<uint32_t>(md.hidden.size());
  md.d.hidden = md.hidden.data();
  return md;
}

void check_inputs(const Model& model, std::span<const float> params, const Minibatch& batch) {
  if (params.size() != model.param_dim())
    throw ContractError("loss_and_grad: params dim " + std::to_string(params.size()) + " does not match model dim " +
                        std::to_string(model.param_dim()));
  if (batch.rows() == 0) throw ContractError("loss_and_grad: empty batch");
  if (batch.n_features != model.n_features)
    throw ContractError("loss_and_grad: batch has " + std::to_string(batch.n_features) + " features, model wants " +
                        std::to_string(model.n_features));
  if (batch.features.size() != batch.rows() * static_cast<size_t>(batch.n_features))
    throw ContractError("loss_and_grad: batch feature matrix shape mismatch");
  for (uint32_t y : batch.labels)
    if (y >= model.n_classes) throw ContractError("loss_and_grad: label " + std::to_string(y) + " out of range");
}

// One device evaluation; grad may be empty (loss_only).
double device_loss(const Model& model, std::span<const float> params, const Minibatch& batch, std::span<float> grad) {
  const auto md = desc_of(model);
  auto& ctx = detail::DeviceCtx::get();
  const size_t P = params.size(), R = batch.rows(), F = batch.n_features;
  uint64_t ws_bytes = 0;
  check_status(ds_loss_and_grad_workspace(&md.d, static_cast<uint32_t>(R), &ws_bytes), "loss_and_grad");
  auto* dp = static_cast<float*>(ctx.scratch(0, P * sizeof(float)));
  auto* dX = static_cast<float*>(ctx.scratch(1, R * F * sizeof(float)));
  auto* dy = static_cast<uint32_t*>(ctx.scratch(2, R * sizeof(uint32_t)));
  auto* dg = static_cast<float*>(ctx.scratch(3, P * sizeof(float)));
  auto* dws = ctx.scratch(4, ws_bytes);
  auto* dmisc = static_cast<char*>(ctx.scratch(5, 64));
  double* dloss = reinterpret_cast<double*>(dmisc);
  uint32_t* dflags = reinterpret_cast<uint32_t*>(dmisc + 16);
  ctx.upload(dp, params.data(), P * sizeof(float));
  ctx.upload(dX, batch.features.data(), R * F * sizeof(float));
  ctx.upload(dy, batch.labels.data(), R * sizeof(uint32_t));
  check_status(ds_memset(dflags, 0, sizeof(uint32_t), ctx.stream()), "loss_and_grad");
  check_status(ds_loss_and_grad(&md.d, dp, dX, dy, static_cast<uint32_t>(R), grad.empty() ? nullptr : dg, dloss, dws,
                                dflags, ctx.stream()),
               "loss_and_grad");
  double loss = 0.0;
  uint32_t flags = 0;
  ctx.download(&loss, dloss, sizeof(double));
  ctx.download(&flags, dflags, sizeof(uint32_t));
  if (!grad.empty()) ctx.download(grad.data(), dg, P * sizeof(float));
  ctx.sync();
  const char* who = grad.empty() ? "loss_only" : "loss_and_grad";
  if (flags & DS_FLAG_LABEL_RANGE) throw ContractError(std::string(who) + ": label out of range");
  if (flags & DS_FLAG_LOSS_NONFINITE) throw NumericError(std::string(who) + ": non-finite loss");
  if (flags & DS_FLAG_GRAD_NONFINITE) throw NumericError("loss_and_grad: non-finite gradient");
  return loss;
}

}  // namespace

void gather_batch(const Dataset& ds, std::span<const uint32_t> idx, Minibatch& out) {
  out.n_features = ds.n_features;
  out.labels.resize(idx.size());
  out.features.resize(idx.size() * ds.n_features);
  for (size_t i = 0; i < idx.size(); ++i) {
    out.labels[i] = ds.labels[idx[i]];
    const auto r = ds.row(idx[i]);
    std::copy(r.begin(), r.end(), out.features.begin() + i * ds.n_features);
  }
}

Model Model::softmax(uint32_t n_features, uint32_t n_classes) {
  Model m;
  m.kind = ModelKind::SoftmaxRegression;
  m.n_features = n_features;
  m.n_classes = n_classes;
  m.validate();
  return m;
}

Model Model::mlp(uint32_t n_features, std::vector<uint32_t> hidden, uint32_t n_classes) {
  Model m;
  m.kind = ModelKind::Mlp;
  m.n_features = n_features;
  m.n_classes = n_classes;
  m.hidden = std::move(hidden);
  m.validate();
  return m;
}

Model Model::cifar10_quick(uint32_t n_classes) {
  Model m;
  m.kind = ModelKind::Cifar10Quick;
  m.n_features = 3072;
  m.n_classes = n_classes;
  m.validate();
  return m;
}

Model Model::alexnet(uint32_t side, uint32_t n_classes) {
  Model m;
  m.kind = ModelKind::AlexNet;
  m.n_features = 3 * side * side;
  m.n_classes = n_classes;
  m.validate();
  return m;
}

namespace {
uint32_t alex_side(uint32_t n_features) {  // S with 3*S*S == n_features and S >= 55, else 0
  uint32_t s = 0;
  while (3ull * (s + 1) * (s + 1) <= n_features) ++s;
  return (3ull * s * s == n_features && s >= 55) ? s : 0;
}
}  // namespace

void Model::validate() const {
  if (kind == ModelKind::AlexNet) {
    if (!alex_side(n_features)) throw ContractError("model: alexnet takes 3*S*S features, S >= 55");
    if (n_classes < 2) throw ContractError("model: n_classes must be at least 2");
    if (!hidden.empty()) throw ContractError("model: alexnet has no hidden list");
    return;
  }
  if (kind == ModelKind::Cifar10Quick) {
    if (n_features != 3072) throw ContractError("model: cifar10_quick takes 3072 features");
    if (n_classes < 2) throw ContractError("model: n_classes must be at least 2");
    if (!hidden.empty()) throw ContractError("model: cifar10_quick has no hidden list");
    return;
  }
  if (n_features == 0) throw ContractError("model: n_features must be positive");
  if (n_classes < 2) throw ContractError("model: n_classes must be at least 2");
  if (kind == ModelKind::SoftmaxRegression && !hidden.empty())
    throw ContractError("model: softmax regression has no hidden layers");
  if (kind == ModelKind::Mlp && hidden.empty()) throw ContractError("model: mlp needs at least one hidden layer");
  if (std::find(hidden.begin(), hidden.end(), 0u) != hidden.end())
    throw ContractError("model: hidden sizes must be positive");
}

Model Model::parse(const std::string& text) {
  std::vector<std::string> parts;
  {
    std::stringstream ss(text);
    std::string p;
    while (std::getline(ss, p, ':')) parts.push_back(p);
  }
  auto positive = [&](const std::string& s) -> uint32_t {
    size_t used = 0;
    unsigned long v = 0;
    try {
      v = std::stoul(s, &used);
    } catch (const std::exception&) {
      used = std::string::npos;
    }
    if (used != s.size() || v == 0 || v > UINT32_MAX) throw ContractError("model: bad integer '" + s + "' in '" + text + "'");
    return static_cast<uint32_t>(v);
  };
  if (parts.size() == 3 && parts[0] == "softmax") return softmax(positive(parts[1]), positive(parts[2]));
  if (parts.size() == 3 && parts[0] == "cifar10_quick") {
    if (positive(parts[1]) != 3072) throw ContractError("model: cifar10_quick takes 3072 features");
    return cifar10_quick(positive(parts[2]));
  }
  if (parts.size() == 3 && parts[0] == "alexnet") {
    const uint32_t s = alex_side(positive(parts[1]));
    if (!s) throw ContractError("model: alexnet takes 3*S*S features, S >= 55");
    return alexnet(s, positive(parts[2]));
  }
  if (parts.size() == 4 && parts[0] == "mlp") {
    std::vector<uint32_t> hidden;
    std::stringstream hs(parts[2]);
    std::string h;
    while (std::getline(hs, h, ',')) hidden.push_back(positive(h));
    if (hidden.empty()) throw ContractError("model: empty hidden list in '" + text + "'");
    return mlp(positive(parts[1]), std::move(hidden), positive(parts[3]));
  }
  throw ContractError("model: cannot parse '" + text +
                      "' (want softmax:<features>:<classes> or mlp:<features>:<h1,...>:<classes>)");
}

std::string Model::to_string() const {
  std::ostringstream os;
  if (kind == ModelKind::SoftmaxRegression) {
    os << "softmax:" << n_features << ':' << n_classes;
    return os.str();
  }
  if (kind == ModelKind::Cifar10Quick) {
    os << "cifar10_quick:" << n_features << ':' << n_classes;
    return os.str();
  }
  if (kind == ModelKind::AlexNet) {
    os << "alexnet:" << n_features << ':' << n_classes;
    return os.str();
  }
  os << "mlp:" << n_features << ':';
  for (size_t i = 0; i < hidden.size(); ++i) os << (i ? "," : "") << hidden[i];
  os << ':' << n_classes;
  return os.str();
}

std::vector<Model::Layer> Model::layers() const {
  std::vector<Layer> out;
  if (kind == ModelKind::AlexNet) {  // conv1..5 (fan_in = Cin/g * k * k), fc6..8 (oracle/ds_oracle_alex.h)
    const uint32_t S = alex_side(n_features), H1 = (S - 11) / 4 + 1, P1 = (H1 - 2) / 2 + 1, P2 = (P1 - 2) / 2 + 1,
                   P5 = (P2 - 2) / 2 + 1;
    const uint32_t fan[8] = {363, 1200, 2304, 1728, 1728, 256 * P5 * P5, 4096, 4096};
    const uint32_t width[8] = {96, 256, 384, 384, 256, 4096, 4096, n_classes};
    size_t off = 0;
    for (int l = 0; l < 8; ++l) {
      Layer L{off, off + static_cast<size_t>(width[l]) * fan[l], fan[l], width[l]};
      off = L.b_off + width[l];
      out.push_back(L);
    }
    return out;
  }
  if (kind == ModelKind::Cifar10Quick) {  // conv1..3 (fan_in = Cin*25), ip1, ip2
    const uint32_t fan[5] = {75, 800, 800, 1024, 64}, width[5] = {32, 32, 64, 64, n_classes};
    size_t off = 0;
    for (int l = 0; l < 5; ++l) {
      Layer L{off, off + static_cast<size_t>(width[l]) * fan[l], fan[l], width[l]};
      off = L.b_off + width[l];
      out.push_back(L);
    }
    return out;
  }
  size_t off = 0;
  uint32_t in = n_features;
  std::vector<uint32_t> widths = hidden;
  widths.push_back(n_classes);
  for (uint32_t width : widths) {
    Layer l{off, off + static_cast<size_t>(width) * in, in, width};
    off = l.b_off + width;
    out.push_back(l);
    in = width;
  }
  return out;
}

size_t Model::param_dim() const {
  const auto ls = layers();
  return ls.back().b_off + ls.back().out_dim;
}

uint64_t Model::fingerprint() const {
  uint64_t h = 0xcbf29ce484222325ULL;  // FNV-1a offset basis
  auto mix = [&h](uint64_t v, int nbytes) {
    for (int i = 0; i < nbytes; ++i) {
      h ^= (v >> (8 * i)) & 0xffu;
      h *= 0x100000001b3ULL;  // FNV prime
    }
  };
  mix(static_cast<uint64_t>(model_kind_code(kind)) + 1, 1);
  mix(n_features, 4);
  mix(n_classes, 4);
  mix(hidden.size(), 4);
  for (uint32_t w : hidden) mix(w, 4);
  return h;
}

ParamVector init_params(const Model& model, uint64_t seed) {
  model.validate();
  Rng rng(mix_seed(seed, 0x1e17));
  ParamVector params(model.param_dim());
  for (const Model::Layer& l : model.layers()) {
    const double bound = 1.0 / std::sqrt(static_cast<double>(l.in_dim));
    const size_t count = static_cast<size_t>(l.out_dim) * l.in_dim + l.out_dim;  // weights then biases
    for (size_t i = 0; i < count; ++i) params[l.w_off + i] = static_cast<float>(rng.uniform(-bound, bound));
  }
  return params;
}

double loss_and_grad(const Model& model, std::span<const float> params, const Minibatch& batch,
                     std::span<float> grad_out) {
  check_inputs(model, params, batch);
  if (grad_out.size() != params.size()) throw ContractError("loss_and_grad: grad buffer dim mismatch");
  return device_loss(model, params, batch, grad_out);
}

double loss_only(const Model& model, std::span<const float> params, const Minibatch& batch) {
  check_inputs(model, params, batch);
  return device_loss(model, params, batch, {});
}

double grad_check(const Model& model, const ParamVector& params, const Minibatch& batch, double h) {
  if (!(h >= 1e-6 && h <= 1e-2)) throw ContractError("grad_check: h must lie in [1e-6, 1e-2]");
  ParamVector grad(params.size());
  loss_and_grad(model, params, batch, grad);
  ParamVector probe = params;
  double worst = 0.0;
  for (size_t i = 0; i < params.size(); ++i) {
    const float orig = probe[i];
    const float up = static_cast<float>(static_cast<double>(orig) + h);
    const float dn = static_cast<float>(static_cast<double>(orig) - h);
    probe[i] = up;
    const double lp = loss_only(model, probe, batch);
    probe[i] = dn;
    const double lm = loss_only(model, probe, batch);
    probe[i] = orig;
    const double fd = (lp - lm) / (static_cast<double>(up) - static_cast<double>(dn));
    const double a = static_cast<double>(grad[i]);
    worst = std::max(worst, std::abs(a - fd) / (std::abs(a) + std::abs(fd) + 1e-12));
  }
  return worst;
}

uint32_t predict(const Model& model, std::span<const float> params, std::span<const float> row) {
  if (params.size() != model.param_dim()) throw ContractError("predict: params dim mismatch");
  if (row.size() != model.n_features) throw ContractError("predict: row width mismatch");
  const auto md = desc_of(model);
  auto& ctx = detail::DeviceCtx::get();
  auto* dp = static_cast<float*>(ctx.scratch(0, params.size() * sizeof(float)));
  auto* dX = static_cast<float*>(ctx.scratch(1, row.size() * sizeof(float)));
  auto* dout = static_cast<uint32_t*>(ctx.scratch(2, sizeof(uint32_t)));
  ctx.upload(dp, params.data(), params.size() * sizeof(float));
  ctx.upload(dX, row.data(), row.size() * sizeof(float));
  check_status(ds_predict(&md.d, dp, dX, 1, dout, ctx.stream()), "predict");
  uint32_t out = 0;
  ctx.download(&out, dout, sizeof(uint32_t));
  ctx.sync();
  return out;
}

double accuracy(const Model& model, std::span<const float> params, const Dataset& ds) {
  ds.validate();
  if (params.size() != model.param_dim()) throw ContractError("accuracy: params dim mismatch");
  const auto md = desc_of(model);
  auto& ctx = detail::DeviceCtx::get();
  const size_t n = ds.size(), F = ds.n_features;
  auto* dp = static_cast<float*>(ctx.scratch(0, params.size() * sizeof(float)));
  auto* dX = static_cast<float*>(ctx.scratch(1, n * F * sizeof(float)));
  auto* dy = static_cast<uint32_t*>(ctx.scratch(2, n * sizeof(uint32_t)));
  auto* dh = static_cast<unsigned long long*>(ctx.scratch(5, 64));
  ctx.upload(dp, params.data(), params.size() * sizeof(float));
  ctx.upload(dX, ds.features.data(), n * F * sizeof(float));
  ctx.upload(dy, ds.labels.data(), n * sizeof(uint32_t));
  check_status(ds_memset(dh, 0, sizeof(unsigned long long), ctx.stream()), "accuracy");
  check_status(ds_count_hits(&md.d, dp, dX, dy, n, dh, ctx.stream()), "accuracy");
  unsigned long long hits = 0;
  ctx.download(&hits, dh, sizeof(hits));
  ctx.sync();
  return static_cast<double>(hits) / static_cast<double>(n);
}

}  // namespace deepspark
