// model.cu — layer-wise f64 forward/backward of the built-in classifiers, any depth.
//
// Restates sample_loss_grad / loss_and_grad / loss_only / predict (model.cpp:185-318)
// with the reference's exact per-element operation order: every output of a dot product
// is one thread's sequential sum (bias first, then i = 0..in-1, one rounding per
// multiply and per add — the reference binary has no FMA), and every gradient element
// is one thread's sequential sum over the batch rows r = 0..R-1. Only the libm
// transcendental calls (tanh/exp/log) come from CUDA's double-precision library instead
// of glibc; everything else is bit-reproducible.
//
// This is the general path (softmax regression and MLPs of any depth). The fused
// single-kernel step in mlp_fused.cu covers <= 1 hidden layer at much lower latency.
#include <cmath>

#include "ds_common.cuh"
#include "model.cuh"

namespace dsb {

int model_from_desc(const ds_model_desc* d, ModelInfo& out) {
  if (!d) return set_error(DS_E_CONTRACT, "model: null descriptor");
  if (d->kind == DS_MODEL_CIFAR10_QUICK) {  // NOT IN REFERENCE (convnet.cu)
    if (d->n_features != 3072) return set_error(DS_E_CONTRACT, "model: cifar10_quick takes 3072 features");
    if (d->n_classes < 2) return set_error(DS_E_CONTRACT, "model: n_classes must be at least 2");
    if (d->n_hidden != 0) return set_error(DS_E_CONTRACT, "model: cifar10_quick has no hidden list");
    out = ModelInfo{};
    out.kind = d->kind;
    out.n_features = 3072;
    out.n_classes = d->n_classes;
    const uint32_t fan[5] = {75, 800, 800, 1024, 64}, width[5] = {32, 32, 64, 64, d->n_classes};
    uint64_t off = 0;
    for (int l = 0; l < 5; ++l) {
      LayerInfo L;
      L.w_off = off;
      off += static_cast<uint64_t>(width[l]) * fan[l];
      L.b_off = off;
      off += width[l];
      L.in_dim = fan[l];
      L.out_dim = width[l];
      out.layers.push_back(L);
    }
    out.P = off;
    out.max_out = 64;
    out.sum_out = 0;
    return DS_OK;
  }
  if (d->kind == DS_MODEL_ALEXNET) {  // NOT IN REFERENCE (alexnet.cu); layout as oracle/ds_oracle_alex.c
    uint32_t S = 0;
    while (3ull * (S + 1) * (S + 1) <= d->n_features) ++S;
    if (3ull * S * S != d->n_features || S < 55)
      return set_error(DS_E_CONTRACT, "model: alexnet takes 3*S*S features, S >= 55");
    if (d->n_classes < 2) return set_error(DS_E_CONTRACT, "model: n_classes must be at least 2");
    if (d->n_hidden != 0) return set_error(DS_E_CONTRACT, "model: alexnet has no hidden list");
    out = ModelInfo{};
    out.kind = d->kind;
    out.n_features = d->n_features;
    out.n_classes = d->n_classes;
    out.alex_side = S;
    const uint32_t H1 = (S - 11) / 4 + 1, P1 = (H1 - 2) / 2 + 1, P2 = (P1 - 2) / 2 + 1, P5 = (P2 - 2) / 2 + 1;
    const uint32_t fan[8] = {363, 1200, 2304, 1728, 1728, 256 * P5 * P5, 4096, 4096};
    const uint32_t width[8] = {96, 256, 384, 384, 256, 4096, 4096, d->n_classes};
    uint64_t off = 0;
    for (int l = 0; l < 8; ++l) {
      LayerInfo L;
      L.w_off = off;
      off += static_cast<uint64_t>(width[l]) * fan[l];
      L.b_off = off;
      off += width[l];
      L.in_dim = fan[l];
      L.out_dim = width[l];
      out.layers.push_back(L);
    }
    out.P = off;
    out.max_out = 4096;
    return DS_OK;
  }
  if (d->kind != 0 && d->kind != 1) return set_error(DS_E_CONTRACT, "model: unknown kind %d", d->kind);
  if (d->n_features == 0) return set_error(DS_E_CONTRACT, "model: n_features must be positive");
  if (d->n_classes < 2) return set_error(DS_E_CONTRACT, "model: n_classes must be at least 2");
  if (d->kind == 0 && d->n_hidden != 0)
    return set_error(DS_E_CONTRACT, "model: softmax regression has no hidden layers");
  if (d->kind == 1 && d->n_hidden == 0)
    return set_error(DS_E_CONTRACT, "model: mlp needs at least one hidden layer");
  out = ModelInfo{};
  out.kind = d->kind;
  out.n_features = d->n_features;
  out.n_classes = d->n_classes;
  for (uint32_t i = 0; i < d->n_hidden; ++i) {
    if (d->hidden[i] == 0) return set_error(DS_E_CONTRACT, "model: hidden sizes must be positive");
    out.hidden.push_back(d->hidden[i]);
  }
  uint64_t off = 0;
  uint32_t in = d->n_features;
  for (size_t li = 0; li <= out.hidden.size(); ++li) {
    const uint32_t o = li < out.hidden.size() ? out.hidden[li] : d->n_classes;
    LayerInfo L;
    L.w_off = off;
    off += static_cast<uint64_t>(o) * in;
    L.b_off = off;
    off += o;
    L.in_dim = in;
    L.out_dim = o;
    out.layers.push_back(L);
    out.max_out = o > out.max_out ? o : out.max_out;
    out.sum_out += o;
    in = o;
  }
  out.P = off;
  return DS_OK;
}

uint64_t layered_workspace_doubles(const ModelInfo& m, uint32_t R) {
  if (m.kind == DS_MODEL_CIFAR10_QUICK) return (cnn_workspace_bytes(m, R) + 7) / 8;
  if (m.kind == DS_MODEL_ALEXNET) return (alex_workspace_bytes(m, R) + 7) / 8;
  // activations A_1..A_L, two delta buffers, per-row loss
  return static_cast<uint64_t>(R) * (m.sum_out + 2ull * m.max_out + 1);
}

namespace {

constexpr int kT = 128;

__device__ __forceinline__ bool gated(const uint32_t* gate) { return gate && *gate; }

// Dense forward for one layer: out[r,o] = act(b[o] + sum_i W[o,i]*a[r,i]).
// Input is either f32 rows of X (optionally gathered through idx) or f64 activations.
template <bool kInF32>
__global__ void __launch_bounds__(kT) fwd_layer(const float* __restrict__ W, const float* __restrict__ b,
                                                const float* __restrict__ X, const uint32_t* __restrict__ idx,
                                                const double* __restrict__ Ain, uint32_t R, uint32_t in,
                                                uint32_t out_dim, bool hidden, double* __restrict__ Aout,
                                                const uint32_t* gate) {
  if (gated(gate)) return;
  const uint32_t o = blockIdx.x * kT + threadIdx.x;
  const uint32_t r = blockIdx.y;
  if (o >= out_dim || r >= R) return;
  const float* w = W + static_cast<uint64_t>(o) * in;
  double z = static_cast<double>(b[o]);
  if constexpr (kInF32) {
    const uint64_t row = idx ? idx[r] : r;
    const float* x = X + row * in;
    for (uint32_t i = 0; i < in; ++i) z = dadd(z, dmul(static_cast<double>(w[i]), static_cast<double>(x[i])));
  } else {
    const double* a = Ain + static_cast<uint64_t>(r) * in;
    for (uint32_t i = 0; i < in; ++i) z = dadd(z, dmul(static_cast<double>(w[i]), a[i]));
  }
  Aout[static_cast<uint64_t>(r) * out_dim + o] = hidden ? tanh(z) : z;
}

// Max-shifted softmax cross-entropy per row; delta = softmax - onehot (model.cpp:202-214).
__global__ void __launch_bounds__(kT) softmax_ce(const double* __restrict__ Z, const uint32_t* __restrict__ y,
                                                 const uint32_t* __restrict__ idx, uint32_t R, uint32_t C,
                                                 double* __restrict__ delta, double* __restrict__ loss_rows,
                                                 uint32_t* flags, const uint32_t* gate) {
  if (gated(gate)) return;
  const uint32_t r = blockIdx.x * kT + threadIdx.x;
  if (r >= R) return;
  const uint32_t label = y[idx ? idx[r] : r];
  if (label >= C) {
    atomicOr(flags, DS_FLAG_LABEL_RANGE);
    loss_rows[r] = 0.0;
    return;
  }
  const double* z = Z + static_cast<uint64_t>(r) * C;
  double zmax = z[0];
  for (uint32_t c = 1; c < C; ++c) zmax = z[c] > zmax ? z[c] : zmax;
  double sum = 0.0;
  for (uint32_t c = 0; c < C; ++c) sum = dadd(sum, exp(dsub(z[c], zmax)));
  const double lse = dadd(zmax, log(sum));
  loss_rows[r] = dsub(lse, z[label]);
  if (delta) {
    double* d = delta + static_cast<uint64_t>(r) * C;
    for (uint32_t c = 0; c < C; ++c) d[c] = dsub(exp(dsub(z[c], lse)), c == label ? 1.0 : 0.0);
  }
}

// loss = (sum_r loss_r) * (1/R) for loss_and_grad (model.cpp:253-255); / R for loss_only
// (model.cpp:272). The sum is sequential in r, as the reference's.
__global__ void loss_reduce(const double* __restrict__ loss_rows, uint32_t R, bool grad_mode,
                            double* loss_out, uint32_t* flags, const uint32_t* gate) {
  if (gated(gate)) return;
  double s = 0.0;
  for (uint32_t r = 0; r < R; ++r) s = dadd(s, loss_rows[r]);
  const double loss = grad_mode ? dmul(s, 1.0 / static_cast<double>(R)) : s / static_cast<double>(R);
  *loss_out = loss;
  if (!isfinite(loss)) atomicOr(flags, DS_FLAG_LOSS_NONFINITE);
}

// delta_prev[r,i] = (sum_o delta[r,o] * W[o,i]) * (1 - a[r,i]^2)   (model.cpp:225-233)
__global__ void __launch_bounds__(kT) bwd_delta(const double* __restrict__ delta, const float* __restrict__ W,
                                                const double* __restrict__ A, uint32_t R, uint32_t n_in,
                                                uint32_t n_out, double* __restrict__ prev, const uint32_t* gate) {
  if (gated(gate)) return;
  const uint32_t i = blockIdx.x * kT + threadIdx.x;
  const uint32_t r = blockIdx.y;
  if (i >= n_in || r >= R) return;
  const double* d = delta + static_cast<uint64_t>(r) * n_out;
  double p = 0.0;
  for (uint32_t o = 0; o < n_out; ++o) p = dadd(p, dmul(d[o], static_cast<double>(W[static_cast<uint64_t>(o) * n_in + i])));
  const double a = A[static_cast<uint64_t>(r) * n_in + i];
  prev[static_cast<uint64_t>(r) * n_in + i] = dmul(p, dsub(1.0, dmul(a, a)));
}

// grad W[o,i] = f32((sum_r delta[r,o] * a[r,i]) * (1/R)), grad b[o] likewise with a = 1
// (model.cpp:216-221 accumulation, 256-261 scaling and rounding).
template <bool kInF32>
__global__ void __launch_bounds__(kT) grad_layer(const double* __restrict__ delta, const float* __restrict__ X,
                                                 const uint32_t* __restrict__ idx, const double* __restrict__ Ain,
                                                 uint32_t R, uint32_t in, uint32_t out_dim, double inv_b,
                                                 float* __restrict__ gW, float* __restrict__ gb,
                                                 uint32_t* flags, const uint32_t* gate) {
  if (gated(gate)) return;
  const uint32_t i = blockIdx.x * kT + threadIdx.x;  // input index, or == in for the bias
  const uint32_t o = blockIdx.y;
  if (i > in || o >= out_dim) return;
  double acc = 0.0;
  if (i == in) {
    for (uint32_t r = 0; r < R; ++r) acc = dadd(acc, delta[static_cast<uint64_t>(r) * out_dim + o]);
  } else if constexpr (kInF32) {
    for (uint32_t r = 0; r < R; ++r) {
      const uint64_t row = idx ? idx[r] : r;
      acc = dadd(acc, dmul(delta[static_cast<uint64_t>(r) * out_dim + o], static_cast<double>(X[row * in + i])));
    }
  } else {
    for (uint32_t r = 0; r < R; ++r)
      acc = dadd(acc, dmul(delta[static_cast<uint64_t>(r) * out_dim + o], Ain[static_cast<uint64_t>(r) * in + i]));
  }
  const double g = dmul(acc, inv_b);
  if (!isfinite(g)) atomicOr(flags, DS_FLAG_GRAD_NONFINITE);
  if (i == in) gb[o] = static_cast<float>(g);
  else gW[static_cast<uint64_t>(o) * in + i] = static_cast<float>(g);
}

// argmax with first-max-wins (std::max_element, model.cpp:317) and hit counting.
__global__ void __launch_bounds__(kT) argmax_hits(const double* __restrict__ Z, const uint32_t* __restrict__ y,
                                                  uint32_t R, uint32_t C, unsigned long long* hits,
                                                  uint32_t* pred) {
  const uint32_t r = blockIdx.x * kT + threadIdx.x;
  uint32_t hit = 0;
  if (r < R) {
    const double* z = Z + static_cast<uint64_t>(r) * C;
    uint32_t best = 0;
    for (uint32_t c = 1; c < C; ++c)
      if (z[c] > z[best]) best = c;
    if (pred) pred[r] = best;
    hit = (y && y[r] == best) ? 1u : 0u;
  }
  const unsigned n = __reduce_add_sync(0xffffffffu, hit);
  if (hits && (threadIdx.x & 31) == 0 && n) atomicAdd(hits, static_cast<unsigned long long>(n));
}

struct WsView {
  std::vector<double*> act;  // A_1..A_L
  double* d0;
  double* d1;
  double* loss_rows;
};

WsView carve(const ModelInfo& m, uint32_t R, double* ws) {
  WsView v;
  double* p = ws;
  for (const auto& L : m.layers) {
    v.act.push_back(p);
    p += static_cast<uint64_t>(R) * L.out_dim;
  }
  v.d0 = p;
  p += static_cast<uint64_t>(R) * m.max_out;
  v.d1 = p;
  p += static_cast<uint64_t>(R) * m.max_out;
  v.loss_rows = p;
  return v;
}

int forward(const ModelInfo& m, const float* params, const float* X, const uint32_t* idx, uint32_t R,
            const WsView& v, const uint32_t* gate, cudaStream_t s) {
  const size_t nl = m.layers.size();
  for (size_t li = 0; li < nl; ++li) {
    const LayerInfo& L = m.layers[li];
    dim3 grid((L.out_dim + kT - 1) / kT, R);
    const bool hidden = li + 1 < nl;
    if (li == 0) {
      fwd_layer<true><<<grid, kT, 0, s>>>(params + L.w_off, params + L.b_off, X, idx, nullptr, R, L.in_dim,
                                          L.out_dim, hidden, v.act[0], gate);
    } else {
      fwd_layer<false><<<grid, kT, 0, s>>>(params + L.w_off, params + L.b_off, nullptr, nullptr, v.act[li - 1],
                                           R, L.in_dim, L.out_dim, hidden, v.act[li], gate);
    }
  }
  return DS_OK;
}

}  // namespace

int launch_loss_and_grad(const ModelInfo& m, const float* params, const float* X, const uint32_t* idx,
                         const uint32_t* y, uint32_t R, float* grad, double* loss_out, double* ws,
                         uint32_t* flags, const uint32_t* gate, cudaStream_t s) {
  if (R == 0) return set_error(DS_E_CONTRACT, "loss_and_grad: empty batch");
  if (R > 65535) return set_error(DS_E_CONTRACT, "loss_and_grad: at most 65535 rows per call");
  if (m.kind == DS_MODEL_CIFAR10_QUICK)
    return launch_cnn_loss_and_grad(m, params, X, idx, y, R, grad, loss_out, ws, flags, gate, s);
  if (m.kind == DS_MODEL_ALEXNET)
    return launch_alex_loss_and_grad(m, params, X, idx, y, R, grad, loss_out, ws, flags, gate, s);
  const WsView v = carve(m, R, ws);
  forward(m, params, X, idx, R, v, gate, s);
  const size_t nl = m.layers.size();
  const uint32_t C = m.n_classes;
  softmax_ce<<<(R + kT - 1) / kT, kT, 0, s>>>(v.act[nl - 1], y, idx, R, C, grad ? v.d0 : nullptr,
                                              v.loss_rows, flags, gate);
  loss_reduce<<<1, 1, 0, s>>>(v.loss_rows, R, grad != nullptr, loss_out, flags, gate);
  if (grad) {
    const double inv_b = 1.0 / static_cast<double>(R);
    double* cur = v.d0;
    double* nxt = v.d1;
    for (size_t li = nl; li-- > 0;) {
      const LayerInfo& L = m.layers[li];
      dim3 g((L.in_dim + 1 + kT - 1) / kT, L.out_dim);
      if (li == 0) {
        grad_layer<true><<<g, kT, 0, s>>>(cur, X, idx, nullptr, R, L.in_dim, L.out_dim, inv_b, grad + L.w_off,
                                          grad + L.b_off, flags, gate);
      } else {
        grad_layer<false><<<g, kT, 0, s>>>(cur, nullptr, nullptr, v.act[li - 1], R, L.in_dim, L.out_dim, inv_b,
                                           grad + L.w_off, grad + L.b_off, flags, gate);
        dim3 gd((L.in_dim + kT - 1) / kT, R);
        bwd_delta<<<gd, kT, 0, s>>>(cur, params + L.w_off, v.act[li - 1], R, L.in_dim, L.out_dim, nxt, gate);
        double* t = cur;
        cur = nxt;
        nxt = t;
      }
    }
  }
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

int launch_count_hits(const ModelInfo& m, const float* params, const float* X, const uint32_t* y, uint32_t R,
                      double* ws, unsigned long long* hits, uint32_t* pred, cudaStream_t s) {
  if (R == 0) return DS_OK;
  if (m.kind == DS_MODEL_CIFAR10_QUICK) return launch_cnn_count_hits(m, params, X, y, R, ws, hits, pred, s);
  if (m.kind == DS_MODEL_ALEXNET) return launch_alex_count_hits(m, params, X, y, R, ws, hits, pred, s);
  const WsView v = carve(m, R, ws);
  forward(m, params, X, nullptr, R, v, nullptr, s);
  argmax_hits<<<(R + kT - 1) / kT, kT, 0, s>>>(v.act[m.layers.size() - 1], y, R, m.n_classes, hits, pred);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

}  // namespace dsb

// ------------------------------------------------------------------------------------
// C-ABI
// ------------------------------------------------------------------------------------
extern "C" int ds_param_dim(const ds_model_desc* model, uint64_t* dim) {
  dsb::ModelInfo m;
  DS_TRY(dsb::model_from_desc(model, m));
  *dim = m.P;
  return DS_OK;
}

extern "C" int ds_loss_and_grad_workspace(const ds_model_desc* model, uint32_t rows, uint64_t* bytes) {
  dsb::ModelInfo m;
  DS_TRY(dsb::model_from_desc(model, m));
  *bytes = dsb::layered_workspace_doubles(m, rows) * sizeof(double);
  return DS_OK;
}

extern "C" int ds_loss_and_grad(const ds_model_desc* model, const float* params, const float* X,
                                const uint32_t* y, uint32_t rows, float* grad, double* loss_out,
                                void* workspace, uint32_t* flags_dev, void* stream) {
  dsb::ModelInfo m;
  DS_TRY(dsb::model_from_desc(model, m));
  if (rows == 0) return dsb::set_error(DS_E_CONTRACT, "loss_and_grad: empty batch");
  if (!params || !X || !y || !loss_out || !workspace)
    return dsb::set_error(DS_E_CONTRACT, "loss_and_grad: null pointer");
  return dsb::launch_loss_and_grad(m, params, X, nullptr, y, rows, grad, loss_out,
                                   static_cast<double*>(workspace), flags_dev, nullptr,
                                   dsb::as_stream(stream));
}

extern "C" int ds_predict(const ds_model_desc* model, const float* params, const float* X, uint64_t rows,
                          uint32_t* pred_out, void* stream) {
  dsb::ModelInfo m;
  DS_TRY(dsb::model_from_desc(model, m));
  cudaStream_t s = dsb::as_stream(stream);
  const uint32_t chunk = m.kind == DS_MODEL_ALEXNET ? 128 : 4096;  // alexnet workspace grows ~25 MB per row
  double* ws = nullptr;
  DS_CUDA_TRY(cudaMallocAsync(&ws, dsb::layered_workspace_doubles(m, chunk) * sizeof(double), s));
  int rc = DS_OK;
  for (uint64_t r0 = 0; r0 < rows && rc == DS_OK; r0 += chunk) {
    const uint32_t R = static_cast<uint32_t>(rows - r0 < chunk ? rows - r0 : chunk);
    rc = dsb::launch_count_hits(m, params, X + r0 * m.n_features, nullptr, R, ws, nullptr, pred_out + r0, s);
  }
  cudaFreeAsync(ws, s);
  return rc;
}

extern "C" int ds_count_hits(const ds_model_desc* model, const float* params, const float* X, const uint32_t* y,
                             uint64_t rows, unsigned long long* hits_out, void* stream) {
  dsb::ModelInfo m;
  DS_TRY(dsb::model_from_desc(model, m));
  cudaStream_t s = dsb::as_stream(stream);
  const uint32_t chunk = m.kind == DS_MODEL_ALEXNET ? 128 : 4096;  // alexnet workspace grows ~25 MB per row
  double* ws = nullptr;
  DS_CUDA_TRY(cudaMallocAsync(&ws, dsb::layered_workspace_doubles(m, chunk) * sizeof(double), s));
  int rc = DS_OK;
  for (uint64_t r0 = 0; r0 < rows && rc == DS_OK; r0 += chunk) {
    const uint32_t R = static_cast<uint32_t>(rows - r0 < chunk ? rows - r0 : chunk);
    rc = dsb::launch_count_hits(m, params, X + r0 * m.n_features, y + r0, R, ws, hits_out, nullptr, s);
  }
  cudaFreeAsync(ws, s);
  return rc;
}

void dsb::warm_model_kernels() {
  dsb::load_kernels(dsb::fwd_layer<true>, dsb::fwd_layer<false>, dsb::softmax_ce, dsb::loss_reduce, dsb::bwd_delta,
                    dsb::grad_layer<true>, dsb::grad_layer<false>, dsb::argmax_hits);
}
