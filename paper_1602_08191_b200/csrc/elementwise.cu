// elementwise.cu — the memory-bound update kernels of the EASGD hot path.
//
//   elastic update   (param_vector.hpp:34-38, param_vector.cpp:41-57, exchanger.cpp:76-92)
//   SGD + L2 fold    (param_vector.cpp:21-39, engine.cpp:75-79)
//
// Both stream their operands exactly once: 16 B/element (elastic: read w, read m,
// write w', write m') and 12 B/element (SGD: read x, read g, write x'). They are
// HBM-bound on B200: 128-bit vector loads/stores with evict-first hints, 4 independent
// 16-byte loads per operand in flight per thread, grid sized to 8 CTAs per SM.
// The _rn intrinsics keep the reference's f32 rounding points (no FFMA contraction).
#include "ds_common.cuh"
#include "elementwise.cuh"

namespace dsb {

namespace {

constexpr int kThreads = 256;
constexpr int kUnroll = 4;

__device__ __forceinline__ float4 ld_cs(const float4* p) { return __ldcs(p); }
__device__ __forceinline__ void st_cs(float4* p, const float4& v) { __stcs(p, v); }

__device__ __forceinline__ void elastic4(const float4& w, const float4& m, float a, float4& wo,
                                         float4& mo) {
  elastic_elem(w.x, m.x, a, wo.x, mo.x);
  elastic_elem(w.y, m.y, a, wo.y, mo.y);
  elastic_elem(w.z, m.z, a, wo.z, mo.z);
  elastic_elem(w.w, m.w, a, wo.w, mo.w);
}

// w_out may alias w_in (in-place update): every element is loaded before it is stored
// by the same thread and no two threads touch the same element.
__global__ void __launch_bounds__(kThreads) elastic_vec_kernel(const float* w_in, float* w_out,
                                                               float* __restrict__ m, uint64_t n,
                                                               float a) {
  const uint64_t n4 = n >> 2;
  const float4* w4 = reinterpret_cast<const float4*>(w_in);
  float4* o4 = reinterpret_cast<float4*>(w_out);
  float4* m4 = reinterpret_cast<float4*>(m);
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kThreads;
  uint64_t i = static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x;
  for (; i + (kUnroll - 1) * stride < n4; i += kUnroll * stride) {
    float4 wv[kUnroll], mv[kUnroll];
#pragma unroll
    for (int j = 0; j < kUnroll; ++j) {
      wv[j] = ld_cs(w4 + i + j * stride);
      mv[j] = ld_cs(m4 + i + j * stride);
    }
#pragma unroll
    for (int j = 0; j < kUnroll; ++j) {
      float4 wo, mo;
      elastic4(wv[j], mv[j], a, wo, mo);
      st_cs(o4 + i + j * stride, wo);
      st_cs(m4 + i + j * stride, mo);
    }
  }
  for (; i < n4; i += stride) {
    float4 wo, mo;
    elastic4(ld_cs(w4 + i), ld_cs(m4 + i), a, wo, mo);
    st_cs(o4 + i, wo);
    st_cs(m4 + i, mo);
  }
  // scalar tail (n % 4 elements)
  const uint64_t t = (n4 << 2) + static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x;
  if (t < n) {
    float wo, mo;
    elastic_elem(w_in[t], m[t], a, wo, mo);
    w_out[t] = wo;
    m[t] = mo;
  }
}

__global__ void __launch_bounds__(kThreads) elastic_scalar_kernel(const float* w_in, float* w_out,
                                                                  float* m, uint64_t n, float a) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kThreads;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x; i < n; i += stride) {
    float wo, mo;
    elastic_elem(w_in[i], m[i], a, wo, mo);
    w_out[i] = wo;
    m[i] = mo;
  }
}

__device__ __forceinline__ float sgd_elem(float x, float g, float eta, float wd, uint32_t& bad) {
  if (!finite_f(x)) bad |= DS_FLAG_X_NONFINITE;
  if (wd > 0.0f) g = fadd(g, fmul(wd, x));  // engine.cpp:75-78: grad += f32(wd) * x
  if (!finite_f(g)) bad |= DS_FLAG_G_NONFINITE;
  const float o = fsub(x, fmul(eta, g));  // param_vector.cpp:33: x - eta_f * grad
  if (!finite_f(o)) bad |= DS_FLAG_OUT_NONFINITE;
  return o;
}

__device__ __forceinline__ void flush_flags(uint32_t bad, uint32_t* flags) {
  // warp-aggregated: one atomic per warp that saw anything
  const uint32_t any = __reduce_or_sync(0xffffffffu, bad);
  if (any && flags && (threadIdx.x & 31) == 0) atomicOr(flags, any);
}

__global__ void __launch_bounds__(kThreads) sgd_vec_kernel(float* out, const float* x,
                                                           const float* __restrict__ g, uint64_t n,
                                                           float eta, float wd, uint32_t* flags,
                                                           const uint32_t* gate) {
  if (gate && *gate) return;
  const uint64_t n4 = n >> 2;
  const float4* x4 = reinterpret_cast<const float4*>(x);
  const float4* g4 = reinterpret_cast<const float4*>(g);
  float4* o4 = reinterpret_cast<float4*>(out);
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kThreads;
  uint32_t bad = 0;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x; i < n4; i += stride) {
    const float4 xv = ld_cs(x4 + i), gv = ld_cs(g4 + i);
    float4 o;
    o.x = sgd_elem(xv.x, gv.x, eta, wd, bad);
    o.y = sgd_elem(xv.y, gv.y, eta, wd, bad);
    o.z = sgd_elem(xv.z, gv.z, eta, wd, bad);
    o.w = sgd_elem(xv.w, gv.w, eta, wd, bad);
    st_cs(o4 + i, o);
  }
  const uint64_t t = (n4 << 2) + static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x;
  if (t < n) out[t] = sgd_elem(x[t], g[t], eta, wd, bad);
  flush_flags(bad, flags);
}

__global__ void __launch_bounds__(kThreads) sgd_scalar_kernel(float* out, const float* x,
                                                              const float* g, uint64_t n, float eta,
                                                              float wd, uint32_t* flags,
                                                              const uint32_t* gate) {
  if (gate && *gate) return;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kThreads;
  uint32_t bad = 0;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x; i < n; i += stride)
    out[i] = sgd_elem(x[i], g[i], eta, wd, bad);
  flush_flags(bad, flags);
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

unsigned grid_for(uint64_t vec_items, int device_sms) {
  const uint64_t want = (vec_items + kThreads * kUnroll - 1) / (kThreads * kUnroll);
  const uint64_t cap = static_cast<uint64_t>(device_sms) * 8;  // 8 x 256 threads per SM
  uint64_t g = want < cap ? want : cap;
  return static_cast<unsigned>(g == 0 ? 1 : g);
}

int current_sms() {
  int dev = 0;
  cudaGetDevice(&dev);
  return sm_count(dev);
}

}  // namespace

int launch_elastic(const float* w_in, float* w_out, float* m, uint64_t n, float alpha,
                   cudaStream_t s) {
  if (n == 0) return DS_OK;
  const int sms = current_sms();
  if (aligned16(w_in) && aligned16(w_out) && aligned16(m)) {
    elastic_vec_kernel<<<grid_for(n >> 2, sms), kThreads, 0, s>>>(w_in, w_out, m, n, alpha);
  } else {
    elastic_scalar_kernel<<<grid_for(n, sms), kThreads, 0, s>>>(w_in, w_out, m, n, alpha);
  }
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

int launch_sgd(float* out, const float* x, const float* g, uint64_t n, float eta, float wd,
               uint32_t* flags, cudaStream_t s, const uint32_t* gate) {
  if (n == 0) return DS_OK;
  const int sms = current_sms();
  if (aligned16(out) && aligned16(x) && aligned16(g)) {
    sgd_vec_kernel<<<grid_for(n >> 2, sms), kThreads, 0, s>>>(out, x, g, n, eta, wd, flags, gate);
  } else {
    sgd_scalar_kernel<<<grid_for(n, sms), kThreads, 0, s>>>(out, x, g, n, eta, wd, flags, gate);
  }
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

// Momentum SGD (SURVEY §8 a21 — NOT IN THE REFERENCE, whose Hyperparams has no mu):
// g' = g + f32(wd)*x; v = mu*v + g'; out = x - eta*v, f32 with separate roundings.
// mu == 0 gives v = g' and out = x - eta*g', i.e. exactly sgd_step (param_vector.cpp:33).
__global__ void __launch_bounds__(kThreads) momentum_kernel(float* out, const float* x, float* v,
                                                            const float* __restrict__ g, uint64_t n, float eta,
                                                            float mu, float wd, uint32_t* flags,
                                                            const uint32_t* gate) {
  if (gate && *gate) return;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * kThreads;
  uint32_t bad = 0;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * kThreads + threadIdx.x; i < n; i += stride) {
    const float xi = x[i];
    float gi = g[i];
    if (!finite_f(xi)) bad |= DS_FLAG_X_NONFINITE;
    if (wd > 0.0f) gi = fadd(gi, fmul(wd, xi));
    if (!finite_f(gi)) bad |= DS_FLAG_G_NONFINITE;
    const float vi = mu != 0.0f ? fadd(fmul(mu, v[i]), gi) : gi;
    v[i] = vi;
    const float o = fsub(xi, fmul(eta, vi));
    if (!finite_f(o)) bad |= DS_FLAG_OUT_NONFINITE;
    out[i] = o;
  }
  flush_flags(bad, flags);
}

int launch_momentum(float* out, const float* x, float* v, const float* g, uint64_t n, float eta, float mu, float wd,
                    uint32_t* flags, cudaStream_t s, const uint32_t* gate) {
  if (n == 0) return DS_OK;
  momentum_kernel<<<grid_for(n, current_sms()), kThreads, 0, s>>>(out, x, v, g, n, eta, mu, wd, flags, gate);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

}  // namespace dsb

// ------------------------------------------------------------------------------------
// C-ABI
// ------------------------------------------------------------------------------------
extern "C" int ds_elastic_update(float* w, float* m, uint64_t n, float alpha, void* stream) {
  if (n && (!w || !m)) return dsb::set_error(DS_E_CONTRACT, "elastic_update: null pointer");
  return dsb::launch_elastic(w, w, m, n, alpha, dsb::as_stream(stream));
}

extern "C" int ds_elastic_exchange(const float* worker, float* master, float* out, uint64_t n,
                                   float alpha, void* stream) {
  if (n && (!worker || !master || !out))
    return dsb::set_error(DS_E_CONTRACT, "elastic_exchange: null pointer");
  return dsb::launch_elastic(worker, out, master, n, alpha, dsb::as_stream(stream));
}

extern "C" int ds_sgd_update(float* out, const float* x, const float* g, uint64_t n, float eta,
                             float wd, uint32_t* flags_dev, void* stream) {
  if (n && (!out || !x || !g)) return dsb::set_error(DS_E_CONTRACT, "sgd_update: null pointer");
  return dsb::launch_sgd(out, x, g, n, eta, wd, flags_dev, dsb::as_stream(stream));
}

extern "C" int ds_sgd_step_checked(float* out, const float* x, const float* g, uint64_t n,
                                   double eta, void* stream) {
  // param_vector.cpp:21-39, in the reference's check order
  if (!(eta > 0.0)) return dsb::set_error(DS_E_CONTRACT, "sgd_step: eta must be positive");
  uint32_t* flags = nullptr;
  cudaStream_t s = dsb::as_stream(stream);
  DS_CUDA_TRY(cudaMallocAsync(&flags, sizeof(uint32_t), s));
  DS_CUDA_TRY(cudaMemsetAsync(flags, 0, sizeof(uint32_t), s));
  int rc = dsb::launch_sgd(out, x, g, n, static_cast<float>(eta), 0.0f, flags, s);
  uint32_t h = 0;
  if (rc == DS_OK) {
    cudaMemcpyAsync(&h, flags, sizeof(uint32_t), cudaMemcpyDeviceToHost, s);
    cudaError_t e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) rc = dsb::set_error(DS_E_CUDA, "sgd_step: %s", cudaGetErrorString(e));
  }
  cudaFreeAsync(flags, s);
  if (rc != DS_OK) return rc;
  if (h & DS_FLAG_X_NONFINITE) return dsb::set_error(DS_E_CONTRACT, "sgd_step: x contains a non-finite value");
  if (h & DS_FLAG_G_NONFINITE) return dsb::set_error(DS_E_CONTRACT, "sgd_step: grad contains a non-finite value");
  if (h & DS_FLAG_OUT_NONFINITE) return dsb::set_error(DS_E_NUMERIC, "sgd_step: non-finite result");
  return DS_OK;
}

// ------------------------------------------------------------------------------------
// Synchronous SGD helpers (simulator.cpp:192-209)
// ------------------------------------------------------------------------------------
namespace {

__global__ void __launch_bounds__(256) grad_accumulate_kernel(double* __restrict__ gsum, const float* __restrict__ g,
                                                              uint64_t n) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * 256;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * 256 + threadIdx.x; i < n; i += stride)
    gsum[i] = __dadd_rn(gsum[i], static_cast<double>(g[i]));
}

__global__ void __launch_bounds__(256) grad_average_kernel(float* __restrict__ out, const double* __restrict__ gsum,
                                                           uint64_t n, double nw, float wd, const float* __restrict__ x) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * 256;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * 256 + threadIdx.x; i < n; i += stride) {
    float v = static_cast<float>(__ddiv_rn(gsum[i], nw));
    if (wd > 0.0f) v = __fadd_rn(v, __fmul_rn(wd, x[i]));
    out[i] = v;
  }
}

// gather_batch (model.cpp:12-21) on the device: one warp per row, float4 when aligned.
__global__ void __launch_bounds__(256) gather_rows_kernel(float* __restrict__ dst, uint32_t* __restrict__ y_dst,
                                                          const float* __restrict__ X, const uint32_t* __restrict__ y,
                                                          const uint32_t* __restrict__ idx, uint32_t rows,
                                                          uint32_t F, bool vec) {
  const uint32_t warp = (blockIdx.x * 256 + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (warp >= rows) return;
  const uint32_t src = idx[warp];
  if (lane == 0 && y_dst) y_dst[warp] = y[src];
  const float* s = X + static_cast<uint64_t>(src) * F;
  float* d = dst + static_cast<uint64_t>(warp) * F;
  if (vec) {
    for (uint32_t q = lane; q < F / 4; q += 32)
      reinterpret_cast<float4*>(d)[q] = __ldg(reinterpret_cast<const float4*>(s) + q);
  } else {
    for (uint32_t i = lane; i < F; i += 32) d[i] = __ldg(s + i);
  }
}

unsigned grid_n(uint64_t n) {
  int dev = 0;
  cudaGetDevice(&dev);
  const uint64_t want = (n + 255) / 256, cap = static_cast<uint64_t>(dsb::sm_count(dev)) * 8;
  return static_cast<unsigned>(want < 1 ? 1 : (want < cap ? want : cap));
}

}  // namespace

extern "C" int ds_grad_accumulate(double* gsum, const float* g, uint64_t n, void* stream) {
  if (n == 0) return DS_OK;
  if (!gsum || !g) return dsb::set_error(DS_E_CONTRACT, "grad_accumulate: null");
  grad_accumulate_kernel<<<grid_n(n), 256, 0, dsb::as_stream(stream)>>>(gsum, g, n);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

extern "C" int ds_grad_average(float* out, const double* gsum, uint64_t n, uint32_t n_workers, float wd,
                               const float* x, void* stream) {
  if (n == 0) return DS_OK;
  if (!out || !gsum || n_workers == 0 || (wd > 0.0f && !x))
    return dsb::set_error(DS_E_CONTRACT, "grad_average: bad arguments");
  grad_average_kernel<<<grid_n(n), 256, 0, dsb::as_stream(stream)>>>(out, gsum, n, static_cast<double>(n_workers),
                                                                    wd, x);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

extern "C" int ds_gather_rows(float* dst, uint32_t* y_dst, const float* X, const uint32_t* y, const uint32_t* idx,
                              uint32_t rows, uint32_t features, void* stream) {
  if (rows == 0) return DS_OK;
  if (!dst || !X || !idx || features == 0 || (y_dst && !y)) return dsb::set_error(DS_E_CONTRACT, "gather_rows: bad arguments");
  const bool vec = (features % 4) == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(dst) & 15) == 0;
  gather_rows_kernel<<<(rows + 7) / 8, 256, 0, dsb::as_stream(stream)>>>(dst, y_dst, X, y, idx, rows, features, vec);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

extern "C" int ds_sgd_momentum_update(float* out, const float* x, float* velocity, const float* g, uint64_t n,
                                      float eta, float mu, float wd, uint32_t* flags_dev, void* stream) {
  if (n && (!out || !x || !velocity || !g)) return dsb::set_error(DS_E_CONTRACT, "sgd_momentum: null pointer");
  if (!(eta > 0.0f)) return dsb::set_error(DS_E_CONTRACT, "sgd_step: eta must be positive");
  if (!(mu >= 0.0f && mu < 1.0f)) return dsb::set_error(DS_E_CONTRACT, "sgd_momentum: mu must be in [0,1)");
  return dsb::launch_momentum(out, x, velocity, g, n, eta, mu, wd, flags_dev, dsb::as_stream(stream), nullptr);
}

void dsb::warm_elementwise_kernels() {
  dsb::load_kernels(dsb::elastic_vec_kernel, dsb::elastic_scalar_kernel, dsb::sgd_vec_kernel, dsb::sgd_scalar_kernel,
                    dsb::momentum_kernel, grad_accumulate_kernel, grad_average_kernel, gather_rows_kernel);
}
