// ds_common.cuh — shared host/device helpers for the B200 EASGD hot path (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdio>
#include <initializer_list>
#include <string>

#include "ds_cuda.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ < 1000)
#error "paper_1602_08191_b200 targets sm_100a (B200) only"
#endif

namespace dsb {

// ---------------------------------------------------------------------------------
// Error state (thread-local, surfaced by ds_last_error)
// ---------------------------------------------------------------------------------
std::string& last_error();
int set_error(int code, const char* fmt, ...);

#define DS_CUDA_TRY(expr)                                                              \
  do {                                                                                 \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess) {                                                           \
      return ::dsb::set_error(e_ == cudaErrorMemoryAllocation ? DS_E_NOMEM : DS_E_CUDA, \
                              "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_),  \
                              __FILE__, __LINE__);                                     \
    }                                                                                  \
  } while (0)

#define DS_TRY(expr)           \
  do {                         \
    int rc_ = (expr);          \
    if (rc_ != DS_OK) return rc_; \
  } while (0)

// Guard that makes `device` current for the scope and restores the previous one.
struct DeviceScope {
  int prev = -1;
  explicit DeviceScope(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceScope() {
    int now = -1;
    cudaGetDevice(&now);
    if (prev >= 0 && now != prev) cudaSetDevice(prev);
  }
};

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int sm_count(int device);

// Loads kernels now (CUDA lazy loading otherwise loads each on its first launch, which
// lands inside the caller's first timed step): cudaFuncGetAttributes forces the load.
template <typename... K>
inline void load_kernels(K... k) {
  cudaFuncAttributes a;
  (void)std::initializer_list<int>{(cudaFuncGetAttributes(&a, reinterpret_cast<const void*>(k)), 0)...};
  cudaGetLastError();
}
// Per-file warmers (engine / master creation call the ones their paths launch).
void warm_model_kernels();
void warm_elementwise_kernels();
void warm_fused_kernels();
void warm_tc_kernels();
void warm_master_kernels();

// ---------------------------------------------------------------------------------
// Device arithmetic with the reference's rounding points. The reference is compiled
// for x86-64 without FMA (no -march), so every multiply and add rounds separately;
// nvcc would otherwise contract a*b+c into one FFMA/DFMA. The _rn intrinsics are never
// contracted.
// ---------------------------------------------------------------------------------
__device__ __forceinline__ float fmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float fadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float fsub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }

// elastic_update_elem (param_vector.hpp:34-38): e = a*(w-m); w' = w-e; m' = m+e.
__device__ __forceinline__ void elastic_elem(float w, float m, float a, float& w_out,
                                             float& m_out) {
  const float e = fmul(a, fsub(w, m));
  w_out = fsub(w, e);
  m_out = fadd(m, e);
}

__device__ __forceinline__ bool finite_f(float v) { return isfinite(v); }

// System-scope acquire/release on 64-bit words (peer-mapped flags over NVLink).
__device__ __forceinline__ uint64_t ld_acquire_sys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long atom_add_sys(unsigned long long* p,
                                                           unsigned long long v) {
  return atomicAdd_system(p, v);
}
__device__ __forceinline__ void nanosleep_ns(unsigned ns) { __nanosleep(ns); }

// Bounded acquire-wait until *p == want. Returns false after kSeqTimeoutNs: a peer that
// stopped early (non-finite step) or died never advances the word, so the waiter raises
// an error flag instead of hanging every GPU of the group.
constexpr unsigned long long kSeqTimeoutNs = 30ull * 1000 * 1000 * 1000;
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ bool wait_seq_eq(const uint64_t* p, uint64_t want, unsigned sleep_ns) {
  if (ld_acquire_sys(p) == want) return true;
  const unsigned long long t0 = globaltimer_ns();
  while (ld_acquire_sys(p) != want) {
    if (globaltimer_ns() - t0 > kSeqTimeoutNs) return false;
    __nanosleep(sleep_ns);
  }
  return true;
}

}  // namespace dsb
