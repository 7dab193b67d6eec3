// elementwise.cuh — launchers for the memory-bound update kernels (elementwise.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace dsb {
// w_out may equal w_in. alpha is already f32 (param_vector.cpp:50 rounding).
int launch_elastic(const float* w_in, float* w_out, float* m, uint64_t n, float alpha,
                   cudaStream_t s);
// out may equal x; flags may be null; gate (may be null): skip when *gate != 0.
int launch_sgd(float* out, const float* x, const float* g, uint64_t n, float eta, float wd,
               uint32_t* flags, cudaStream_t s, const uint32_t* gate = nullptr);
int launch_momentum(float* out, const float* x, float* v, const float* g, uint64_t n, float eta, float mu, float wd,
                    uint32_t* flags, cudaStream_t s, const uint32_t* gate);
}  // namespace dsb
