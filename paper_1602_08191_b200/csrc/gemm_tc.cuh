// gemm_tc.cuh — TMA + tcgen05 tf32 GEMM (gemm_tc.cu): D = epi(scale * A . B^T), both
// operands K-major row-major f32 (A [M x K] leading dimension lda, B [N x K] ldb; lda and
// ldb multiples of 4, bases 16-byte aligned).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace dsb {

struct GemmEpilogue {
  float* D = nullptr;
  uint64_t ldd = 0;
  uint64_t split_stride = 0;   // set internally for split-K slabs
  float scale = 1.f;
  const float* bias_n = nullptr;  // per output column
  const float* bias_m = nullptr;  // per output row
  bool relu = false;
  const float* mask = nullptr;    // x = mask[row * ldm + col] > 0 ? x : 0 (ReLU backward)
  uint64_t ldm = 0;
  const uint32_t* gate = nullptr; // nonzero: the launch does nothing (a failed step froze the engine)
  bool raw = false;               // internal: store the bare accumulator (split slabs)
};

// splits > 1: K is cut into `splits` ranges whose raw partials go to `part`
// (splits * M * N floats) and are summed in split order (deterministic) by a reduce
// kernel that applies the epilogue. DS_GEMM_3XTF32=1 (diagnostics) runs every product as
// three tf32 GEMMs on hi/lo operand splits, f32-accurate.
int launch_gemm_tf32(const float* A, uint64_t lda, const float* B, uint64_t ldb, uint32_t M, uint32_t N, uint32_t K,
                     const GemmEpilogue& ep, uint32_t splits, float* part, cudaStream_t s);
uint32_t gemm_pick_bn(uint32_t N);

}  // namespace dsb
