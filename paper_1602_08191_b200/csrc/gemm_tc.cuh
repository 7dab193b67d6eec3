// gemm_tc.cuh — TMA + tcgen05 tf32 GEMM (gemm_tc.cu).
//
// D = epi(scale * A . B^T): A and B are K-major row-major f32 tensors in HBM (rows x cols,
// leading dimension ld: a multiple of 4, base 16-byte aligned). Three addressing modes:
//   plain      A [M x K], B [N x K]; split-K over K (`splits` slabs reduced in order).
//   taps       implicit GEMM: the K loop runs over `n` taps, each contributing `kt` columns
//              read at per-tap (row, col) offsets of A and B. A convolution over a spatially
//              zero-padded NHWC map is this mode with one tap per filter position: the tap's
//              A row offset is the pixel shift, so no im2col matrix is ever written. Row
//              coordinates may run outside the tensor: TMA zero-fills them.
//   taps/per_z one output block per tap (grid z = tap x split): the weight gradient of such a
//              convolution, K = pixels, tap t writes D columns [t*d_col_step, ...).
// Optional epilogue row map: the M rows index a padded grid (Hp x Hp per image, border
// `pad`); border rows are skipped and interior rows land at the unpadded (H x H) or the
// same padded index of D.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace dsb {

constexpr int kMaxTaps = 25;

struct GemmTaps {
  int32_t n = 0;            // 0: plain GEMM
  int32_t per_z = 0;        // 1: tap = blockIdx.z / splits, separate outputs; 0: taps accumulate
  uint32_t kt = 0;          // accumulate mode: K columns per tap (multiple of 8)
  uint32_t d_col_step = 0;  // per_z: D column offset per tap
  int32_t a_row[kMaxTaps], a_col[kMaxTaps], b_row[kMaxTaps], b_col[kMaxTaps];
  int32_t halo_lo = 0;      // internal (halo mode): first A row of the halo relative to m0
  uint32_t halo_rows = 0;   // internal: rows per halo load (0 = per-tap A loads)
  uint32_t tpc = 1;         // internal (per_z): taps per CTA, their B tiles stacked along N
  uint32_t n_tap = 0;       // internal (per_z, tpc > 1): N columns per tap
};

struct GemmEpilogue {
  float* D = nullptr;
  uint64_t ldd = 0;
  uint64_t split_stride = 0;      // internal: split-K slab stride
  float scale = 1.f;
  const float* bias_n = nullptr;  // per output column
  const float* bias_m = nullptr;  // per output row
  bool relu = false;
  const float* mask = nullptr;    // x = mask[out_row * ldm + col] > 0 ? x : 0 (ReLU backward)
  uint64_t ldm = 0;
  const uint32_t* gate = nullptr; // nonzero: the launch does nothing (a failed step froze the engine)
  bool raw = false;               // internal: store the bare accumulator (split slabs)
  uint32_t map_Hp = 0, map_pad = 0, map_H = 0;  // row map (map_Hp == 0: identity)
  bool map_out_padded = false;
};

struct GemmOperand {
  const float* p = nullptr;
  uint64_t rows = 0, cols = 0, ld = 0;
};

// splits > 1 (plain or per_z): raw partial slabs go to `part` (splits * M * N floats per
// tap) and are summed in split order (deterministic) by a reduce kernel that applies the
// epilogue. DS_GEMM_3XTF32=1 (diagnostics) runs every product as three tf32 GEMMs on
// hi/lo operand splits: f32-accurate.
int launch_gemm(const GemmOperand& A, const GemmOperand& B, uint32_t M, uint32_t N, uint32_t K, const GemmTaps* taps,
                const GemmEpilogue& ep, uint32_t splits, float* part, cudaStream_t s);
// plain mode shorthand: A [M x K] (lda), B [N x K] (ldb)
int launch_gemm_tf32(const float* A, uint64_t lda, const float* B, uint64_t ldb, uint32_t M, uint32_t N, uint32_t K,
                     const GemmEpilogue& ep, uint32_t splits, float* part, cudaStream_t s);
uint32_t gemm_pick_bn(uint32_t N);
uint32_t gemm_ctas_per_sm(uint32_t bn);

}  // namespace dsb
