// conv_tc.cuh — tcgen05 (5th-generation tensor core) building blocks for the convnet:
// canonical K-major no-swizzle shared-memory descriptors, the kind::tf32 instruction
// descriptor, single-thread MMA issue with mbarrier commit, TMEM allocation and the
// 32-lane x 32-column accumulator load. Encodings follow CUTLASS's UMMA::SmemDescriptor /
// UMMA::InstrDescriptor (cute/arch/mma_sm100_desc.hpp); tools/tc_gemm_test.cu checks them
// against a CPU GEMM.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace dsb {
namespace tc {

__device__ __forceinline__ uint32_t saddr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

// Canonical K-major, no swizzle: a "core matrix" is 8 rows x 16 bytes (4 tf32). The
// element (row, k) of a [rows x K] operand lives at byte
//   (k / 4) * lbo + (row / 8) * 128 + (row % 8) * 16 + (k % 4) * 4,   lbo = rows / 8 * 128.
__device__ __forceinline__ uint32_t kmajor_off(uint32_t row, uint32_t k, uint32_t rows) {
  return (k >> 2) * (rows >> 3) * 128 + (row >> 3) * 128 + (row & 7) * 16 + (k & 3) * 4;
}

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((addr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= 1ull << 46;  // descriptor version 1 (sm_100); base offset 0; layout SWIZZLE_NONE
  return d;
}

// kind::tf32, f32 accumulate, both operands K-major
__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(m >> 4) << 24);
}

// D[tmem] (+)= A[rows=128 x K=8] * B[rows=n x K=8]^T for one 8-deep K step. a_addr/b_addr
// point at the step's first core-matrix column (k = 8t), lbo = rows/8 * 128.
__device__ __forceinline__ void mma_tf32(uint32_t tmem, uint32_t a_addr, uint32_t a_lbo, uint32_t b_addr,
                                         uint32_t b_lbo, uint32_t idesc, bool accumulate) {
  const uint64_t da = sdesc(a_addr, a_lbo, 128), db = sdesc(b_addr, b_lbo, 128);
  const uint32_t acc = accumulate ? 1u : 0u;
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void commit(uint64_t* mbar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(mbar))
               : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\nWAIT_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra WAIT_%=;\n\t}" ::"r"(
          saddr(b)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

template <uint32_t kCols>
__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem) {  // one full warp
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(saddr(dst_smem)),
               "n"(kCols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
template <uint32_t kCols>
__device__ __forceinline__ void tmem_free(uint32_t tmem) {  // the allocating warp
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(kCols));
}

// D[tmem] (+)= A[tmem: 128 lanes x 8 columns] * B[smem, rows=n x K=8]^T
__device__ __forceinline__ void mma_tf32_ta(uint32_t tmem_d, uint32_t tmem_a, uint32_t b_addr, uint32_t b_lbo,
                                            uint32_t idesc, bool accumulate) {
  const uint64_t db = sdesc(b_addr, b_lbo, 128);
  const uint32_t acc = accumulate ? 1u : 0u;
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(tmem_d),
      "r"(tmem_a), "l"(db), "r"(idesc), "r"(acc));
}

// this warp's 32 TMEM lanes x 32 consecutive columns <- v[0..31] (one row per thread),
// complete (tcgen05.wait::st) on return
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])),
      "r"(__float_as_uint(v[15])), "r"(__float_as_uint(v[16])), "r"(__float_as_uint(v[17])),
      "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])), "r"(__float_as_uint(v[20])),
      "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])), "r"(__float_as_uint(v[23])),
      "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])), "r"(__float_as_uint(v[26])),
      "r"(__float_as_uint(v[27])), "r"(__float_as_uint(v[28])), "r"(__float_as_uint(v[29])),
      "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31]))
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// 32 consecutive accumulator columns of this warp's 32 TMEM lanes into v[0..31]
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

}  // namespace tc

// conv_tc.cu: 5x5 pad-2 convolution (forward, or backward-data with flipped/transposed
// weights) as a tcgen05 implicit GEMM; instantiated for the convnet's layer shapes. Wpk:
// scratch of conv5_tc_wpk_floats(CIN, COUT) floats for the packed weight chunks.
// flip: W is the forward weight of the layer being back-propagated ([COUT][CIN] swapped),
// packed as its transposed, rotated kernel.
template <int CIN, int COUT, int H>
int launch_conv5_tc(const float* in, const float* W, bool flip, float* Wpk, const float* b, float* out, uint32_t R,
                    bool relu, const uint32_t* gate, cudaStream_t s);
// conv_tc.cu: weight and bias gradients of a 5x5 pad-2 convolution as a tcgen05 GEMM over
// the batch's pixels; part: scratch of conv5_wgrad_part_floats floats.
template <int CIN, int COUT, int H, int SPS>
int launch_conv5_wgrad_tc(const float* in, const float* dout, float* part, float* gW, float* gb, uint32_t R,
                          float inv_b, uint32_t* flags, const uint32_t* gate, cudaStream_t s);
inline constexpr uint64_t conv5_wgrad_part_floats(uint32_t cin, uint32_t cout, uint32_t R, uint32_t sps) {
  return static_cast<uint64_t>((R + sps - 1) / sps) * (cin * 25 + 1) * cout;
}
inline constexpr uint32_t conv5_tc_wpk_floats(uint32_t cin, uint32_t cout) { return (cin * 25 + 31) / 32 * 32 * cout; }

}  // namespace dsb
