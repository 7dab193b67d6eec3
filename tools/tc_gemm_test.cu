// tc_gemm_test.cu — minimal tcgen05 (5th-gen tensor core) GEMM check, kind::tf32, both
// operands K-major in the canonical no-swizzle layout, accumulator in TMEM. Tool only:
// validates the descriptor encodings used by csrc/conv_tc.cu against a CPU product.
//   D[M x N] = A[M x K] * B[N x K]^T,  M = 128, N = 32, K = 64
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_runtime.h>

constexpr int M = 128, N = 32, K = 64;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// canonical K-major, no swizzle: core matrix = 8 rows x 16 bytes; (row, kchunk) at
// kchunk * (rows/8 * 128) + (row/8) * 128 + (row%8) * 16
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((addr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= 1ull << 46;  // version (Blackwell)
  // base_offset 0, lbo_mode 0, layout SWIZZLE_NONE (0) in bits 61..63
  return d;
}
__host__ __device__ constexpr uint32_t idesc_tf32(int m, int n) {
  return (1u << 4)                      // c_format F32
         | (2u << 7) | (2u << 10)       // a/b format TF32
         | (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(m >> 4) << 24);
}

template <int kAMN>
__global__ void __launch_bounds__(128) tc_gemm(const float* A, const float* B, float* D) {
  __shared__ __align__(128) float sa[M * K];
  __shared__ __align__(128) float sb[N * K];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x, warp = tid / 32;
  // operands -> canonical layout (chunks of 4 tf32 = 16 B)
  for (int i = tid; i < M * K; i += 128) {
    const int m = i / K, k = i % K, c = k / 4;
    if (kAMN)  // MN-major: (m-quad, k): 16 B rows of 4 consecutive m; 8 k-rows per core matrix;
               // m-quads 128 B apart (SBO), 8-k groups (M/4)*128 B apart (LBO)
      sa[((m / 4) * 128 + (k / 8) * (M / 4) * 128 + (k % 8) * 16) / 4 + m % 4] = A[i];
    else
      sa[(c * (M / 8) * 128 + (m / 8) * 128 + (m % 8) * 16) / 4 + k % 4] = A[i];
  }
  for (int i = tid; i < N * K; i += 128) {
    const int n = i / K, k = i % K, c = k / 4;
    sb[(c * (N / 8) * 128 + (n / 8) * 128 + (n % 8) * 16) / 4 + k % 4] = B[i];
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> tensor core
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  if (tid == 0) {
    const uint32_t id = idesc_tf32(M, N) | (kAMN ? (1u << 15) : 0u);
    for (int t = 0; t < K / 8; ++t) {  // K = 8 per tf32 MMA = 2 chunks
      const uint64_t da = kAMN == 1 ? sdesc(smem_u32(sa) + t * (M / 4) * 128, (M / 4) * 128, 128)
                        : kAMN == 2 ? sdesc(smem_u32(sa) + t * (M / 4) * 128, 128, (M / 4) * 128)
                                    : sdesc(smem_u32(sa) + 2 * t * (M / 8) * 128, (M / 8) * 128, 128);
      const uint64_t db = sdesc(smem_u32(sb) + 2 * t * (N / 8) * 128, (N / 8) * 128, 128);
      const uint32_t acc = t > 0;
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
          "l"(da), "l"(db), "r"(id), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&mbar))
                 : "memory");
  }
  // wait for the MMAs
  asm volatile(
      "{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(
          smem_u32(&mbar))
      : "memory");
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  uint32_t v[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
        "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
        "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(tmem + (static_cast<uint32_t>(warp * 32) << 16)));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int n = 0; n < N; ++n) D[tid * N + n] = __uint_as_float(v[n]);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

int main() {
  float *hA = new float[M * K], *hB = new float[N * K], *hD = new float[M * N];
  srand(1);
  for (int i = 0; i < M * K; ++i) hA[i] = (rand() % 2001 - 1000) / 1000.0f;
  for (int i = 0; i < N * K; ++i) hB[i] = (rand() % 2001 - 1000) / 1000.0f;
  float *A, *B, *D;
  cudaMalloc(&A, M * K * 4);
  cudaMalloc(&B, N * K * 4);
  cudaMalloc(&D, M * N * 4);
  cudaMemcpy(A, hA, M * K * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(B, hB, N * K * 4, cudaMemcpyHostToDevice);
  cudaMemset(D, 0, M * N * 4);
  for (int mode = 0; mode < 3; ++mode) {
  cudaMemset(D, 0, M * N * 4);
  if (mode == 0) tc_gemm<0><<<1, 128>>>(A, B, D);
  else if (mode == 1) tc_gemm<1><<<1, 128>>>(A, B, D);
  else tc_gemm<2><<<1, 128>>>(A, B, D);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(hD, D, M * N * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0, maxref = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double r = 0;
      for (int k = 0; k < K; ++k) r += (double)hA[m * K + k] * hB[n * K + k];
      maxerr = fmax(maxerr, fabs(r - hD[m * N + n]));
      maxref = fmax(maxref, fabs(r));
    }
  printf("tcgen05 tf32 GEMM %dx%dx%d A %s-major: %s, max |err| %.3e (max |ref| %.3e), D[0]=%f D[last]=%f\n", M, N,
         K, mode == 0 ? "K" : (mode == 1 ? "MN(lbo=kgrp)" : "MN(lbo=128)"), cudaGetErrorString(e), maxerr, maxref, hD[0], hD[M * N - 1]);
  }
  return 0;
}
