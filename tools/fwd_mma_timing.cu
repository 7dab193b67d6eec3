// fwd_mma_timing.cu — tool (not product): the tensor-core step's forward MMA chain in
// isolation (csrc/mlp_tc.cu): 49 x tcgen05.mma kind::f16 M64 N16 K16 with A = the staged
// batch (K-major SWIZZLE_128B, 32-row atoms of 64 features, 4 KB each, walking 13 atoms)
// and B = the CTA's bf16 W1 rows, either MN-major SWIZZLE_32B (the kernel's layout) or
// K-major SWIZZLE_128B (16-row atoms). Also: the same chain with A fixed to one atom (the
// umma_timing.cu setting), and M = 128. Prints cycles per MMA (issue -> commit done).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/fwd_mma_timing tools/fwd_mma_timing.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo, uint64_t layout) {
  return static_cast<uint64_t>((addr >> 4) & 0x3FFF) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (layout << 61);
}
__host__ __device__ constexpr uint32_t idesc_bf16(int m, int n, int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(a_mn) << 15) | (static_cast<uint32_t>(b_mn) << 16) |
         (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(m >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t tmem, uint64_t da, uint64_t db, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
               "l"(da), "l"(db), "r"(id), "r"(acc));
}

// mode 0: A walks 13 atoms, B MN-major SW32 (kernel); 1: A walks, B K-major SW128;
// 2: A fixed atom, B MN-major; 3: A walks, B MN-major, M = 128;
// 4..: kernel layout, MMA k accumulates into TMEM columns (k % nacc) * 16 (independent chains)
__global__ void __launch_bounds__(128) fwd_timing(int mode, int nacc, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  for (int i = tid; i < (96 * 1024) / 4; i += 128) reinterpret_cast<float*>(sm)[i] = 0.f;
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tbase;
  uint32_t phase = 0;
  long long best = 1ll << 60;
  const uint32_t a0 = smem_u32(sm), b0 = smem_u32(sm + 60 * 1024);
  const bool kmaj = mode == 1;
  const uint32_t id = idesc_bf16(mode == 3 ? 128 : 64, 16, 0, kmaj ? 0 : 1);
  const uint64_t da = sdesc(a0, 16, 1024, 2);
  const uint64_t db = kmaj ? sdesc(b0, 16, 1024, 2) : sdesc(b0, 0, 256, 6);
  for (int rep = 0; rep < 12; ++rep) {
    if (tid == 0) {
      const long long t0 = clock64();
      for (uint32_t k = 0; k < 49; ++k) {
        const uint64_t ao = (mode == 2 ? 0u : (k >> 2) * 256u) + (k & 3) * 2;
        const uint64_t bo = kmaj ? (k >> 2) * 128u + (k & 3) * 2 : k * 32u;
        mma(tmem + (k % nacc) * 16, da + ao, db + bo, id, k >= (uint32_t)nacc);
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
      asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(&bar)),
                   "r"(phase) : "memory");
      const long long t1 = clock64();
      if (rep >= 2) best = min(best, t1 - t0);
    }
    phase ^= 1;
    __syncthreads();
  }
  if (tid == 0) out[blockIdx.x] = best;
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

// nw warps each issue their share of the 49 MMAs (warp w: k = w, w + nw, ...) into their own
// accumulator (TMEM columns w * 16); one commit per warp; cycles from a common start until
// every warp's commit completed (CTA 0, best of 10)
__global__ void __launch_bounds__(128) multi_issue(int nw, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar[4];
  __shared__ uint32_t tbase;
  __shared__ long long t0s;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  for (int i = tid; i < (96 * 1024) / 4; i += 128) reinterpret_cast<float*>(sm)[i] = 0.f;
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tbase;
  const uint32_t a0 = smem_u32(sm), b0 = smem_u32(sm + 60 * 1024);
  const uint32_t id = idesc_bf16(64, 16, 0, 1);
  const uint64_t da = sdesc(a0, 16, 1024, 2);
  const uint64_t db = sdesc(b0, 0, 256, 6);
  long long best = 1ll << 60;
  for (int rep = 0; rep < 12; ++rep) {
    __syncthreads();
    if (tid == 0) t0s = clock64();
    __syncthreads();
    if (warp < nw && lane == 0) {
      for (uint32_t k = warp, j = 0; k < 49; k += nw, ++j) {
        const uint64_t ao = (k >> 2) * 256u + (k & 3) * 2;
        mma(tmem + warp * 16, da + ao, db + k * 32u, id, j > 0);
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar[warp])) : "memory");
      asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(&bar[warp])),
                   "r"(rep & 1) : "memory");
    }
    __syncthreads();
    if (tid == 0 && rep >= 2) best = min(best, clock64() - t0s);
  }
  if (tid == 0) out[blockIdx.x] = best;
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

// single issuing lane, kernel layout, the issue loop unrolled U times (U = 49: straight line)
template <int U>
__global__ void __launch_bounds__(128) unroll_timing(long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  for (int i = tid; i < (96 * 1024) / 4; i += 128) reinterpret_cast<float*>(sm)[i] = 0.f;
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tbase;
  long long best = 1ll << 60;
  const uint32_t id = idesc_bf16(64, 16, 0, 1);
  const uint64_t da = sdesc(smem_u32(sm), 16, 1024, 2);
  const uint64_t db = sdesc(smem_u32(sm + 60 * 1024), 0, 256, 6);
  for (int rep = 0; rep < 12; ++rep) {
    if (tid == 0) {
      const long long t0 = clock64();
      uint64_t a = da, b = db;
#pragma unroll U
      for (uint32_t k = 0; k < 49; ++k, b += 32) {
        mma(tmem, a + (k & 3) * 2, b, id, k > 0);
        if ((k & 3) == 3) a += 256;
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
      asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(&bar)),
                   "r"(rep & 1) : "memory");
      const long long t1 = clock64();
      if (rep >= 2) best = min(best, t1 - t0);
    }
    __syncthreads();
  }
  if (tid == 0) out[blockIdx.x] = best;
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}
template <int U>
void run_unroll(long long* d) {
  CK(cudaFuncSetAttribute(unroll_timing<U>, cudaFuncAttributeMaxDynamicSharedMemorySize, 97 * 1024));
  unroll_timing<U><<<1, 128, 97 * 1024>>>(d);
  CK(cudaDeviceSynchronize());
  long long h;
  CK(cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost));
  printf("one lane, issue loop unrolled %2d: 49 MMAs %6lld cycles = %.1f cyc/MMA\n", U, h, double(h) / 49);
}

int main() {
  long long* d;
  CK(cudaMalloc(&d, 148 * 8));
  CK(cudaFuncSetAttribute(fwd_timing, cudaFuncAttributeMaxDynamicSharedMemorySize, 97 * 1024));
  const char* names[] = {"A walks 13 atoms, B MN-major SW32 (kernel layout)", "A walks, B K-major SW128",
                         "A fixed atom, B MN-major SW32", "A walks, B MN-major SW32, M = 128"};
  for (int mode = 0; mode < 4; ++mode) {
    fwd_timing<<<1, 128, 97 * 1024>>>(mode, 1, d);
    CK(cudaDeviceSynchronize());
    long long h;
    CK(cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost));
    printf("%-52s: 49 MMAs %6lld cycles = %.1f cyc/MMA\n", names[mode], h, double(h) / 49);
  }
  for (int na : {2, 4, 7, 8, 14}) {
    fwd_timing<<<1, 128, 97 * 1024>>>(0, na, d);
    CK(cudaDeviceSynchronize());
    long long h;
    CK(cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost));
    printf("kernel layout, %2d independent accumulators (N16 each): 49 MMAs %6lld cycles = %.1f cyc/MMA\n", na, h, double(h) / 49);
  }
  CK(cudaFuncSetAttribute(multi_issue, cudaFuncAttributeMaxDynamicSharedMemorySize, 97 * 1024));
  for (int nw : {1, 2, 4}) {
    multi_issue<<<1, 128, 97 * 1024>>>(nw, d);
    CK(cudaDeviceSynchronize());
    long long h;
    CK(cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost));
    printf("%d issuing warps (own accumulators): 49 MMAs %6lld cycles = %.1f cyc/MMA\n", nw, h, double(h) / 49);
  }
  run_unroll<1>(d);
  run_unroll<4>(d);
  run_unroll<8>(d);
  run_unroll<49>(d);
  // the same chain on many SMs at once (the step runs 16 CTAs per worker, 2 SMs per TPC)
  for (int nb : {2, 16, 32, 148}) {
    fwd_timing<<<nb, 128, 97 * 1024>>>(0, 1, d);
    CK(cudaDeviceSynchronize());
    long long h[148];
    CK(cudaMemcpy(h, d, nb * 8, cudaMemcpyDeviceToHost));
    long long mx = 0, mn = 1ll << 60;
    for (int i = 0; i < nb; ++i) mx = h[i] > mx ? h[i] : mx, mn = h[i] < mn ? h[i] : mn;
    printf("kernel layout on %3d CTAs at once: %.1f .. %.1f cyc/MMA\n", nb, double(mn) / 49, double(mx) / 49);
  }
  return 0;
}
