// umma_timing.cu — tool (not product): per-instruction cost of small tcgen05.mma chains and
// the cost of gathering one 32 x 784 f32 batch into one SM, which together pick the work
// split of the fast MLP step (csrc/mlp_tc.cu). Results: profiles/r02_umma_timing.md.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/umma_timing tools/umma_timing.cu
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t sdesc128(uint32_t addr, uint32_t sbo) {
  return static_cast<uint64_t>((addr >> 4) & 0x3FFF) | (1ull << 16) | (static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32) |
         (1ull << 46) | (2ull << 61);
}
// kind 0: tf32 (K = 8), kind 1: bf16 (K = 16); f32 accumulate
__host__ __device__ constexpr uint32_t idesc(int kind, int m, int n) {
  return (1u << 4) | (kind == 0 ? (2u << 7) | (2u << 10) : (1u << 7) | (1u << 10)) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(m >> 4) << 24);
}
template <int KIND>
__device__ __forceinline__ void mma(uint32_t tmem, uint64_t da, uint64_t db, uint32_t id, uint32_t acc) {
  if (KIND == 0)
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                 "l"(da), "l"(db), "r"(id), "r"(acc));
  else
    asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                 "l"(da), "l"(db), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void wait_bar(uint64_t* bar, uint32_t phase) {
  asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(bar)), "r"(phase) : "memory");
}

// A: one SW128 atom of 128 rows (16 KB), B: one atom of 256 rows (32 KB); contents irrelevant.
template <int KIND>
__global__ void __launch_bounds__(128) mma_timing(int M, int N, int nmma, int nacc, long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x;
  for (int i = tid; i < (48 * 1024) / 4; i += 128) reinterpret_cast<float*>(sm)[i] = 0.f;
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
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
  long long best_issue = 1ll << 60, best_done = 1ll << 60;
  for (int rep = 0; rep < 12; ++rep) {
    if (tid == 0) {
      const uint32_t id = idesc(KIND, M, N);
      const uint32_t a0 = smem_u32(sm), b0 = smem_u32(sm + 16384);
      const long long t0 = clock64();
#pragma unroll 4
      for (int k = 0; k < nmma; ++k) {
        const uint32_t ko = (k & 3) * 32;
        const uint32_t acc_col = nacc == 2 ? (k & 1) * 256 : 0;
        mma<KIND>(tmem + acc_col, sdesc128(a0 + ko, 1024), sdesc128(b0 + ko, 1024), id, k >= nacc);
      }
      const long long t1 = clock64();
      commit(&bar);
      wait_bar(&bar, phase);
      const long long t2 = clock64();
      if (rep >= 2) {
        best_issue = min(best_issue, t1 - t0);
        best_done = min(best_done, t2 - t0);
      }
    }
    phase ^= 1;
    __syncthreads();
  }
  if (tid == 0) {
    out[0] = best_issue;
    out[1] = best_done;
  }
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

constexpr int F = 784;
// Batch gather variants (32 random rows x 784 f32 -> smem), per CTA:
//  0: cp.async 16 B, warp request = 8 rows x 4 chunks, dst = canonical interleaved (chunk*512 + row*16)
//  1: cp.async 16 B, warp request = 32 chunks of one row (512 contiguous bytes), dst interleaved
//  2: cp.async 16 B, row-contiguous src and dst (row-major smem)
//  3: ld.global.v4 (25 in flight per thread) + st.shared, row-major
//  4: cp.async.bulk (TMA 1-D) one 3136-byte row per lane of warp 0, mbarrier complete_tx
__global__ void __launch_bounds__(256) load_probe(const float* Xg, const uint32_t* rows, int variant, long long* cyc,
                                                  int nrep, int hot) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x, lane = tid % 32, warp = tid / 32;
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t phase = 0;
  for (int rep = 0; rep < nrep; ++rep) {
    __syncthreads();
    const long long t0 = clock64();
    const uint32_t* rr = rows + (hot ? 0 : (rep * 32) % 4096);
    if (variant == 0) {
      for (int g = warp; g < 4 * 49; g += 8) {
        const int rg = g / 49, cg = g % 49;
        const int b = rg * 8 + (lane % 8), c = cg * 4 + lane / 8;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sm + c * 512 + b * 16)),
                     "l"(Xg + static_cast<size_t>(rr[b]) * F + c * 4) : "memory");
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
    } else if (variant == 1 || variant == 2) {
      for (int b = warp; b < 32; b += 8) {
        const float* src = Xg + static_cast<size_t>(rr[b]) * F;
        for (int c = lane; c < 196; c += 32) {
          const uint32_t dst = variant == 1 ? smem_u32(sm + c * 512 + b * 16) : smem_u32(sm + b * 3136 + c * 16);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src + c * 4) : "memory");
        }
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
    } else if (variant == 3) {
      float4 v[25];
      int cnt = 0;
#pragma unroll
      for (int i = 0; i < 25; ++i) {
        const int p = tid + 256 * i;  // piece: row p/196, chunk p%196
        if (p < 32 * 196) v[i] = __ldcg(reinterpret_cast<const float4*>(Xg + static_cast<size_t>(rr[p / 196]) * F + (p % 196) * 4));
      }
#pragma unroll
      for (int i = 0; i < 25; ++i) {
        const int p = tid + 256 * i;
        if (p < 32 * 196) { *reinterpret_cast<float4*>(sm + (p / 196) * 3136 + (p % 196) * 16) = v[i]; ++cnt; }
      }
      if (cnt < 0) cyc[0] = 0;
    } else {
      if (warp == 0) {
        if (lane == 0)
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(32 * 3136) : "memory");
        __syncwarp();
        asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         smem_u32(sm + lane * 3136)),
                     "l"(Xg + static_cast<size_t>(rr[lane]) * F), "r"(3136), "r"(smem_u32(&bar))
                     : "memory");
      }
      wait_bar(&bar, phase);
      phase ^= 1;
    }
    __syncthreads();
    if (tid == 0) cyc[blockIdx.x * nrep + rep] = clock64() - t0;
  }
}

__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
// mode 0: push with st.shared::cluster.v4; 1: pull the same volume with ld.shared::cluster.v4;
// 2: cp.async.bulk.shared::cluster.shared::cta, one copy per destination (warp 0 lanes 0..15)
__global__ void __launch_bounds__(256) dsmem_probe(int bytes, int mode, long long* cyc, int nrep) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t bar;
  const int tid = threadIdx.x;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int i = tid; i < 16384; i += 256) reinterpret_cast<float*>(sm)[i] = static_cast<float>(i);
  cluster_sync_all();
  const int per = bytes / 16;  // bytes to each destination
  uint32_t phase = 0;
  float acc = 0.f;
  for (int rep = 0; rep < nrep; ++rep) {
    cluster_sync_all();
    const long long t0 = clock64();
    if (mode == 0) {
      for (int i = tid; i < bytes / 16; i += 256) {  // 16-byte pieces; piece i goes to CTA i % 16
        const uint32_t dst = mapa(smem_u32(sm + 32768 + rank * per + (i / 16) * 16), i % 16);
        asm volatile("st.shared::cluster.v4.f32 [%0], {%1,%1,%1,%1};" ::"r"(dst), "f"(1.f) : "memory");
      }
    } else if (mode == 1) {
      for (int i = tid; i < bytes / 16; i += 256) {
        const uint32_t src = mapa(smem_u32(sm + rank * per + (i / 16) * 16), i % 16);
        float4 v;
        asm volatile("ld.shared::cluster.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(src) : "memory");
        acc += v.x + v.w;
      }
    } else {
      if (tid == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(bytes) : "memory");
      cluster_sync_all();  // every receiver armed before any copy lands
      if (tid < 16) {
        const uint32_t dst = mapa(smem_u32(sm + 32768 + rank * per), tid);
        const uint32_t rb = mapa(smem_u32(&bar), tid);
        asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                     "r"(smem_u32(sm + tid * per)), "r"(per), "r"(rb) : "memory");
      }
      asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(&bar)), "r"(phase) : "memory");
      phase ^= 1;
    }
    cluster_sync_all();
    if (tid == 0) cyc[rank * nrep + rep] = clock64() - t0;
  }
  if (acc == 12345.f) cyc[0] = 0;
}

int main() {
  long long* d;
  CK(cudaMalloc(&d, 16 * 8));
  CK(cudaFuncSetAttribute(mma_timing<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024 + 1024));
  CK(cudaFuncSetAttribute(mma_timing<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024 + 1024));
  struct Cfg { int kind, M, N, n, acc; };
  const Cfg cfgs[] = {{0, 64, 16, 98, 1},  {0, 64, 16, 98, 2},  {0, 64, 32, 98, 1},  {0, 64, 64, 98, 1},
                      {0, 64, 128, 98, 1}, {0, 64, 256, 98, 1}, {0, 128, 16, 98, 1}, {0, 128, 64, 98, 1},
                      {0, 128, 256, 98, 1}, {0, 128, 256, 7, 1}, {0, 128, 32, 7, 1}, {0, 64, 256, 7, 1},
                      {0, 128, 16, 4, 1},  {0, 128, 256, 4, 1}, {1, 64, 16, 49, 1}, {1, 128, 256, 49, 1},
                      {0, 128, 16, 1, 1},  {0, 128, 256, 1, 1}};
  for (const Cfg& c : cfgs) {
    if (c.kind == 0) mma_timing<0><<<1, 128, 48 * 1024 + 1024>>>(c.M, c.N, c.n, c.acc, d);
    else mma_timing<1><<<1, 128, 48 * 1024 + 1024>>>(c.M, c.N, c.n, c.acc, d);
    CK(cudaDeviceSynchronize());
    long long h[2];
    CK(cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost));
    printf("%s M=%3d N=%3d x%3d MMAs (%d acc): issue %6lld cyc, issue->done %6lld cyc = %.1f cyc/MMA\n",
           c.kind ? "bf16" : "tf32", c.M, c.N, c.n, c.acc, h[0], h[1], double(h[1]) / c.n);
  }
  const size_t n = 48000;
  float* Xg;
  uint32_t* rows;
  long long* lc;
  CK(cudaMalloc(&Xg, n * F * 4));
  CK(cudaMemset(Xg, 0, n * F * 4));
  std::vector<uint32_t> hr(4096 + 64);
  srand(3);
  for (auto& v : hr) v = rand() % n;
  CK(cudaMalloc(&rows, hr.size() * 4));
  CK(cudaMemcpy(rows, hr.data(), hr.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&lc, 148 * 64 * 8));
  CK(cudaFuncSetAttribute(load_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024));
  for (int hot = 0; hot < 2; ++hot)
  for (int v = 0; v < 5; ++v)
    for (int nb : {1, 16, 148}) {
      load_probe<<<nb, 256, 110 * 1024>>>(Xg, rows, v, lc, 64, hot);
      CK(cudaDeviceSynchronize());
      std::vector<long long> c(static_cast<size_t>(nb) * 64);
      CK(cudaMemcpy(c.data(), lc, c.size() * 8, cudaMemcpyDeviceToHost));
      std::vector<long long> s(c.begin() + 8, c.begin() + 64);
      std::sort(s.begin(), s.end());
      printf("gather variant %d, %3d CTA(s), %s: median %6lld cycles for 100,352 B (CTA 0)\n", v, nb,
             hot ? "L2-hot rows" : "fresh rows", s[s.size() / 2]);
    }
  // DSMEM: each CTA of a 16-CTA cluster pushes `bytes` split over all 16 CTAs, then a cluster barrier
  CK(cudaFuncSetAttribute(dsmem_probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute(dsmem_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024));
  for (int mode = 0; mode < 3; ++mode)
    for (int bytes : {0, 2048, 8192, 20480, 32768}) {
      if (mode == 2 && bytes == 0) continue;
      cudaLaunchConfig_t q = {};
      q.gridDim = dim3(16);
      q.blockDim = dim3(256);
      q.dynamicSmemBytes = 64 * 1024;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 16; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      q.attrs = at; q.numAttrs = 1;
      CK(cudaLaunchKernelEx(&q, dsmem_probe, bytes, mode, lc, 64));
      CK(cudaDeviceSynchronize());
      std::vector<long long> c(16 * 64);
      CK(cudaMemcpy(c.data(), lc, c.size() * 8, cudaMemcpyDeviceToHost));
      std::vector<long long> s(c.begin() + 8, c.begin() + 64);
      std::sort(s.begin(), s.end());
      printf("dsmem %s: %5d B out per CTA (16-CTA cluster) + cluster barrier: median %5lld cycles\n",
             mode == 0 ? "st.shared::cluster.v4 push" : mode == 1 ? "ld.shared::cluster.v4 pull" : "cp.async.bulk smem->dsmem",
             bytes, s[s.size() / 2]);
    }
  return 0;
}
