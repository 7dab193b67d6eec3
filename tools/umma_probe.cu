// umma_probe.cu — tool (not product): settles the tcgen05 / DSMEM questions the fast MLP
// step (csrc/mlp_tc.cu) depends on, on the real B200. Results: profiles/r02_umma_timing.md.
//   modes 0-2 (kind::f16, bf16 operands, f32 accumulate, SWIZZLE_128B):
//     0: forward  D[64 x 16] = X[32 (+32 aliased rows) x 784] . W[16 x 784]^T, both K-major;
//     1: weight gradient D[128 x 16] = X^T[128 features x 32] . d[32 x 16] with A = the SAME
//        X bytes read MN-major (LBO = atom stride, SBO = 8-row group stride);
//     2: as 1 with LBO/SBO swapped;
//   (tf32: MN-major A was measured wrong in both no-swizzle and SW128 layouts, so the fast
//   step computes in bf16.)
//   dsmem: two-phase tiny-message all-reduce over a 16-CTA cluster with st.async +
//   mbarrier complete_tx (the fast step's logits reduce-scatter + delta all-gather).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/umma_probe tools/umma_probe.cu
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

constexpr int B = 32, F = 784, NU = 16;
constexpr int XA = F / 64 + 1;  // 13 atoms of 64 bf16 features (832 padded)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint64_t sdesc128(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return static_cast<uint64_t>((addr >> 4) & 0x3FFF) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ uint64_t sdesc32(uint32_t addr, uint32_t lbo, uint32_t sbo) {  // SWIZZLE_32B
  return static_cast<uint64_t>((addr >> 4) & 0x3FFF) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (6ull << 61);
}
// MN-major SW32 [K rows][16 N-elements = 32 B], 8-row atoms of 256 B: chunk ^= (row >> 2) & 1
__device__ __forceinline__ uint32_t mn32_off(int n, int k) {
  return (k / 8) * 256 + (k % 8) * 32 + (((n / 8) ^ ((k % 8) >> 2)) * 16) + (n % 8) * 2;
}
__host__ __device__ constexpr uint32_t idesc_bf16(int m, int n, int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(a_mn) << 15) | (static_cast<uint32_t>(b_mn) << 16) |
         (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(m >> 4) << 24);
}
__device__ __forceinline__ void mma(uint32_t tmem, uint64_t da, uint64_t db, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
               "l"(da), "l"(db), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void wait_bar(uint64_t* bar, uint32_t phase) {
  asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(smem_u32(bar)), "r"(phase) : "memory");
}
__device__ __forceinline__ void ld16(uint32_t taddr, float* v) {  // 32 lanes x 16 columns
  uint32_t r[16];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
                 "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
// SW128 K-major, 64 bf16 per 128-B row: [atom a][row group g][row%8][128 B], chunk ^= row%8
__device__ __forceinline__ uint32_t off128(int row, int k, int rows_per_atom) {
  const int a = k / 64, c = (k % 64) / 8;
  return a * (rows_per_atom * 128) + (row / 8) * 1024 + (row % 8) * 128 + ((c ^ (row % 8)) * 16) + (k % 8) * 2;
}

__global__ void __launch_bounds__(128) probe(const float* X, const float* W, const float* Dl, float* out, int mode) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __nv_bfloat16* xs = reinterpret_cast<__nv_bfloat16*>(sm);                  // XA atoms x 4 KB (+ 4 KB slack)
  __nv_bfloat16* ws = reinterpret_cast<__nv_bfloat16*>(sm + (XA + 1) * 4096);  // XA atoms x 2 KB
  __nv_bfloat16* ds = reinterpret_cast<__nv_bfloat16*>(sm + (XA + 1) * 4096 + XA * 2048);  // 16 x 32: 1 atom x 2 KB
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  const int tid = threadIdx.x, warp = tid / 32;
  for (int i = tid; i < ((XA + 1) * 4096 + XA * 2048 + 2048) / 4; i += 128) reinterpret_cast<float*>(sm)[i] = 0.f;
  __syncthreads();
  for (int i = tid; i < B * F; i += 128) xs[off128(i / F, i % F, 32) / 2] = __float2bfloat16_rn(X[i]);
  for (int i = tid; i < NU * F; i += 128)
    ws[(mode >= 3 ? mn32_off(i / F, i % F) : off128(i / F, i % F, 16)) / 2] = __float2bfloat16_rn(W[i]);
  for (int i = tid; i < NU * B; i += 128) ds[off128(i / B, i % B, 16) / 2] = __float2bfloat16_rn(Dl[i]);
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(smem_u32(&tbase)));
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
  if (tid == 0) {
    if (mode == 3) {  // forward with B = W MN-major SW32 (units contiguous per feature row)
      const uint32_t id = idesc_bf16(64, NU, 0, 1);
      for (int k = 0; k < F / 16; ++k) {
        const uint32_t xo = (k / 4) * 4096 + (k % 4) * 32;
        mma(tmem, sdesc128(smem_u32(sm) + xo, 16, 1024), sdesc32(smem_u32(ws) + k * 512, 0, 256), id, k > 0);
      }
    } else if (mode == 4) {
      const uint32_t id = idesc_bf16(64, NU, 0, 1);
      for (int k = 0; k < F / 16; ++k) {
        const uint32_t xo = (k / 4) * 4096 + (k % 4) * 32;
        mma(tmem, sdesc128(smem_u32(sm) + xo, 16, 1024), sdesc32(smem_u32(ws) + k * 512, 256, 0), id, k > 0);
      }
    } else if (mode == 0) {
      const uint32_t id = idesc_bf16(64, NU, 0, 0);
      for (int k = 0; k < F / 16; ++k) {  // K = 16 per MMA = 32 B inside a 128-B row
        const uint32_t xo = (k / 4) * 4096 + (k % 4) * 32, wo = (k / 4) * 2048 + (k % 4) * 32;
        mma(tmem, sdesc128(smem_u32(sm) + xo, 16, 1024), sdesc128(smem_u32(ws) + wo, 16, 1024), id, k > 0);
      }
    } else {
      const uint32_t id = idesc_bf16(128, NU, 1, 0);
      for (int k = 0; k < B / 16; ++k) {  // K = 16 batch rows = 2 row groups
        const uint64_t da = mode == 1 ? sdesc128(smem_u32(sm) + k * 2048, 4096, 1024) : sdesc128(smem_u32(sm) + k * 2048, 1024, 4096);
        mma(tmem, da, sdesc128(smem_u32(ds) + k * 32, 16, 1024), id, k > 0);
      }
    }
    commit(&bar);
  }
  wait_bar(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  float v[16];
  ld16(tmem + (static_cast<uint32_t>(warp * 32) << 16), v);
  const int lane = warp * 32 + (tid % 32);
  for (int n = 0; n < NU; ++n) out[lane * NU + n] = v[n];
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem));
}

// ---- DSMEM: 16-CTA tiny-message two-phase exchange (st.async + mbarrier complete_tx) ----
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async_v4(uint32_t raddr, float4 v, uint32_t rbar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1,%2,%3,%4}, [%5];" ::"r"(raddr),
               "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(rbar) : "memory");
}
__global__ void __launch_bounds__(256) allreduce_probe(long long* cyc, int nrep, int msg16) {
  __shared__ __align__(16) float4 inbox[2][16][8];
  __shared__ __align__(8) uint64_t bars[2];
  const int tid = threadIdx.x;
  uint32_t rank, ncta;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(ncta));
  if (tid == 0) {
    for (int p = 0; p < 2; ++p) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bars[p])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  uint32_t ph = 0;
  for (int rep = 0; rep < nrep; ++rep) {
    const long long t0 = clock64();
    for (int p = 0; p < 2; ++p) {
      if (tid == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bars[p])),
                     "r"((ncta - 1) * msg16 * 16) : "memory");
      if (tid < static_cast<int>(ncta) * msg16) {  // thread -> (peer, piece)
        const uint32_t peer = tid / msg16, piece = tid % msg16;
        if (peer != rank)
          st_async_v4(mapa(smem_u32(&inbox[p][rank][piece]), peer), make_float4(1.f, 2.f, 3.f, 4.f),
                      mapa(smem_u32(&bars[p]), peer));
      }
      wait_bar(&bars[p], ph);
    }
    ph ^= 1;
    if (tid == 0) cyc[rank * nrep + rep] = clock64() - t0;
    __syncthreads();
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

int main() {
  std::vector<float> X(B * F), W(NU * F), D(NU * B);
  srand(1);
  for (auto& v : X) v = (rand() % 2001 - 1000) / 1000.f;
  for (auto& v : W) v = (rand() % 2001 - 1000) / 1000.f;
  for (auto& v : D) v = (rand() % 2001 - 1000) / 1000.f;
  auto bf = [](float x) { return __bfloat162float(__float2bfloat16_rn(x)); };
  float *dX, *dW, *dD, *dO;
  CK(cudaMalloc(&dX, X.size() * 4)); CK(cudaMalloc(&dW, W.size() * 4)); CK(cudaMalloc(&dD, D.size() * 4));
  CK(cudaMalloc(&dO, 128 * NU * 4));
  CK(cudaMemcpy(dX, X.data(), X.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dW, W.data(), W.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dD, D.data(), D.size() * 4, cudaMemcpyHostToDevice));
  const int smem = (XA + 1) * 4096 + XA * 2048 + 2048;
  CK(cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  for (int mode = 0; mode < 5; ++mode) {
    CK(cudaMemset(dO, 0, 128 * NU * 4));
    probe<<<1, 128, smem>>>(dX, dW, dD, dO, mode);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("mode %d: CUDA error %s\n", mode, cudaGetErrorString(e)); return 1; }
    std::vector<float> O(128 * NU);
    CK(cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost));
    double maxerr = 0, maxref = 0;
    const bool fwd = mode == 0 || mode >= 3;
    for (int r = 0; r < (fwd ? B : 128); ++r)
      for (int n = 0; n < NU; ++n) {
        double ref = 0;
        if (fwd) for (int k = 0; k < F; ++k) ref += (double)bf(X[r * F + k]) * bf(W[n * F + k]);
        else for (int b = 0; b < B; ++b) ref += (double)bf(X[b * F + r]) * bf(D[n * B + b]);
        const int lane = fwd ? (r % 16) + 32 * (r / 16) : r;
        maxerr = fmax(maxerr, fabs(ref - O[lane * NU + n]));
        maxref = fmax(maxref, fabs(ref));
      }
    printf("bf16 mode %d: max|err| %.3g (max|ref| %.3g) %s\n", mode, maxerr, maxref, maxerr < 1e-4 * maxref ? "OK" : "WRONG");
  }
  long long* lc;
  CK(cudaMalloc(&lc, 16 * 64 * 8));
  CK(cudaFuncSetAttribute(allreduce_probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  for (int cl : {16, 8, 4})
    for (int msg : {1, 5, 8}) {
      cudaLaunchConfig_t q = {};
      q.gridDim = dim3(cl);
      q.blockDim = dim3(256);
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = cl; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
      q.attrs = at; q.numAttrs = 1;
      CK(cudaLaunchKernelEx(&q, allreduce_probe, lc, 64, msg));
      CK(cudaDeviceSynchronize());
      std::vector<long long> c(cl * 64);
      CK(cudaMemcpy(c.data(), lc, c.size() * 8, cudaMemcpyDeviceToHost));
      std::vector<long long> s(c.begin() + 8, c.begin() + 64);
      std::sort(s.begin(), s.end());
      printf("st.async 2-phase exchange, %2d CTAs, %3d B to each peer per phase: median %lld cycles (both phases)\n", cl,
             msg * 16, s[s.size() / 2]);
    }
  return 0;
}
