// tma_gather_probe.cu — tool (not product): TMA tile::gather4 of bf16 rows into the
// SWIZZLE_128B K-major layout the fast MLP step's MMA reads (csrc/mlp_tc.cu), with and
// without cluster multicast; which tensor-map box height gather4 wants; and its cost.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tma_gather_probe tools/tma_gather_probe.cu
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

constexpr int NR = 4096, FC = 832, B = 32, NA = FC / 64;  // rows, padded features, batch, atoms

__device__ __forceinline__ uint32_t saddr(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t ph) {
  asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}" ::"r"(saddr(b)), "r"(ph) : "memory");
}
__device__ __forceinline__ uint32_t cta_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

// every CTA of the cluster ends with the whole batch (32 rows x NA atoms) in smem; CTA q
// issues the gathers g with g % ncta == q and multicasts them (mask = all) when mc
__global__ void __launch_bounds__(128) gather_kernel(const __grid_constant__ CUtensorMap tm, const int* rows, int mc,
                                                     __nv_bfloat16* out, long long* cyc, int nrep) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* sm = smem_raw + ((1024 - (saddr(smem_raw) & 1023)) & 1023);
  __shared__ __align__(8) uint64_t bar;
  uint32_t ncta;
  asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(ncta));
  const uint32_t rank = cta_rank();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(saddr(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  for (int rep = 0; rep < nrep; ++rep) {
    const int* rr = rows + (rep % 8) * B;
    const long long t0 = clock64();
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(&bar)), "r"(B * NA * 128) : "memory");
    }
    if (mc) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    // gathers: (atom a, 4-row group g4): 8 groups x NA atoms
    for (uint32_t g = threadIdx.x; g < 8 * NA; g += 128) {
      if (mc && g % ncta != rank) continue;
      const uint32_t a = g / 8, g4 = g % 8;
      const uint32_t dst = saddr(sm + a * 4096 + g4 * 512);
      const int c0 = a * 64;
      const int r0 = rr[g4 * 4], r1 = rr[g4 * 4 + 1], r2 = rr[g4 * 4 + 2], r3 = rr[g4 * 4 + 3];
      if (mc) {
        const uint16_t mask = static_cast<uint16_t>((1u << ncta) - 1);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes.multicast::cluster"
            " [%0], [%1, {%3, %4, %5, %6, %7}], [%2], %8;" ::"r"(dst),
            "l"(&tm), "r"(saddr(&bar)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "h"(mask)
            : "memory");
      } else {
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(dst),
            "l"(&tm), "r"(saddr(&bar)), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
            : "memory");
      }
    }
    mbar_wait(&bar, rep & 1);
    const long long t1 = clock64();
    if (threadIdx.x == 0 && rank == 0) cyc[rep] = t1 - t0;
    __syncthreads();
    if (mc) asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
  }
  // unswizzle this CTA's copy of the last rep into out[rank][b][f]
  for (uint32_t i = threadIdx.x; i < B * FC; i += 128) {
    const uint32_t b = i / FC, f = i % FC, a = f / 64, q = (f % 64) / 8;
    const uint32_t off = a * 4096 + (b / 8) * 1024 + (b % 8) * 128 + ((q ^ (b % 8)) * 16) + (f % 8) * 2;
    out[(static_cast<size_t>(rank) * B + b) * FC + f] = *reinterpret_cast<const __nv_bfloat16*>(sm + off);
  }
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

int main(int argc, char** argv) {
  // "host": the rows live in pinned, mapped HOST memory (the tensor map addresses it over
  // PCIe) — the stream-mode question: can the step's TMA gather read host batches directly?
  const bool host = argc > 1 && std::string(argv[1]) == "host";
  std::vector<__nv_bfloat16> G(static_cast<size_t>(NR) * FC);
  for (int r = 0; r < NR; ++r)
    for (int f = 0; f < FC; ++f) G[static_cast<size_t>(r) * FC + f] = __float2bfloat16(static_cast<float>((r * 7 + f) % 251));
  __nv_bfloat16 *dG, *dO;
  int* dR;
  long long* dC;
  if (host) {
    CK(cudaHostAlloc(&dG, G.size() * 2, cudaHostAllocMapped));
    std::memcpy(dG, G.data(), G.size() * 2);
  } else {
    CK(cudaMalloc(&dG, G.size() * 2));
    CK(cudaMemcpy(dG, G.data(), G.size() * 2, cudaMemcpyHostToDevice));
  }
  std::vector<int> rows(8 * B);
  srand(5);
  for (auto& v : rows) v = rand() % NR;
  CK(cudaMalloc(&dR, rows.size() * 4));
  CK(cudaMemcpy(dR, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&dO, 16 * B * FC * 2));
  CK(cudaMalloc(&dC, 64 * 8));
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q{};
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  const int smem = (NA + 1) * 4096 + 1024;
  CK(cudaFuncSetAttribute(gather_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  CK(cudaFuncSetAttribute(gather_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  for (int bh : {1}) {
    CUtensorMap tm;
    const cuuint64_t dims[2] = {FC, NR};
    const cuuint64_t strides[1] = {FC * 2};
    const cuuint32_t box[2] = {64, static_cast<cuuint32_t>(bh)};
    const cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, dG, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      printf("box height %d: encode failed %d\n", bh, static_cast<int>(r));
      continue;
    }
    for (int cl : {1, 16}) {
      for (int mc : {0, 1}) {
        if (cl == 1 && mc) continue;
        cudaLaunchConfig_t c = {};
        c.gridDim = dim3(cl);
        c.blockDim = dim3(128);
        c.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cl;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        c.attrs = at;
        c.numAttrs = 1;
        CK(cudaMemset(dO, 0, 16 * B * FC * 2));
        const int nrep = 32;
        cudaError_t e = cudaLaunchKernelEx(&c, gather_kernel, tm, dR, mc, dO, dC, nrep);
        if (e == cudaSuccess) e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
          printf("box %d cluster %d mc %d: CUDA error %s\n", bh, cl, mc, cudaGetErrorString(e));
          return 1;
        }
        std::vector<__nv_bfloat16> O(static_cast<size_t>(cl) * B * FC);
        std::vector<long long> cy(nrep);
        CK(cudaMemcpy(O.data(), dO, O.size() * 2, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(cy.data(), dC, nrep * 8, cudaMemcpyDeviceToHost));
        const int* last = rows.data() + ((nrep - 1) % 8) * B;
        long bad = 0;
        for (int k = 0; k < cl; ++k)
          for (int b = 0; b < B; ++b)
            for (int f = 0; f < FC; ++f)
              if (__bfloat162float(O[(static_cast<size_t>(k) * B + b) * FC + f]) !=
                  __bfloat162float(G[static_cast<size_t>(last[b]) * FC + f]))
                ++bad;
        std::sort(cy.begin() + 4, cy.end());
        printf("%s rows, box height %d, cluster %2d, multicast %d: %s (%ld mismatches), batch gather %lld cycles (median)\n", host ? "host" : "device", bh, cl,
               mc, bad ? "WRONG" : "OK", bad, cy[4 + (nrep - 4) / 2]);
      }
    }
  }
  return 0;
}
