// tma_align_probe.cu — tool (not product): does a 2-D tiled TMA load (f32, SWIZZLE_128B,
// 32-float inner box) accept an inner start coordinate that is not 16-byte aligned?
// Loads box {32, 8} at x = 0..7 from a [64 x 256] f32 matrix (value = row * 1000 + col),
// un-swizzles the smem tile and compares with the expected shifted window.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/tma_align_probe tools/tma_align_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstring>

__global__ void probe(const __grid_constant__ CUtensorMap tm, int x0, float* out) {
  __shared__ __align__(1024) float tile[8 * 32];
  __shared__ __align__(8) uint64_t bar;
  const uint32_t b = static_cast<uint32_t>(__cvta_generic_to_shared(&bar));
  const uint32_t t = static_cast<uint32_t>(__cvta_generic_to_shared(tile));
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(8 * 32 * 4) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(t),
        "l"(reinterpret_cast<uint64_t>(&tm)), "r"(x0), "r"(3), "r"(b)
        : "memory");
    asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n\t}" ::"r"(b)
                 : "memory");
  }
  __syncthreads();
  // SWIZZLE_128B: 16-byte chunk c of row r sits at chunk c ^ (r % 8)
  for (int i = threadIdx.x; i < 8 * 32; i += blockDim.x) {
    const int r = i / 32, col = i % 32, c = col / 4, w = col % 4;
    out[i] = tile[r * 32 + ((c ^ (r & 7)) * 4) + w];
  }
}

int main() {
  const int R = 64, Cc = 256;
  float* h = new float[R * Cc];
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < Cc; ++c) h[r * Cc + c] = r * 1000.f + c;
  float *d, *o;
  cudaMalloc(&d, R * Cc * 4);
  cudaMalloc(&o, 8 * 32 * 4);
  cudaMemcpy(d, h, R * Cc * 4, cudaMemcpyHostToDevice);
  CUtensorMap tm;
  cuuint64_t dims[2] = {(cuuint64_t)Cc, (cuuint64_t)R};
  cuuint64_t strides[1] = {(cuuint64_t)Cc * 4};
  cuuint32_t box[2] = {32, 8}, es[2] = {1, 1};
  CUresult rc = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, dims, strides, box, es,
                                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                       CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (rc != CUDA_SUCCESS) {
    printf("encode failed %d\n", rc);
    return 1;
  }
  float got[256];
  for (int x0 = 0; x0 < 8; ++x0) {
    probe<<<1, 128>>>(tm, x0, o);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("x0=%d: %s\n", x0, cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(got, o, sizeof(got), cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int r = 0; r < 8; ++r)
      for (int c = 0; c < 32; ++c)
        if (got[r * 32 + c] != (3 + r) * 1000.f + (x0 + c)) ++bad;
    printf("inner start x0 = %d (%s): %d of 256 elements wrong; first row %g %g .. %g\n", x0,
           (x0 * 4) % 16 ? "not 16-B aligned" : "16-B aligned", bad, got[0], got[1], got[31]);
  }
  return 0;
}
