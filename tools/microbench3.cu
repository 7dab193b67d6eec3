// microbench3.cu — the fused kernel's reference-order dot products in isolation:
// 64 threads x (784-long f32 dot, exact f64 chain), one CTA, clock64. Tool only.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double mb_dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double mb_dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ void products16(const float4* w4, const float4* x4, unsigned blk, double (&p)[16]) {
  float4 wv[4], xv[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) { wv[k] = w4[4 * blk + k]; xv[k] = x4[4 * blk + k]; }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    p[4 * k + 0] = mb_dmul((double)wv[k].x, (double)xv[k].x);
    p[4 * k + 1] = mb_dmul((double)wv[k].y, (double)xv[k].y);
    p[4 * k + 2] = mb_dmul((double)wv[k].z, (double)xv[k].z);
    p[4 * k + 3] = mb_dmul((double)wv[k].w, (double)xv[k].w);
  }
}
template <int kMode>
__global__ void k(double* out, long long* cyc, unsigned n) {
  extern __shared__ float sm[];
  float* w = sm;            // 2 x n
  float* x = sm + 2 * n;    // 32 x (n+4)
  for (unsigned i = threadIdx.x; i < 2 * n + 32 * (n + 4); i += blockDim.x) sm[i] = 1.0f + 1e-3f * (i % 97);
  __syncthreads();
  long long t0 = clock64();
  double z = 0.5;
  if (threadIdx.x < 64) {
    const unsigned r = threadIdx.x / 2, u = threadIdx.x % 2;
    const float* wr = w + u * n;
    const float* xr = x + r * (n + 4);
    if (kMode == 0) {
      for (unsigned i = 0; i < n; ++i) z = mb_dadd(z, mb_dmul((double)wr[i], (double)xr[i]));
    } else {
      const float4* w4 = reinterpret_cast<const float4*>(wr);
      const float4* x4 = reinterpret_cast<const float4*>(xr);
      double p[16], q[16];
      products16(w4, x4, 0, p);
      for (unsigned b = 1; b < n / 16; ++b) {
        products16(w4, x4, b, q);
#pragma unroll
        for (int j = 0; j < 16; ++j) z = mb_dadd(z, p[j]);
#pragma unroll
        for (int j = 0; j < 16; ++j) p[j] = q[j];
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) z = mb_dadd(z, p[j]);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  out[threadIdx.x] = z;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  const unsigned n = 784;
  double* o; long long* c;
  cudaMalloc(&o, 4096 * 8); cudaMalloc(&c, 8);
  size_t smem = (2 * n + 32 * (n + 4)) * 4;
  for (int threads : {64, 384}) {
    cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    long long h;
    k<0><<<1, threads, smem>>>(o, c, n); k<0><<<1, threads, smem>>>(o, c, n);
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("threads=%d naive   : %lld cycles (%.1f/elem)\n", threads, h, double(h) / n);
    k<1><<<1, threads, smem>>>(o, c, n); k<1><<<1, threads, smem>>>(o, c, n);
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("threads=%d pipelined: %lld cycles (%.1f/elem)\n", threads, h, double(h) / n);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
