// microbench5.cu — per-element cost of reference-order f64 dot products (784 long),
// 64 chains per CTA as in the fused kernel. Tool only.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double Dm(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double Da(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ void prod8(const double2* w2, const double2* a2, unsigned blk, double (&p)[8]) {
  double2 wv[4], av[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) { wv[k] = w2[4 * blk + k]; av[k] = a2[4 * blk + k]; }
#pragma unroll
  for (int k = 0; k < 4; ++k) { p[2 * k] = Dm(wv[k].x, av[k].x); p[2 * k + 1] = Dm(wv[k].y, av[k].y); }
}
template <int kMode>
__global__ void k(double* out, long long* cyc, unsigned n) {
  extern __shared__ double sm[];
  double* w = sm;             // 2 rows x n
  double* x = sm + 2 * n;     // 32 rows x (n+2)
  for (unsigned i = threadIdx.x; i < 2 * n + 32 * (n + 2); i += blockDim.x) sm[i] = 1.0 + 1e-3 * (i % 97);
  __syncthreads();
  long long t0 = clock64();
  double z = 0.25;
  const unsigned r = threadIdx.x / 2, u = threadIdx.x % 2;
  if (kMode == 0 && threadIdx.x < 64) {  // pipelined blocks of 8, double2 loads
    const double2* w2 = reinterpret_cast<const double2*>(w + u * n);
    const double2* a2 = reinterpret_cast<const double2*>(x + r * (n + 2));
    double p[8], q[8];
    prod8(w2, a2, 0, p);
    for (unsigned b = 1; b < n / 8; ++b) {
      prod8(w2, a2, b, q);
#pragma unroll
      for (int j = 0; j < 8; ++j) z = Da(z, p[j]);
#pragma unroll
      for (int j = 0; j < 8; ++j) p[j] = q[j];
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) z = Da(z, p[j]);
  }
  if (kMode == 1 && threadIdx.x < 64) {  // products precomputed (no loads): chain only
    double p[8];
    for (int j = 0; j < 8; ++j) p[j] = 1.0 + j * 1e-3 + threadIdx.x;
    for (unsigned b = 0; b < n / 8; ++b) {
#pragma unroll
      for (int j = 0; j < 8; ++j) z = Da(z, p[j]);
    }
  }
  if (kMode == 2 && threadIdx.x < 32) {  // 2 chains per thread (both units), one warp
    const double2* w0 = reinterpret_cast<const double2*>(w);
    const double2* w1 = reinterpret_cast<const double2*>(w + n);
    const double2* a2 = reinterpret_cast<const double2*>(x + threadIdx.x * (n + 2));
    double z1 = 0.5;
    for (unsigned i = 0; i < n / 2; ++i) {
      const double2 a = a2[i], b0 = w0[i], b1 = w1[i];
      const double p0 = Dm(b0.x, a.x), p1 = Dm(b1.x, a.x), p2 = Dm(b0.y, a.y), p3 = Dm(b1.y, a.y);
      z = Da(z, p0); z1 = Da(z1, p1); z = Da(z, p2); z1 = Da(z1, p3);
    }
    z += z1;
  }
  if (kMode == 3 && threadIdx.x < 64) {  // register-resident w, x streams: DMUL+DADD per element
    double a = 1.0 + threadIdx.x * 1e-3, b = 2.0;
    for (unsigned i = 0; i < n; ++i) { z = Da(z, Dm(a, b)); a = Da(a, 1e-9); }
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
  const size_t smem = (2 * n + 32 * (n + 2)) * 8;
  long long h;
  auto run = [&](auto kern, const char* name, int threads) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<1, threads, smem>>>(o, c, n); kern<<<1, threads, smem>>>(o, c, n);
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-52s %7lld cycles  %.2f per element  (%s)\n", name, h, double(h) / n, cudaGetErrorString(cudaGetLastError()));
  };
  run(k<0>, "pipelined double2 blocks of 8, 64 threads", 384);
  run(k<1>, "DADD chain only (products in regs), 64 threads", 384);
  run(k<2>, "2 chains/thread, 1 warp", 384);
  run(k<3>, "DMUL->DADD dependent-ish (regs), 64 threads", 384);
  return 0;
}
