// microbench4.cu — isolates the cost of F2F.F64.F32 in the exact-order dot product.
// Variants over a 784-long chain per thread (64 threads = 2 warps, one CTA):
//  0: f32 w,x  -> 2x F2F + DMUL + DADD
//  1: f64 w, f32 x -> 1x F2F + DMUL + DADD
//  2: f64 w,x  -> DMUL + DADD
//  3: F2F throughput only (8 independent per iter, int xor sink), 384 threads
#include <cstdio>
#include <cuda_runtime.h>
template <int kMode>
__global__ void k(double* out, long long* cyc, unsigned n) {
  extern __shared__ double smd[];
  double* wd = smd;                         // n doubles
  double* xd = smd + n;                     // 64 x n doubles? too big -> one row per thread pair
  float* wf = reinterpret_cast<float*>(smd + 2 * n);
  float* xf = wf + n;
  for (unsigned i = threadIdx.x; i < n; i += blockDim.x) {
    wd[i] = 1.0 + 1e-3 * (i % 97); xd[i] = 0.5 + 1e-3 * (i % 89);
    wf[i] = 1.0f + 1e-3f * (i % 97); xf[i] = 0.5f + 1e-3f * (i % 89);
  }
  __syncthreads();
  long long t0 = clock64();
  double z = threadIdx.x;
  unsigned sink = 0;
  if (kMode < 3) {
    if (threadIdx.x < 64) {
#pragma unroll 16
      for (unsigned i = 0; i < n; ++i) {
        double p;
        if (kMode == 0) p = __dmul_rn((double)wf[i], (double)xf[i]);
        if (kMode == 1) p = __dmul_rn(wd[i], (double)xf[i]);
        if (kMode == 2) p = __dmul_rn(wd[i], xd[i]);
        z = __dadd_rn(z, p);
      }
    }
  } else {
    float f[8];
    for (int j = 0; j < 8; ++j) f[j] = threadIdx.x + j;
    for (unsigned i = 0; i < n; ++i) {
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const double d = (double)f[j];
        sink ^= __double2hiint(d);
        f[j] = __int_as_float(__float_as_int(f[j]) + 1);
      }
    }
  }
  __syncthreads();
  long long t1 = clock64();
  out[threadIdx.x] = z + sink;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}
int main() {
  const unsigned n = 784;
  double* o; long long* c;
  cudaMalloc(&o, 4096 * 8); cudaMalloc(&c, 8);
  const size_t smem = n * 8 * 2 + n * 4 * 2;
  long long h;
  auto run = [&](auto kern, const char* name, int threads, double per) {
    kern<<<1, threads, smem>>>(o, c, n); kern<<<1, threads, smem>>>(o, c, n);
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-40s %8lld cycles  %.2f per unit\n", name, h, double(h) / per);
  };
  run(k<0>, "f32 w,x: 2 F2F + DMUL + DADD (/elem)", 64, n);
  run(k<1>, "f64 w, f32 x: F2F + DMUL + DADD (/elem)", 64, n);
  run(k<2>, "f64 w,x: DMUL + DADD (/elem)", 64, n);
  run(k<3>, "F2F only, 384 thr (lanes/cycle)", 384, 1.0);
  printf("F2F lanes/cycle/SM = %.2f\n", double(n) * 8 * 384 / double(h));
  return 0;
}
