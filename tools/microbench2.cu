// microbench2.cu — per-SM throughput (12 warps, 8 independent streams per thread) of
// F2F.F64.F32, DADD, DMUL, FFMA and an integer float->double bit conversion. Tool only.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double f2d_bits(float f) {
  const unsigned b = __float_as_uint(f);
  const unsigned mag = b & 0x7fffffffu;
  const unsigned hi = mag ? ((b & 0x80000000u) | ((mag >> 3) + (896u << 20))) : (b & 0x80000000u);
  return __hiloint2double(static_cast<int>(hi), static_cast<int>(b << 29));
}

template <int kOp>
__global__ void thr(double* out, long long* cyc, int n, float seed) {
  double d[8];
  float f[8];
  for (int k = 0; k < 8; ++k) { d[k] = seed + k + threadIdx.x; f[k] = seed * (k + 1) + threadIdx.x; }
  __syncthreads();
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      if (kOp == 0) d[k] += (double)f[k];                 // F2F + DADD
      if (kOp == 1) d[k] = __dadd_rn(d[k], 1.0000001);
      if (kOp == 2) d[k] = __dmul_rn(d[k], 1.0000001);
      if (kOp == 3) f[k] = __fmaf_rn(f[k], 1.0000001f, 0.5f);
      if (kOp == 4) d[k] = __dadd_rn(d[k], f2d_bits(f[k]));  // int conversion + DADD
    }
    if (kOp == 0 || kOp == 4) {
#pragma unroll
      for (int k = 0; k < 8; ++k) f[k] = __int_as_float(__float_as_int(f[k]) ^ 1);
    }
  }
  __syncthreads();
  long long t1 = clock64();
  double s = 0;
  for (int k = 0; k < 8; ++k) s += d[k] + f[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

template <int kOp>
void run(const char* name, int n, int threads) {
  double* o; long long* c;
  cudaMalloc(&o, 4096 * 8); cudaMalloc(&c, 8);
  thr<kOp><<<1, threads>>>(o, c, n, 1.5f);
  thr<kOp><<<1, threads>>>(o, c, n, 1.5f);
  long long h = 0;
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  const double ops = double(n) * 8 * threads;
  printf("%-34s threads=%4d  %.2f ops/cycle/SM\n", name, threads, ops / double(h));
  cudaFree(o); cudaFree(c);
}

int main() {
  const int n = 4096;
  for (int t : {64, 384}) {
    run<0>("F2F.F64.F32 + DADD", n, t);
    run<1>("DADD", n, t);
    run<2>("DMUL", n, t);
    run<3>("FFMA", n, t);
    run<4>("int f2d + DADD", n, t);
  }
  return 0;
}
