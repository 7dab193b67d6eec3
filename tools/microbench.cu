// microbench.cu — dependent-chain latency of the arithmetic the fused step relies on
// (DADD, DMUL, DFMA, FFMA, FADD, F2F.F64.F32), one warp, clock64 deltas. Tool only.
#include <cstdio>

#include <cuda_runtime.h>

template <int kOp>
__global__ void chain(double* out, float* outf, long long* cyc, int n, double a, float af) {
  double x = a, y = a * 0.5;
  float xf = af;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    if (kOp == 0) x = __dadd_rn(x, y);
    if (kOp == 1) x = __dmul_rn(x, 1.0000001);
    if (kOp == 2) x = __fma_rn(x, 1.0000001, y);
    if (kOp == 3) xf = __fmaf_rn(xf, 1.0000001f, 0.5f);
    if (kOp == 4) xf = __fadd_rn(xf, 0.5f);
    if (kOp == 5) { x = __dadd_rn(x, (double)xf); xf = __fadd_rn(xf, 1.0f); }
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  outf[threadIdx.x] = xf;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

template <int kOp>
void run(const char* name, int n) {
  double* o;
  float* of;
  long long* c;
  cudaMalloc(&o, 1024 * 8);
  cudaMalloc(&of, 1024 * 4);
  cudaMalloc(&c, 8);
  chain<kOp><<<1, 32>>>(o, of, c, n, 1.0, 1.0f);
  chain<kOp><<<1, 32>>>(o, of, c, n, 1.0, 1.0f);
  long long h = 0;
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("%-28s %.2f cycles/op\n", name, double(h) / n);
  cudaFree(o);
  cudaFree(of);
  cudaFree(c);
}

int main() {
  const int n = 1 << 14;
  run<0>("DADD dependent", n);
  run<1>("DMUL dependent", n);
  run<2>("DFMA dependent", n);
  run<3>("FFMA dependent", n);
  run<4>("FADD dependent", n);
  run<5>("DADD(F2F) + FADD", n);
  return 0;
}
