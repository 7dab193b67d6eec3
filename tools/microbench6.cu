// microbench6.cu — does F2F.F64.F32 conversion work in other warps slow the
// reference-order f64 dot-product chains (784 long) of the fused forward? Tool only.
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
__device__ __forceinline__ double chain(const double* w, const double* x, unsigned n, double z) {
  const double2* w2 = reinterpret_cast<const double2*>(w);
  const double2* a2 = reinterpret_cast<const double2*>(x);
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
  return z;
}
// deeper: loads two blocks ahead via explicit register rotation
__device__ __forceinline__ double chain2(const double* w, const double* x, unsigned n, double z) {
  const double2* w2 = reinterpret_cast<const double2*>(w);
  const double2* a2 = reinterpret_cast<const double2*>(x);
  double2 wa[4], xa[4], wb[4], xb[4];
  double p[8];
#pragma unroll
  for (int k = 0; k < 4; ++k) { wa[k] = w2[k]; xa[k] = a2[k]; wb[k] = w2[4 + k]; xb[k] = a2[4 + k]; }
#pragma unroll
  for (int k = 0; k < 4; ++k) { p[2 * k] = Dm(wa[k].x, xa[k].x); p[2 * k + 1] = Dm(wa[k].y, xa[k].y); }
  const unsigned nb = n / 8;
  for (unsigned b = 0; b < nb; ++b) {
    // loads for block b+2 (into wa/xa, free since p holds block b products)
    if (b + 2 < nb) {
#pragma unroll
      for (int k = 0; k < 4; ++k) { wa[k] = w2[4 * (b + 2) + k]; xa[k] = a2[4 * (b + 2) + k]; }
    }
    double q[8];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      z = Da(z, p[2 * k]);
      q[2 * k] = Dm(wb[k].x, xb[k].x);
      z = Da(z, p[2 * k + 1]);
      q[2 * k + 1] = Dm(wb[k].y, xb[k].y);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) p[k] = q[k];
#pragma unroll
    for (int k = 0; k < 4; ++k) { wb[k] = wa[k]; xb[k] = xa[k]; }
  }
  return z;
}
template <int kMode, int kChainWarps, int kLanes>
__global__ void k(double* out, long long* cyc, unsigned n, int busy) {
  extern __shared__ double sm[];
  double* w = sm;                                      // 2 rows x n
  double* x = sm + 2 * n;                              // 16 rows x (n+2)
  float* xf = reinterpret_cast<float*>(x + 16 * (n + 2));  // 16 x (n+4) f32
  double* xd = x + 16 * (n + 2) + 8 * (n + 4);         // conversion target 16 x 130
  for (unsigned i = threadIdx.x; i < 2 * n + 16 * (n + 2); i += blockDim.x) sm[i] = 1.0 + 1e-3 * (i % 97);
  for (unsigned i = threadIdx.x; i < 16 * (n + 4); i += blockDim.x) xf[i] = 1.0f + 1e-3f * (i % 89);
  __syncthreads();
  __shared__ volatile int done;
  if (threadIdx.x == 0) done = 0;
  __syncthreads();
  long long t0 = clock64();
  double z = 0.25;
  const unsigned warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp < kChainWarps) {
    if (lane < kLanes) {
      const unsigned c = warp * kLanes + lane, r = (c / 2) % 16, u = c % 2;
      z = kMode == 0 ? chain(w + u * n, x + r * (n + 2), n, z) : chain2(w + u * n, x + r * (n + 2), n, z);
    }
    __syncwarp();
    if (lane == 0) atomicAdd((int*)&done, 1);
  } else if (busy == 1) {  // F2F producers: convert 128-col chunks repeatedly
    const unsigned pw = warp - kChainWarps, np = blockDim.x / 32 - kChainWarps;
    while (done < kChainWarps) {
      for (unsigned c0 = 0; c0 + 128 <= n; c0 += 128)
        for (unsigned r = pw; r < 16; r += np) {
          const float2 v = reinterpret_cast<const float2*>(xf + r * (n + 4) + c0)[lane];
          reinterpret_cast<double2*>(xd + r * 130)[lane] = make_double2((double)v.x, (double)v.y);
          const float2 v2 = reinterpret_cast<const float2*>(xf + r * (n + 4) + c0)[lane + 32];
          reinterpret_cast<double2*>(xd + r * 130)[lane + 32] = make_double2((double)v2.x, (double)v2.y);
        }
    }
  } else if (busy == 2) {  // integer + LDS/STS only
    const unsigned pw = warp - kChainWarps;
    unsigned acc = pw;
    while (done < kChainWarps) {
      for (unsigned r = 0; r < 16; ++r) {
        const float2 v = reinterpret_cast<const float2*>(xf + r * (n + 4))[lane];
        acc += __float_as_uint(v.x) ^ __float_as_uint(v.y);
        reinterpret_cast<float2*>(xd + r * 130)[lane] = v;
      }
    }
    if (acc == 12345) out[4095] = acc;
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
  const size_t smem = (2 * n + 16 * (n + 2)) * 8 + 16 * (n + 4) * 4 + 16 * 130 * 8;
  long long h;
  auto run = [&](auto kern, const char* name, int busy) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<1, 384, smem>>>(o, c, n, busy); kern<<<1, 384, smem>>>(o, c, n, busy);
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("%-58s busy=%d %7lld cycles  %.2f per element  (%s)\n", name, busy, h, double(h) / n,
           cudaGetErrorString(cudaGetLastError()));
  };
  for (int busy = 0; busy < 3; ++busy) {
    run(k<0, 2, 32>, "chain (pipelined 1 ahead), 2 warps x 32 lanes", busy);
    run(k<1, 2, 32>, "chain2 (loads 2 ahead), 2 warps x 32 lanes", busy);
    run(k<0, 4, 16>, "chain, 4 warps x 16 lanes", busy);
    run(k<1, 4, 16>, "chain2, 4 warps x 16 lanes", busy);
  }
  return 0;
}
