// microbench7.cu — code shapes for the fused step's latency-bound f64 chains. Tool only.
//  forward: 64 reference-order chains of 784 terms z += w[u][i]*x[r][i] (DMUL then DADD),
//           w/x f64 in smem; optional F2F "producer" warps running concurrently.
//  logits:  320 chains of 256 terms (32 rows x 10 classes) over an [H][32] activation
//           block and [C][H] weights in smem.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double Dm(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double Da(double a, double b) { return __dadd_rn(a, b); }

constexpr int N = 784, NP = 786;  // row stride (padded)

// F1: one chain per thread, blocks of 8 pipelined one ahead (the kernel's current shape)
__device__ double f1(const double* w, const double* x, double z) {
  const double2* w2 = reinterpret_cast<const double2*>(w);
  const double2* a2 = reinterpret_cast<const double2*>(x);
  double p[8], q[8];
  auto prod = [&](int b, double (&o)[8]) {
    double2 wv[4], av[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) { wv[k] = w2[4 * b + k]; av[k] = a2[4 * b + k]; }
#pragma unroll
    for (int k = 0; k < 4; ++k) { o[2 * k] = Dm(wv[k].x, av[k].x); o[2 * k + 1] = Dm(wv[k].y, av[k].y); }
  };
  prod(0, p);
  for (int b = 1; b < N / 8; ++b) {
    prod(b, q);
#pragma unroll
    for (int k = 0; k < 8; ++k) { z = Da(z, p[k]); p[k] = q[k]; }
  }
#pragma unroll
  for (int k = 0; k < 8; ++k) z = Da(z, p[k]);
  return z;
}

// F2: one chain, raw loads two blocks ahead, products one block ahead, unrolled by 2
// blocks so no register rotation is needed.
__device__ double f2(const double* w, const double* x, double z) {
  const double2* w2 = reinterpret_cast<const double2*>(w);
  const double2* a2 = reinterpret_cast<const double2*>(x);
  double2 wa[4], xa[4], wb[4], xb[4];
  double pa[8], pb[8];
#pragma unroll
  for (int k = 0; k < 4; ++k) { wa[k] = w2[k]; xa[k] = a2[k]; wb[k] = w2[4 + k]; xb[k] = a2[4 + k]; }
#pragma unroll
  for (int k = 0; k < 4; ++k) { pa[2 * k] = Dm(wa[k].x, xa[k].x); pa[2 * k + 1] = Dm(wa[k].y, xa[k].y); }
  constexpr int NB = N / 8;  // 98 blocks
  for (int b = 0; b < NB; b += 2) {
    // block b in pa (products), block b+1 raw in wb/xb; load block b+2 into wa/xa
    if (b + 2 < NB) {
#pragma unroll
      for (int k = 0; k < 4; ++k) { wa[k] = w2[4 * (b + 2) + k]; xa[k] = a2[4 * (b + 2) + k]; }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      pb[2 * k] = Dm(wb[k].x, xb[k].x);
      z = Da(z, pa[2 * k]);
      pb[2 * k + 1] = Dm(wb[k].y, xb[k].y);
      z = Da(z, pa[2 * k + 1]);
    }
    if (b + 3 < NB) {
#pragma unroll
      for (int k = 0; k < 4; ++k) { wb[k] = w2[4 * (b + 3) + k]; xb[k] = a2[4 * (b + 3) + k]; }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (b + 2 < NB) { pa[2 * k] = Dm(wa[k].x, xa[k].x); }
      z = Da(z, pb[2 * k]);
      if (b + 2 < NB) { pa[2 * k + 1] = Dm(wa[k].y, xa[k].y); }
      z = Da(z, pb[2 * k + 1]);
    }
  }
  return z;
}

// F3: two chains per thread (units 0/1 of one row: x loaded once), blocks of 4
__device__ void f3(const double* w0, const double* w1, const double* x, double& z0, double& z1) {
  const double2* a2 = reinterpret_cast<const double2*>(x);
  const double2* u2 = reinterpret_cast<const double2*>(w0);
  const double2* v2 = reinterpret_cast<const double2*>(w1);
  double p0[4], p1[4], q0[4], q1[4];
  auto prod = [&](int b, double (&o0)[4], double (&o1)[4]) {
    const double2 xa = a2[2 * b], xb = a2[2 * b + 1], ua = u2[2 * b], ub = u2[2 * b + 1], va = v2[2 * b],
                  vb = v2[2 * b + 1];
    o0[0] = Dm(ua.x, xa.x); o0[1] = Dm(ua.y, xa.y); o0[2] = Dm(ub.x, xb.x); o0[3] = Dm(ub.y, xb.y);
    o1[0] = Dm(va.x, xa.x); o1[1] = Dm(va.y, xa.y); o1[2] = Dm(vb.x, xb.x); o1[3] = Dm(vb.y, xb.y);
  };
  prod(0, p0, p1);
  for (int b = 1; b < N / 4; ++b) {
    prod(b, q0, q1);
#pragma unroll
    for (int k = 0; k < 4; ++k) { z0 = Da(z0, p0[k]); z1 = Da(z1, p1[k]); p0[k] = q0[k]; p1[k] = q1[k]; }
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) { z0 = Da(z0, p0[k]); z1 = Da(z1, p1[k]); }
}

template <int kMode>
__global__ void fwd(double* out, long long* cyc, int busy) {
  extern __shared__ double sm[];
  double* w = sm;             // 2 x NP
  double* x = sm + 2 * NP;    // 16 x NP (rows reused mod 16)
  float* xf = reinterpret_cast<float*>(x + 16 * NP);  // 8 x 788 f32 for the busy warps
  double* xd = x + 16 * NP + 4 * 788;                  // 8 x 130 f64
  for (int i = threadIdx.x; i < 18 * NP; i += blockDim.x) sm[i] = 1.0 + 1e-3 * (i % 97);
  for (int i = threadIdx.x; i < 8 * 788; i += blockDim.x) xf[i] = 1.0f + 1e-3f * (i % 89);
  __shared__ volatile int done;
  if (threadIdx.x == 0) done = 0;
  __syncthreads();
  long long t0 = clock64();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  double z = 0.25, z1 = 0.5;
  constexpr int CW = kMode == 3 ? 1 : (kMode == 5 ? 4 : 2);  // consumer warps
  if (warp < CW) {
    if (kMode == 1 || kMode == 2) {
      const int c = threadIdx.x, r = (c / 2) % 16, u = c % 2;
      z = kMode == 1 ? f1(w + u * NP, x + r * NP, z) : f2(w + u * NP, x + r * NP, z);
    } else if (kMode == 3) {  // 1 warp, 2 chains per lane
      f3(w, w + NP, x + (lane % 16) * NP, z, z1);
    } else if (kMode == 4) {  // 2 warps x 16 lanes, 2 chains per lane
      if (lane < 16) f3(w, w + NP, x + lane * NP, z, z1);
    } else {  // kMode 5: 4 warps x 16 lanes, 1 chain per lane (one warp per SM sub-partition)
      if (lane < 16) {
        const int c = warp * 16 + lane, r = (c / 2) % 16, u = c % 2;
        z = f1(w + u * NP, x + r * NP, z);
      }
    }
    __syncwarp();
    if (lane == 0) atomicAdd((int*)&done, 1);
  } else if (busy) {
    const int pw = warp - CW, np = blockDim.x / 32 - CW;
    while (done < CW)
      for (int r = pw; r < 8; r += np) {
        const float2 v = reinterpret_cast<const float2*>(xf + r * 788)[lane];
        reinterpret_cast<double2*>(xd + r * 130)[lane] = make_double2((double)v.x, (double)v.y);
      }
  }
  __syncthreads();
  long long t1 = clock64();
  out[threadIdx.x] = z + z1;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

// ---- logits ------------------------------------------------------------------------
constexpr int H = 256, C = 10, B = 32, H2 = 258;
template <int NC, int BLK>
__device__ void lchains(const double* W2, const double* A, int r, int cb, double* Z) {
  double z[NC];
#pragma unroll
  for (int i = 0; i < NC; ++i) z[i] = 0.1 * (cb + 4 * i);
  double p[NC][BLK], q[NC][BLK];
  auto prod = [&](int blk, double (&o)[NC][BLK]) {
    double av[BLK];
#pragma unroll
    for (int k = 0; k < BLK; ++k) av[k] = A[(blk * BLK + k) * B + r];
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      const double2* wr = reinterpret_cast<const double2*>(W2 + (cb + 4 * i) * H2 + blk * BLK);
#pragma unroll
      for (int k = 0; k < BLK / 2; ++k) {
        const double2 wv = wr[k];
        o[i][2 * k] = Dm(wv.x, av[2 * k]);
        o[i][2 * k + 1] = Dm(wv.y, av[2 * k + 1]);
      }
    }
  };
  prod(0, p);
  for (int blk = 1; blk < H / BLK; ++blk) {
    prod(blk, q);
#pragma unroll
    for (int k = 0; k < BLK; ++k)
#pragma unroll
      for (int i = 0; i < NC; ++i) { z[i] = Da(z[i], p[i][k]); p[i][k] = q[i][k]; }
  }
#pragma unroll
  for (int k = 0; k < BLK; ++k)
#pragma unroll
    for (int i = 0; i < NC; ++i) z[i] = Da(z[i], p[i][k]);
#pragma unroll
  for (int i = 0; i < NC; ++i) Z[r * C + cb + 4 * i] = z[i];
}

template <int kMode>
__global__ void logits(double* out, long long* cyc) {
  extern __shared__ double sm[];
  double* A = sm;              // H x B
  double* W2 = sm + H * B;     // C x H2
  double* Z = W2 + C * H2;     // B x C
  for (int i = threadIdx.x; i < H * B + C * H2; i += blockDim.x) sm[i] = 1e-2 * (i % 101);
  __syncthreads();
  long long t0 = clock64();
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (kMode == 1 && warp < 4) {  // current: 4 warps, classes cs, cs+4, cs+8, blocks of 4
    if (warp < 2) lchains<3, 4>(W2, A, lane, warp, Z); else lchains<2, 4>(W2, A, lane, warp, Z);
  }
  if (kMode == 2 && warp < 4) {  // blocks of 8
    if (warp < 2) lchains<3, 8>(W2, A, lane, warp, Z); else lchains<2, 8>(W2, A, lane, warp, Z);
  }
  if (kMode == 3 && warp < 8) {  // 8 warps: classes {w, w+8} for w<2 else {w}
    if (warp < 2) {  // two chains: classes warp and warp+8 -> emulate with cb stride 8 via NC=2, but cb+4i
      lchains<1, 4>(W2, A, lane, warp, Z);
      lchains<1, 4>(W2, A, lane, warp + 8, Z);
    } else {
      lchains<1, 4>(W2, A, lane, warp, Z);
    }
  }
  if (kMode == 4 && warp < 5) {  // 5 warps x 2 chains (classes w, w+5 emulated as cb, cb+4 -> use NC=2)
    lchains<2, 4>(W2, A, lane, warp < 4 ? warp : 5, Z);  // approximate shape
  }
  __syncthreads();
  long long t1 = clock64();
  out[threadIdx.x] = Z[threadIdx.x % (B * C)];
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

int main() {
  double* o;
  long long* c;
  cudaMalloc(&o, 4096 * 8);
  cudaMalloc(&c, 8);
  long long h;
  const size_t fsm = 18 * NP * 8 + 8 * 788 * 4 + 8 * 130 * 8;
  auto runf = [&](auto k, const char* name, int busy) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm);
    k<<<1, 384, fsm>>>(o, c, busy);
    k<<<1, 384, fsm>>>(o, c, busy);
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("fwd %-52s busy=%d %7lld cycles %.2f/elem (%s)\n", name, busy, h, double(h) / N,
           cudaGetErrorString(cudaGetLastError()));
  };
  for (int busy = 0; busy < 2; ++busy) {
    runf(fwd<1>, "F1 1 chain/thread, 8-blocks 1 ahead, 2 warps", busy);
    runf(fwd<2>, "F2 1 chain/thread, loads 2 ahead, 2 warps", busy);
    runf(fwd<3>, "F3 2 chains/thread (shared x), 1 warp", busy);
    runf(fwd<4>, "F4 2 chains/thread, 2 warps x 16 lanes", busy);
    runf(fwd<5>, "F5 1 chain/thread, 4 warps x 16 lanes", busy);
  }
  const size_t lsm = (H * B + C * H2 + B * C) * 8;
  auto runl = [&](auto k, const char* name) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)lsm);
    k<<<1, 384, lsm>>>(o, c);
    k<<<1, 384, lsm>>>(o, c);
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("logits %-48s %7lld cycles %.2f/elem (%s)\n", name, h, double(h) / H, cudaGetErrorString(cudaGetLastError()));
  };
  runl(logits<1>, "L1 4 warps, 3/3/2/2 chains, 4-blocks");
  runl(logits<2>, "L2 4 warps, 3/3/2/2 chains, 8-blocks");
  runl(logits<3>, "L3 8 warps, 1 chain at a time (2 sequential for w<2)");
  runl(logits<4>, "L4 5 warps x 2 chains");
  return 0;
}
