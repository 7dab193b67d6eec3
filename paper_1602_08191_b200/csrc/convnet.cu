// convnet.cu — cifar10_quick (model kind 2) loss_and_grad / predict on the B200.
//
// NOT IN THE REFERENCE: the reference ships only softmax regression
// and tanh MLPs. This network follows the reference's conventions (flat per-layer
// W[out x fan_in] + b[out] layout, U(+-1/sqrt(fan_in)) init, mean softmax cross-entropy,
// gradient = batch sum * (1/b)) so it plugs into the same engine, exchanger and
// simulator. Parity is against the f64 CPU restatement oracle/ds_oracle_cnn.c (itself
// gated by central differences); arithmetic here is f32 with FMA, so the bar is a stated
// tolerance, not bit-exactness.
//
// Layout: activations NCHW f32 in the workspace, batch rows = CHW 3x32x32 samples.
//   conv1 5x5 3->32 p2 -> MAX 3x3/2 -> relu -> conv2 5x5 32->32 p2 -> relu -> AVE 3x3/2
//   -> conv3 5x5 32->64 p2 -> relu -> AVE 3x3/2 -> ip1 1024->64 -> ip2 64->C -> softmax
// Every reduction (weight gradients over the batch, pooling backward) is a fixed-order
// gather, never an atomic, so results are deterministic run to run.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>

#include "conv_tc.cuh"
#include "ds_common.cuh"
#include "model.cuh"

namespace dsb {
namespace {


__device__ __forceinline__ uint32_t pooled(uint32_t H) { return (H - 3 + 1) / 2 + 1; }  // ceil((H-3)/2)+1

// ---- 5x5 pad-2 stride-1 convolution (also used for backward-data with flipped,
// transposed weights). One CTA = one sample x COB output channels; a thread owns PPT
// consecutive pixels of a row for all COB channels over a 1/KS slice of the input
// channels (the KS partial sums are combined in a fixed order through smem). The padded
// input planes and the CTA's weights (transposed to [k][COB] so one LDS.128 feeds 4
// channels) live in smem.
template <int CIN, int COUT, int H, int COB, int PPT, int KS>
__global__ void __launch_bounds__(H * H / PPT * KS) conv5_kernel(const float* __restrict__ in,
                                                                 const float* __restrict__ W,
                                                                 const float* __restrict__ bias,
                                                                 float* __restrict__ out, bool relu,
                                                                 const uint32_t* gate) {
  if (gate && *gate) return;
  constexpr int HP = H + 4, K = CIN * 25, NPT = H * H / PPT, NT = NPT * KS, CPK = CIN / KS;
  static_assert(CIN % KS == 0 && COB % 4 == 0, "conv5 tiling");
  extern __shared__ __align__(16) float sm[];
  float* xs = sm;                 // [CIN][HP][HP]
  float* ws = sm + CIN * HP * HP;  // [K][COB]
  const int n = blockIdx.x, co0 = blockIdx.y * COB, tid = threadIdx.x;
  const float* src = in + static_cast<size_t>(n) * CIN * H * H;
  for (int i = tid; i < CIN * HP * HP; i += NT) {
    const int c = i / (HP * HP), r = (i / HP) % HP, q = i % HP;
    const int y = r - 2, x = q - 2;
    xs[i] = (y >= 0 && y < H && x >= 0 && x < H) ? __ldg(src + (c * H + y) * H + x) : 0.0f;
  }
  for (int i = tid; i < K * COB; i += NT) {
    const int k = i / COB, c = i % COB;
    ws[i] = __ldg(W + static_cast<size_t>(co0 + c) * K + k);
  }
  __syncthreads();
  const int ks = tid / NPT, pt = tid % NPT;
  const int p0 = pt * PPT, h = p0 / H, w0 = p0 % H;
  float acc[COB][PPT];
#pragma unroll
  for (int c = 0; c < COB; ++c)
#pragma unroll
    for (int j = 0; j < PPT; ++j) acc[c][j] = 0.0f;
  for (int ci = ks * CPK; ci < (ks + 1) * CPK; ++ci) {
#pragma unroll
    for (int kh = 0; kh < 5; ++kh) {
      const float* xr = xs + (ci * HP + h + kh) * HP + w0;
      float xv[PPT + 4];
#pragma unroll
      for (int j = 0; j < PPT + 4; ++j) xv[j] = xr[j];
#pragma unroll
      for (int kw = 0; kw < 5; ++kw) {
        const float4* wv = reinterpret_cast<const float4*>(ws + ((ci * 5 + kh) * 5 + kw) * COB);
#pragma unroll
        for (int c4 = 0; c4 < COB / 4; ++c4) {
          const float4 wq = wv[c4];
#pragma unroll
          for (int j = 0; j < PPT; ++j) {
            acc[4 * c4 + 0][j] = fmaf(wq.x, xv[j + kw], acc[4 * c4 + 0][j]);
            acc[4 * c4 + 1][j] = fmaf(wq.y, xv[j + kw], acc[4 * c4 + 1][j]);
            acc[4 * c4 + 2][j] = fmaf(wq.z, xv[j + kw], acc[4 * c4 + 2][j]);
            acc[4 * c4 + 3][j] = fmaf(wq.w, xv[j + kw], acc[4 * c4 + 3][j]);
          }
        }
      }
    }
  }
  if constexpr (KS > 1) {  // combine the K-split partials (slice order) through smem
    __syncthreads();
    float* red = sm;  // [KS][COB][H*H], fits in the input planes
#pragma unroll
    for (int c = 0; c < COB; ++c)
#pragma unroll
      for (int j = 0; j < PPT; ++j) red[(ks * COB + c) * H * H + p0 + j] = acc[c][j];
    __syncthreads();
    if (ks != 0) return;
#pragma unroll
    for (int c = 0; c < COB; ++c)
#pragma unroll
      for (int j = 0; j < PPT; ++j) {
        float v = red[c * H * H + p0 + j];
        for (int k = 1; k < KS; ++k) v += red[(k * COB + c) * H * H + p0 + j];
        acc[c][j] = v;
      }
  }
  float* dst = out + static_cast<size_t>(n) * COUT * H * H;
#pragma unroll
  for (int c = 0; c < COB; ++c) {
    const float b = bias ? __ldg(bias + co0 + c) : 0.0f;
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      float v = acc[c][j] + b;
      if (relu) v = v > 0.0f ? v : 0.0f;
      dst[((co0 + c) * H + h) * H + w0 + j] = v;
    }
  }
}

template <int CIN, int COUT, int H, int COB, int PPT, int KS>
int launch_conv5(const float* in, const float* W, const float* b, float* out, uint32_t R, bool relu,
                 const uint32_t* gate, cudaStream_t s) {
  constexpr int HP = H + 4;
  static_assert(KS == 1 || CIN * HP * HP >= KS * COB * H * H, "K-split combine must fit in the input planes");
  const size_t smem = (static_cast<size_t>(CIN) * HP * HP + static_cast<size_t>(CIN) * 25 * COB) * sizeof(float);
  auto k = conv5_kernel<CIN, COUT, H, COB, PPT, KS>;
  static bool attr = false;  // per instantiation, once per process
  if (!attr) {
    DS_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    attr = true;
  }
  k<<<dim3(R, COUT / COB), H * H / PPT * KS, smem, s>>>(in, W, b, out, relu, gate);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

// Wt[ci][co][kh][kw] = W[co][ci][4-kh][4-kw]: backward-data is conv5 of dY with Wt.
__global__ void flip_transpose_kernel(const float* __restrict__ W, float* __restrict__ Wt, uint32_t cout,
                                      uint32_t cin, const uint32_t* gate) {
  if (gate && *gate) return;
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= cout * cin * 25) return;
  const uint32_t kk = i % 25, ci = (i / 25) % cin, co = i / (25 * cin);
  Wt[(static_cast<size_t>(ci) * cout + co) * 25 + (24 - kk)] = W[i];
}

// ---- pooling (3x3 stride 2, ceil mode, pad 0) ---------------------------------------
// pool1: MAX then relu1. arg = window offset (0..8) of the first maximum (Caffe strict >).
__global__ void maxpool_relu_kernel(const float* __restrict__ in, float* __restrict__ out, uint8_t* __restrict__ arg,
                                    uint32_t NC, uint32_t H, const uint32_t* gate) {
  if (gate && *gate) return;
  const uint32_t Ho = pooled(H), i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= NC * Ho * Ho) return;
  const uint32_t pw = i % Ho, ph = (i / Ho) % Ho, nc = i / (Ho * Ho);
  const uint32_t hs = 2 * ph, ws = 2 * pw, he = min(hs + 3, H), we = min(ws + 3, H);
  const float* p = in + static_cast<size_t>(nc) * H * H;
  float best = -INFINITY;
  uint32_t bi = 0;
  for (uint32_t h = hs; h < he; ++h)
    for (uint32_t w = ws; w < we; ++w) {
      const float v = p[h * H + w];
      if (v > best) best = v, bi = (h - hs) * 3 + (w - ws);
    }
  out[i] = best > 0.0f ? best : 0.0f;
  arg[i] = static_cast<uint8_t>(bi | (best > 0.0f ? 0x10u : 0u));  // bit 4: relu1 passed
}

__global__ void avepool_kernel(const float* __restrict__ in, float* __restrict__ out, uint32_t NC, uint32_t H,
                               const uint32_t* gate) {
  if (gate && *gate) return;
  const uint32_t Ho = pooled(H), i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= NC * Ho * Ho) return;
  const uint32_t pw = i % Ho, ph = (i / Ho) % Ho, nc = i / (Ho * Ho);
  const uint32_t hs = 2 * ph, ws = 2 * pw, he = min(hs + 3, H), we = min(ws + 3, H);
  const float* p = in + static_cast<size_t>(nc) * H * H;
  float s = 0.0f;
  for (uint32_t h = hs; h < he; ++h)
    for (uint32_t w = ws; w < we; ++w) s += p[h * H + w];
  out[i] = s / static_cast<float>((he - hs) * (we - ws));
}

// din[n][c][h][w] = sum over windows containing (h,w) of dout/size, times (act > 0) when
// `act` (the relu output feeding the pool) is given.
__global__ void avepool_bwd_kernel(const float* __restrict__ dout, const float* __restrict__ act,
                                   float* __restrict__ din, uint32_t NC, uint32_t H, const uint32_t* gate) {
  if (gate && *gate) return;
  const uint32_t Ho = pooled(H), i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= NC * H * H) return;
  const uint32_t w = i % H, h = (i / H) % H, nc = i / (H * H);
  float s = 0.0f;
  const uint32_t ph0 = h >= 2 ? (h - 1) / 2 : 0, ph1 = min(h / 2, Ho - 1);
  const uint32_t pw0 = w >= 2 ? (w - 1) / 2 : 0, pw1 = min(w / 2, Ho - 1);
  for (uint32_t ph = ph0; ph <= ph1; ++ph)
    for (uint32_t pw = pw0; pw <= pw1; ++pw) {
      const uint32_t hs = 2 * ph, ws = 2 * pw, he = min(hs + 3, H), we = min(ws + 3, H);
      s += dout[(static_cast<size_t>(nc) * Ho + ph) * Ho + pw] / static_cast<float>((he - hs) * (we - ws));
    }
  if (act && !(act[i] > 0.0f)) s = 0.0f;
  din[i] = s;
}

// dc1[n][c][h][w] = sum of dr1 over the windows whose (relu-passing) maximum is (h,w).
__global__ void maxpool_relu_bwd_kernel(const float* __restrict__ dout, const uint8_t* __restrict__ arg,
                                        float* __restrict__ din, uint32_t NC, uint32_t H, const uint32_t* gate) {
  if (gate && *gate) return;
  const uint32_t Ho = pooled(H), i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= NC * H * H) return;
  const uint32_t w = i % H, h = (i / H) % H, nc = i / (H * H);
  float s = 0.0f;
  const uint32_t ph0 = h >= 2 ? (h - 1) / 2 : 0, ph1 = min(h / 2, Ho - 1);
  const uint32_t pw0 = w >= 2 ? (w - 1) / 2 : 0, pw1 = min(w / 2, Ho - 1);
  for (uint32_t ph = ph0; ph <= ph1; ++ph)
    for (uint32_t pw = pw0; pw <= pw1; ++pw) {
      const size_t o = (static_cast<size_t>(nc) * Ho + ph) * Ho + pw;
      const uint32_t a = arg[o];
      if ((a & 0x10u) && (a & 0xfu) == (h - 2 * ph) * 3 + (w - 2 * pw)) s += dout[o];
    }
  din[i] = s;
}

// Even H (H = 2*Ho): one thread per 2x2 input block (ph, pw). Its pixels lie in windows
// (ph-1|ph) x (pw-1|pw) only, so the thread reads those <= 4 pooled values once and
// accumulates each pixel's contributions in ascending (ph, pw) order — the same sums, in
// the same order, as the per-pixel gathers above.
__global__ void maxpool_relu_bwd2_kernel(const float* __restrict__ dout, const uint8_t* __restrict__ arg,
                                         float* __restrict__ din, uint32_t NC, uint32_t Ho, const uint32_t* gate) {
  if (gate && *gate) return;
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= NC * Ho * Ho) return;
  const uint32_t pw = i % Ho, ph = (i / Ho) % Ho, nc = i / (Ho * Ho), H = 2 * Ho;
  float s[2][2] = {{0.f, 0.f}, {0.f, 0.f}};
#pragma unroll
  for (int dh = -1; dh <= 0; ++dh)
#pragma unroll
    for (int dw = -1; dw <= 0; ++dw) {
      const int wh = static_cast<int>(ph) + dh, ww = static_cast<int>(pw) + dw;
      if (wh < 0 || ww < 0) continue;
      const size_t o = (static_cast<size_t>(nc) * Ho + wh) * Ho + ww;
      const uint32_t a = arg[o];
      if (!(a & 0x10u)) continue;
      const int hh = 2 * wh + static_cast<int>((a & 0xfu) / 3) - 2 * static_cast<int>(ph);
      const int wc = 2 * ww + static_cast<int>((a & 0xfu) % 3) - 2 * static_cast<int>(pw);
      if (hh >= 0 && hh < 2 && wc >= 0 && wc < 2) s[hh][wc] += dout[o];
    }
  float* d = din + (static_cast<size_t>(nc) * H + 2 * ph) * H + 2 * pw;
  *reinterpret_cast<float2*>(d) = make_float2(s[0][0], s[0][1]);
  *reinterpret_cast<float2*>(d + H) = make_float2(s[1][0], s[1][1]);
}

__global__ void avepool_bwd2_kernel(const float* __restrict__ dout, const float* __restrict__ act,
                                    float* __restrict__ din, uint32_t NC, uint32_t Ho, const uint32_t* gate) {
  if (gate && *gate) return;
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= NC * Ho * Ho) return;
  const uint32_t pw = i % Ho, ph = (i / Ho) % Ho, nc = i / (Ho * Ho), H = 2 * Ho;
  float s[2][2] = {{0.f, 0.f}, {0.f, 0.f}};
#pragma unroll
  for (int dh = -1; dh <= 0; ++dh)
#pragma unroll
    for (int dw = -1; dw <= 0; ++dw) {
      const int wh = static_cast<int>(ph) + dh, ww = static_cast<int>(pw) + dw;
      if (wh < 0 || ww < 0) continue;
      const uint32_t hs = 2 * wh, ws = 2 * ww, he = min(hs + 3, H), we = min(ws + 3, H);
      const float v = dout[(static_cast<size_t>(nc) * Ho + wh) * Ho + ww] / static_cast<float>((he - hs) * (we - ws));
#pragma unroll
      for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b)
          if (dh == 0 || a == 0)      // window ph-1 reaches only row 2ph
            if (dw == 0 || b == 0) s[a][b] += v;
    }
  const size_t base = (static_cast<size_t>(nc) * H + 2 * ph) * H + 2 * pw;
  float o[2][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) o[a][b] = (act && !(act[base + a * H + b] > 0.0f)) ? 0.0f : s[a][b];
  *reinterpret_cast<float2*>(din + base) = make_float2(o[0][0], o[0][1]);
  *reinterpret_cast<float2*>(din + base + H) = make_float2(o[1][0], o[1][1]);
}

// ---- fully connected ---------------------------------------------------------------
// out[r][o] = b[o] + sum_i W[o][i] a[r][i]; CTA per row, KS-way split over i, fixed-order
// combine of the KS partials.
template <int KS>
__global__ void fc_fwd_kernel(const float* __restrict__ a, const float* __restrict__ W, const float* __restrict__ b,
                              float* __restrict__ out, uint32_t in, uint32_t nout, const uint32_t* gate) {
  if (gate && *gate) return;
  extern __shared__ float fs[];
  float* as = fs;          // [in]
  float* part = fs + in;   // [KS][nout]
  const uint32_t r = blockIdx.x;
  for (uint32_t i = threadIdx.x; i < in; i += blockDim.x) as[i] = a[static_cast<size_t>(r) * in + i];
  __syncthreads();
  for (uint32_t t = threadIdx.x; t < KS * nout; t += blockDim.x) {
    const uint32_t o = t % nout, k = t / nout;
    const uint32_t i0 = k * in / KS, i1 = (k + 1) * in / KS;
    const float* wr = W + static_cast<size_t>(o) * in;
    float s = 0.0f;
    for (uint32_t i = i0; i < i1; ++i) s = fmaf(__ldg(wr + i), as[i], s);
    part[k * nout + o] = s;
  }
  __syncthreads();
  for (uint32_t o = threadIdx.x; o < nout; o += blockDim.x) {
    float s = b[o];
    for (uint32_t k = 0; k < KS; ++k) s += part[k * nout + o];
    out[static_cast<size_t>(r) * nout + o] = s;
  }
}

// out[r][o] = b[o] + sum_i W[o][i] a[r][i] for 64 outputs, split over K: CTA = (16 rows,
// one 128-wide K slice), thread = (row, 4 outputs), 64-wide tiles staged in smem (the W
// tile is shared by the 16 rows); part[slice][r][o], summed in slice order by fc64_reduce.
constexpr uint32_t kFcSlice = 128;
__global__ void __launch_bounds__(256) fc64_fwd_kernel(const float* __restrict__ a, const float* __restrict__ W,
                                                       float* __restrict__ part, uint32_t R, uint32_t in,
                                                       const uint32_t* gate) {
  if (gate && *gate) return;
  __shared__ float as[16][65];
  __shared__ float ws[64][65];
  const uint32_t r0 = blockIdx.x * 16, tid = threadIdx.x, rl = tid >> 4, o4 = (tid & 15) * 4;
  const uint32_t klo = blockIdx.y * kFcSlice, khi = min(klo + kFcSlice, in);
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  for (uint32_t k0 = klo; k0 < khi; k0 += 64) {
    for (uint32_t t = tid; t < 16 * 64; t += 256) {
      const uint32_t r = t >> 6, k = t & 63;
      as[r][k] = (r0 + r < R && k0 + k < khi) ? a[static_cast<size_t>(r0 + r) * in + k0 + k] : 0.0f;
    }
    for (uint32_t t = tid; t < 64 * 64; t += 256) {
      const uint32_t o = t >> 6, k = t & 63;
      ws[o][k] = k0 + k < khi ? __ldg(W + static_cast<size_t>(o) * in + k0 + k) : 0.0f;
    }
    __syncthreads();
#pragma unroll 8
    for (uint32_t k = 0; k < 64; ++k) {
      const float x = as[rl][k];
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[j] = fmaf(ws[o4 + j][k], x, acc[j]);
    }
    __syncthreads();
  }
  if (r0 + rl < R)
#pragma unroll
    for (int j = 0; j < 4; ++j) part[(static_cast<size_t>(blockIdx.y) * R + r0 + rl) * 64 + o4 + j] = acc[j];
}

__global__ void fc64_reduce_kernel(const float* __restrict__ part, const float* __restrict__ b, float* __restrict__ out,
                                   uint32_t R, uint32_t nslice, const uint32_t* gate) {
  if (gate && *gate) return;
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= R * 64) return;
  float s = b[t & 63];
  for (uint32_t k = 0; k < nslice; ++k) s += part[static_cast<size_t>(k) * R * 64 + t];
  out[t] = s;
}

// dW[o][i] = inv_b * sum_r d[r][o] a[r][i]; db[o] = inv_b * sum_r d[r][o] (threads i == 0
// of each o also produce db). One thread per (o, i), rows in order.
__global__ void fc_bwd_w_kernel(const float* __restrict__ d, const float* __restrict__ a, float* __restrict__ gW,
                                float* __restrict__ gb, uint32_t R, uint32_t in, uint32_t nout, float inv_b,
                                uint32_t* flags, const uint32_t* gate) {
  if (gate && *gate) return;
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nout * in) return;
  const uint32_t o = t / in, i = t % in;
  float s = 0.0f;
  for (uint32_t r = 0; r < R; ++r) s = fmaf(d[static_cast<size_t>(r) * nout + o], a[static_cast<size_t>(r) * in + i], s);
  const float g = s * inv_b;
  if (!isfinite(g)) atomicOr(flags, DS_FLAG_GRAD_NONFINITE);
  gW[t] = g;
  if (i == 0) {
    float sb = 0.0f;
    for (uint32_t r = 0; r < R; ++r) sb += d[static_cast<size_t>(r) * nout + o];
    gb[o] = sb * inv_b;
  }
}

// da[r][i] = sum_o d[r][o] W[o][i]
__global__ void fc_bwd_a_kernel(const float* __restrict__ d, const float* __restrict__ W, float* __restrict__ da,
                                uint32_t R, uint32_t in, uint32_t nout, const uint32_t* gate) {
  if (gate && *gate) return;
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= R * in) return;
  const uint32_t r = t / in, i = t % in;
  float s = 0.0f;
  for (uint32_t o = 0; o < nout; ++o) s = fmaf(d[static_cast<size_t>(r) * nout + o], __ldg(W + static_cast<size_t>(o) * in + i), s);
  da[t] = s;
}

// ---- softmax cross-entropy ---------------------------------------------------------
// Per row: loss_r in f64 from the f32 logits (max-shifted LSE), delta = softmax - onehot.
__global__ void softmax_ce_kernel(const float* __restrict__ z, const uint32_t* __restrict__ y,
                                  const uint32_t* __restrict__ idx, uint32_t R, uint32_t C, double* __restrict__ loss_rows,
                                  float* __restrict__ delta, uint32_t* flags, const uint32_t* gate) {
  if (gate && *gate) return;
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  const uint32_t label = y[idx ? idx[r] : r];
  const float* zr = z + static_cast<size_t>(r) * C;
  double zmax = zr[0];
  for (uint32_t c = 1; c < C; ++c) zmax = zr[c] > zmax ? zr[c] : zmax;
  double sum = 0.0;
  for (uint32_t c = 0; c < C; ++c) sum += exp(static_cast<double>(zr[c]) - zmax);
  const double lse = zmax + log(sum);
  if (label >= C) {
    atomicOr(flags, DS_FLAG_LABEL_RANGE);
    loss_rows[r] = 0.0;
  } else {
    loss_rows[r] = lse - static_cast<double>(zr[label]);
  }
  if (delta)
    for (uint32_t c = 0; c < C; ++c)
      delta[static_cast<size_t>(r) * C + c] =
          static_cast<float>(exp(static_cast<double>(zr[c]) - lse) - (c == label ? 1.0 : 0.0));
}

// argmax of the logits (first maximum), hits against labels
__global__ void cnn_hits_kernel(const float* __restrict__ z, const uint32_t* __restrict__ y, uint32_t R, uint32_t C,
                                uint32_t* pred, unsigned long long* hits) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  const float* zr = z + static_cast<size_t>(r) * C;
  uint32_t best = 0;
  for (uint32_t c = 1; c < C; ++c)
    if (zr[c] > zr[best]) best = c;
  if (pred) pred[r] = best;
  if (hits && y && best == y[r]) atomicAdd(hits, 1ull);
}

// ---- convolution weight (and bias) gradients ----------------------------------------
// Partial sums over chunks of CHUNK samples: part[chunk][co][ci][25] and pb[chunk][co].
// Thread = (co in the CTA's CG group, ci, kh) with 5 kw accumulators and a sliding
// register window along w. xs holds the sample's padded input planes (row stride HP+1,
// plane stride odd: the (ci, kh) lanes of a warp land in different banks), dsm its dY
// planes. The bias partial of each co is a strided per-thread sum plus a fixed-order
// combine over the group's threads.
template <int CIN, int H, int CG, int CHUNK>
__global__ void __launch_bounds__(CG * CIN * 5) conv5_bwd_w_kernel(const float* __restrict__ in,
                                                                  const float* __restrict__ dout, float* __restrict__ part,
                                                                  float* __restrict__ pb, uint32_t R, uint32_t cout,
                                                                  const uint32_t* gate) {
  if (gate && *gate) return;
  constexpr int HP = H + 4, RS = HP + 1, PS = RS * HP + 1, NT = CG * CIN * 5, GT = CIN * 5;
  extern __shared__ __align__(16) float sm[];
  float* xs = sm;                   // [CIN][HP][RS] (plane stride PS)
  float* dsm = sm + CIN * PS;       // [CG][H][H]
  float* bred = dsm + CG * H * H;   // [NT]
  const int co0 = blockIdx.x * CG, chunk = blockIdx.y, tid = threadIdx.x;
  const int g = tid / GT, ci = (tid / 5) % CIN, kh = tid % 5, gl = tid % GT;
  float acc[5] = {0.f, 0.f, 0.f, 0.f, 0.f};
  float bacc = 0.0f;
  const uint32_t r0 = chunk * CHUNK, r1 = min(r0 + CHUNK, R);
  for (uint32_t n = r0; n < r1; ++n) {
    __syncthreads();
    const float* src = in + static_cast<size_t>(n) * CIN * H * H;
    for (int i = tid; i < CIN * HP * HP; i += NT) {
      const int c = i / (HP * HP), rr = (i / HP) % HP, q = i % HP;
      const int y = rr - 2, x = q - 2;
      xs[c * PS + rr * RS + q] = (y >= 0 && y < H && x >= 0 && x < H) ? __ldg(src + (c * H + y) * H + x) : 0.0f;
    }
    const float* dsrc = dout + (static_cast<size_t>(n) * cout + co0) * H * H;
    for (int i = tid; i < CG * H * H; i += NT) dsm[i] = __ldg(dsrc + i);
    __syncthreads();
    const float* dp = dsm + g * H * H;
    for (int p = gl; p < H * H; p += GT) bacc += dp[p];
    for (int h = 0; h < H; ++h) {
      const float* xr = xs + ci * PS + (h + kh) * RS;
      float win[5] = {xr[0], xr[1], xr[2], xr[3], 0.f};
#pragma unroll 4
      for (int w = 0; w < H; ++w) {
        win[4] = xr[w + 4];
        const float d = dp[h * H + w];
#pragma unroll
        for (int kw = 0; kw < 5; ++kw) acc[kw] = fmaf(d, win[kw], acc[kw]);
#pragma unroll
        for (int kw = 0; kw < 4; ++kw) win[kw] = win[kw + 1];
      }
    }
  }
  float* dst = part + (static_cast<size_t>(chunk) * cout + co0 + g) * CIN * 25 + ci * 25 + kh * 5;
#pragma unroll
  for (int kw = 0; kw < 5; ++kw) dst[kw] = acc[kw];
  bred[tid] = bacc;
  __syncthreads();
  if (gl == 0) {
    float b = 0.0f;
    for (int k = 0; k < GT; ++k) b += bred[g * GT + k];
    pb[static_cast<size_t>(chunk) * cout + co0 + g] = b;
  }
}

template <int CIN, int H, int CG, int CHUNK>
int launch_conv5_bwd_w(const float* in, const float* dout, float* part, float* pb, uint32_t R, uint32_t cout,
                       const uint32_t* gate, cudaStream_t s) {
  constexpr int HP = H + 4, PS = (HP + 1) * HP + 1;
  const size_t smem = (static_cast<size_t>(CIN) * PS + CG * H * H + CG * CIN * 5) * sizeof(float);
  auto k = conv5_bwd_w_kernel<CIN, H, CG, CHUNK>;
  static bool attr = false;
  if (!attr) {
    DS_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    attr = true;
  }
  const uint32_t nch = (R + CHUNK - 1) / CHUNK;
  k<<<dim3(cout / CG, nch), CG * CIN * 5, smem, s>>>(in, dout, part, pb, R, cout, gate);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

// grad[j] = inv_b * sum_chunks part[chunk][j] (chunk order), j < n
__global__ void reduce_parts_kernel(const float* __restrict__ part, uint32_t nchunks, uint64_t n, float* __restrict__ grad,
                                    float inv_b, uint32_t* flags, const uint32_t* gate) {
  if (gate && *gate) return;
  const uint64_t j = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= n) return;
  float s = 0.0f;
  for (uint32_t c = 0; c < nchunks; ++c) s += part[static_cast<uint64_t>(c) * n + j];
  const float g = s * inv_b;
  if (!isfinite(g)) atomicOr(flags, DS_FLAG_GRAD_NONFINITE);
  grad[j] = g;
}

__global__ void gather_cnn_rows_kernel(const float* __restrict__ X, const uint32_t* __restrict__ idx, uint32_t R,
                                       float* __restrict__ dst, const uint32_t* gate) {
  if (gate && *gate) return;
  const uint32_t r = blockIdx.x;
  const float4* s = reinterpret_cast<const float4*>(X + static_cast<size_t>(idx[r]) * 3072);
  float4* d = reinterpret_cast<float4*>(dst + static_cast<size_t>(r) * 3072);
  for (uint32_t q = threadIdx.x; q < 768; q += blockDim.x) d[q] = __ldg(s + q);
}

__global__ void loss_mean_kernel(const double* __restrict__ loss_rows, uint32_t R, bool grad_mode, double* loss_out,
                                 uint32_t* flags, const uint32_t* gate) {
  if (gate && *gate) return;
  double s = 0.0;
  for (uint32_t r = 0; r < R; ++r) s += loss_rows[r];
  const double loss = grad_mode ? s * (1.0 / static_cast<double>(R)) : s / static_cast<double>(R);
  *loss_out = loss;
  if (!isfinite(loss)) atomicOr(flags, DS_FLAG_LOSS_NONFINITE);
}

// Workspace carve-up (floats unless noted), for R rows.
struct CnnWs {
  float *x0, *c1, *p1, *c2, *p2, *c3, *p3, *h1, *z;       // forward
  float *dz, *dh1, *dp3, *dc3, *dp2, *dc2, *dr1, *dc1;    // backward
  float *wt2, *wt3, *part, *pb;                            // flipped weights, partial dW / db
  float* wpk;                                              // tcgen05 packed weight chunks
  float* fcpart;                                           // ip1 split-K partials
  uint8_t* arg1;
  double* loss_rows;
  size_t bytes;
};

CnnWs carve(uint32_t R, uint32_t C, void* base) {
  CnnWs w{};
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off += (bytes + 255) & ~static_cast<size_t>(255);
    return base ? static_cast<char*>(base) + o : nullptr;
  };
  const size_t f = sizeof(float);
  w.x0 = reinterpret_cast<float*>(take(R * 3072 * f));
  w.c1 = reinterpret_cast<float*>(take(R * 32768 * f));
  w.p1 = reinterpret_cast<float*>(take(R * 8192 * f));
  w.c2 = reinterpret_cast<float*>(take(R * 8192 * f));
  w.p2 = reinterpret_cast<float*>(take(R * 2048 * f));
  w.c3 = reinterpret_cast<float*>(take(R * 4096 * f));
  w.p3 = reinterpret_cast<float*>(take(R * 1024 * f));
  w.h1 = reinterpret_cast<float*>(take(R * 64 * f));
  w.z = reinterpret_cast<float*>(take(static_cast<size_t>(R) * C * f));
  w.dz = reinterpret_cast<float*>(take(static_cast<size_t>(R) * C * f));
  w.dh1 = reinterpret_cast<float*>(take(R * 64 * f));
  w.dp3 = reinterpret_cast<float*>(take(R * 1024 * f));
  w.dc3 = reinterpret_cast<float*>(take(R * 4096 * f));
  w.dp2 = reinterpret_cast<float*>(take(R * 2048 * f));
  w.dc2 = reinterpret_cast<float*>(take(R * 8192 * f));
  w.dr1 = reinterpret_cast<float*>(take(R * 8192 * f));
  w.dc1 = reinterpret_cast<float*>(take(R * 32768 * f));
  w.wt2 = reinterpret_cast<float*>(take(32 * 800 * f));
  w.wt3 = reinterpret_cast<float*>(take(64 * 800 * f));
  // partials: conv1 per sample (100 x 2400), conv2/3 per 4 samples (25 x 51200), or the
  // tensor-core weight-gradient splits
  w.part = reinterpret_cast<float*>(take(std::max<size_t>(
      std::max<size_t>(std::max<size_t>(R * 2400, conv5_wgrad_part_floats(3, 32, R, 1)), ((R + 3) / 4) * 64 * 800),
      std::max<size_t>(conv5_wgrad_part_floats(32, 32, R, 4), conv5_wgrad_part_floats(32, 64, R, 4))) * f));
  w.pb = reinterpret_cast<float*>(take(R * 64 * f));
  w.wpk = reinterpret_cast<float*>(take(conv5_tc_wpk_floats(64, 32) * f));
  w.fcpart = reinterpret_cast<float*>(take(static_cast<size_t>(R) * 64 * (1024 / kFcSlice) * f));  // largest: 64x25 -> 32 (= 32x25 -> 64)
  w.arg1 = reinterpret_cast<uint8_t*>(take(R * 8192));
  w.loss_rows = reinterpret_cast<double*>(take(R * sizeof(double)));
  w.bytes = off;
  return w;
}

unsigned blocks(uint64_t n, unsigned t = 256) { return static_cast<unsigned>((n + t - 1) / t); }

// Convolutions run as tcgen05 implicit GEMMs (tf32 operands, f32 accumulation) unless
// DS_CNN_FFMA=1 selects the f32 CUDA-core kernels (a precision mode for parity checks).
bool use_tensor_cores() {
  const char* e = std::getenv("DS_CNN_FFMA");
  return !(e && e[0] == '1');
}

}  // namespace

uint64_t cnn_workspace_bytes(const ModelInfo& m, uint32_t R) { return carve(R, m.n_classes, nullptr).bytes; }

// Forward to the logits in ws.z (rows gathered through idx when given).
static int cnn_forward(const ModelInfo& m, const float* P, const float* X, const uint32_t* idx, uint32_t R,
                       CnnWs& w, const uint32_t* gate, cudaStream_t s) {
  const LayerInfo* L = m.layers.data();
  const float* x0 = X;
  if (idx) {
    gather_cnn_rows_kernel<<<R, 256, 0, s>>>(X, idx, R, w.x0, gate);
    DS_CUDA_TRY(cudaGetLastError());
    x0 = w.x0;
  }
  const bool tcores = use_tensor_cores();
  if (tcores)
    DS_TRY((launch_conv5_tc<3, 32, 32>(x0, P + L[0].w_off, false, w.wpk, P + L[0].b_off, w.c1, R, false, gate, s)));
  else
    DS_TRY((launch_conv5<3, 32, 32, 16, 4, 1>(x0, P + L[0].w_off, P + L[0].b_off, w.c1, R, false, gate, s)));
  maxpool_relu_kernel<<<blocks(R * 32 * 256), 256, 0, s>>>(w.c1, w.p1, w.arg1, R * 32, 32, gate);
  if (tcores)
    DS_TRY((launch_conv5_tc<32, 32, 16>(w.p1, P + L[1].w_off, false, w.wpk, P + L[1].b_off, w.c2, R, true, gate, s)));
  else
    DS_TRY((launch_conv5<32, 32, 16, 16, 2, 2>(w.p1, P + L[1].w_off, P + L[1].b_off, w.c2, R, true, gate, s)));
  avepool_kernel<<<blocks(R * 32 * 64), 256, 0, s>>>(w.c2, w.p2, R * 32, 16, gate);
  if (tcores)
    DS_TRY((launch_conv5_tc<32, 64, 8>(w.p2, P + L[2].w_off, false, w.wpk, P + L[2].b_off, w.c3, R, true, gate, s)));
  else
    DS_TRY((launch_conv5<32, 64, 8, 16, 1, 4>(w.p2, P + L[2].w_off, P + L[2].b_off, w.c3, R, true, gate, s)));
  avepool_kernel<<<blocks(R * 64 * 16), 256, 0, s>>>(w.c3, w.p3, R * 64, 8, gate);
  fc64_fwd_kernel<<<dim3((R + 15) / 16, 1024 / kFcSlice), 256, 0, s>>>(w.p3, P + L[3].w_off, w.fcpart, R, 1024, gate);
  fc64_reduce_kernel<<<blocks(R * 64), 256, 0, s>>>(w.fcpart, P + L[3].b_off, w.h1, R, 1024 / kFcSlice, gate);
  fc_fwd_kernel<1><<<R, 64, (64 + m.n_classes) * sizeof(float), s>>>(w.h1, P + L[4].w_off, P + L[4].b_off, w.z, 64,
                                                                     m.n_classes, gate);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

namespace {
// Side stream per device for the weight-gradient chain (tensor-core path): it forks off
// the main stream after each layer's output gradient and runs beside the data-gradient
// chain; the event edges are captured into the engine's CUDA graph as parallel branches.
struct CnnSide {
  cudaStream_t s = nullptr;
  cudaEvent_t ev[8] = {};
};
int cnn_side(CnnSide** out) {
  thread_local CnnSide sides[64];  // per host thread: events are not shared across threads
  int dev = 0;
  DS_CUDA_TRY(cudaGetDevice(&dev));
  CnnSide& sd = sides[dev & 63];
  if (!sd.s) {
    DS_CUDA_TRY(cudaStreamCreateWithFlags(&sd.s, cudaStreamNonBlocking));
    for (auto& e : sd.ev) DS_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  *out = &sd;
  return DS_OK;
}
int cnn_edge(cudaStream_t from, cudaStream_t to, cudaEvent_t ev) {
  DS_CUDA_TRY(cudaEventRecord(ev, from));
  DS_CUDA_TRY(cudaStreamWaitEvent(to, ev, 0));
  return DS_OK;
}
}  // namespace

int launch_cnn_loss_and_grad(const ModelInfo& m, const float* P, const float* X, const uint32_t* idx, const uint32_t* y,
                             uint32_t R, float* grad, double* loss_out, void* ws_base, uint32_t* flags,
                             const uint32_t* gate, cudaStream_t s) {
  CnnWs w = carve(R, m.n_classes, ws_base);
  const LayerInfo* L = m.layers.data();
  const uint32_t C = m.n_classes;
  DS_TRY(cnn_forward(m, P, X, idx, R, w, gate, s));
  softmax_ce_kernel<<<blocks(R, 128), 128, 0, s>>>(w.z, y, idx, R, C, w.loss_rows, grad ? w.dz : nullptr, flags, gate);
  loss_mean_kernel<<<1, 1, 0, s>>>(w.loss_rows, R, grad != nullptr, loss_out, flags, gate);
  DS_CUDA_TRY(cudaGetLastError());
  if (!grad) return DS_OK;
  const float inv_b = static_cast<float>(1.0 / static_cast<double>(R));
  const uint32_t nch4 = (R + 3) / 4;
  if (use_tensor_cores()) {  // two streams: weight gradients beside the data-gradient chain
    CnnSide* sd = nullptr;
    DS_TRY(cnn_side(&sd));
    const cudaStream_t s2 = sd->s;
    DS_TRY(cnn_edge(s, s2, sd->ev[0]));
    fc_bwd_w_kernel<<<blocks(C * 64), 256, 0, s2>>>(w.dz, w.h1, grad + L[4].w_off, grad + L[4].b_off, R, 64, C, inv_b,
                                                    flags, gate);
    fc_bwd_a_kernel<<<blocks(R * 64), 256, 0, s>>>(w.dz, P + L[4].w_off, w.dh1, R, 64, C, gate);
    DS_TRY(cnn_edge(s, s2, sd->ev[1]));
    fc_bwd_w_kernel<<<blocks(64 * 1024), 256, 0, s2>>>(w.dh1, w.p3, grad + L[3].w_off, grad + L[3].b_off, R, 1024, 64,
                                                       inv_b, flags, gate);
    fc_bwd_a_kernel<<<blocks(R * 1024), 256, 0, s>>>(w.dh1, P + L[3].w_off, w.dp3, R, 1024, 64, gate);
    avepool_bwd2_kernel<<<blocks(R * 64 * 16), 256, 0, s>>>(w.dp3, w.c3, w.dc3, R * 64, 4, gate);
    DS_CUDA_TRY(cudaGetLastError());
    DS_TRY(cnn_edge(s, s2, sd->ev[2]));
    DS_TRY((launch_conv5_wgrad_tc<32, 64, 8, 4>(w.p2, w.dc3, w.part, grad + L[2].w_off, grad + L[2].b_off, R, inv_b,
                                                flags, gate, s2)));
    DS_TRY((launch_conv5_tc<64, 32, 8>(w.dc3, P + L[2].w_off, true, w.wpk, nullptr, w.dp2, R, false, gate, s)));
    avepool_bwd2_kernel<<<blocks(R * 32 * 64), 256, 0, s>>>(w.dp2, w.c2, w.dc2, R * 32, 8, gate);
    DS_CUDA_TRY(cudaGetLastError());
    DS_TRY(cnn_edge(s, s2, sd->ev[3]));
    DS_TRY((launch_conv5_wgrad_tc<32, 32, 16, 4>(w.p1, w.dc2, w.part, grad + L[1].w_off, grad + L[1].b_off, R, inv_b,
                                                 flags, gate, s2)));
    DS_TRY((launch_conv5_tc<32, 32, 16>(w.dc2, P + L[1].w_off, true, w.wpk, nullptr, w.dr1, R, false, gate, s)));
    maxpool_relu_bwd2_kernel<<<blocks(R * 32 * 256), 256, 0, s>>>(w.dr1, w.arg1, w.dc1, R * 32, 16, gate);
    DS_CUDA_TRY(cudaGetLastError());
    DS_TRY(cnn_edge(s, s2, sd->ev[4]));
    DS_TRY((launch_conv5_wgrad_tc<3, 32, 32, 1>(idx ? w.x0 : X, w.dc1, w.part, grad + L[0].w_off, grad + L[0].b_off, R,
                                                inv_b, flags, gate, s2)));
    DS_TRY(cnn_edge(s2, s, sd->ev[5]));  // join: all gradients written
    DS_CUDA_TRY(cudaGetLastError());
    return DS_OK;
  }
  // ip2, ip1
  fc_bwd_w_kernel<<<blocks(C * 64), 256, 0, s>>>(w.dz, w.h1, grad + L[4].w_off, grad + L[4].b_off, R, 64, C, inv_b,
                                                 flags, gate);
  fc_bwd_a_kernel<<<blocks(R * 64), 256, 0, s>>>(w.dz, P + L[4].w_off, w.dh1, R, 64, C, gate);
  fc_bwd_w_kernel<<<blocks(64 * 1024), 256, 0, s>>>(w.dh1, w.p3, grad + L[3].w_off, grad + L[3].b_off, R, 1024, 64,
                                                    inv_b, flags, gate);
  fc_bwd_a_kernel<<<blocks(R * 1024), 256, 0, s>>>(w.dh1, P + L[3].w_off, w.dp3, R, 1024, 64, gate);
  // pool3 -> relu3 -> conv3
  avepool_bwd2_kernel<<<blocks(R * 64 * 16), 256, 0, s>>>(w.dp3, w.c3, w.dc3, R * 64, 4, gate);
  DS_CUDA_TRY(cudaGetLastError());
  if (use_tensor_cores()) {
    DS_TRY((launch_conv5_wgrad_tc<32, 64, 8, 4>(w.p2, w.dc3, w.part, grad + L[2].w_off, grad + L[2].b_off, R, inv_b,
                                                flags, gate, s)));
  } else {
    DS_TRY((launch_conv5_bwd_w<32, 8, 2, 4>(w.p2, w.dc3, w.part, w.pb, R, 64, gate, s)));
    reduce_parts_kernel<<<blocks(64 * 800), 256, 0, s>>>(w.part, nch4, 64 * 800, grad + L[2].w_off, inv_b, flags, gate);
    reduce_parts_kernel<<<1, 64, 0, s>>>(w.pb, nch4, 64, grad + L[2].b_off, inv_b, flags, gate);
  }
  if (!use_tensor_cores())
    flip_transpose_kernel<<<blocks(64 * 800), 256, 0, s>>>(P + L[2].w_off, w.wt3, 64, 32, gate);
  DS_CUDA_TRY(cudaGetLastError());
  if (use_tensor_cores())
    DS_TRY((launch_conv5_tc<64, 32, 8>(w.dc3, P + L[2].w_off, true, w.wpk, nullptr, w.dp2, R, false, gate, s)));
  else
    DS_TRY((launch_conv5<64, 32, 8, 16, 1, 4>(w.dc3, w.wt3, nullptr, w.dp2, R, false, gate, s)));
  // pool2 -> relu2 -> conv2
  avepool_bwd2_kernel<<<blocks(R * 32 * 64), 256, 0, s>>>(w.dp2, w.c2, w.dc2, R * 32, 8, gate);
  DS_CUDA_TRY(cudaGetLastError());
  if (use_tensor_cores()) {
    DS_TRY((launch_conv5_wgrad_tc<32, 32, 16, 4>(w.p1, w.dc2, w.part, grad + L[1].w_off, grad + L[1].b_off, R, inv_b,
                                                 flags, gate, s)));
  } else {
    DS_TRY((launch_conv5_bwd_w<32, 16, 2, 4>(w.p1, w.dc2, w.part, w.pb, R, 32, gate, s)));
    reduce_parts_kernel<<<blocks(32 * 800), 256, 0, s>>>(w.part, nch4, 32 * 800, grad + L[1].w_off, inv_b, flags, gate);
    reduce_parts_kernel<<<1, 32, 0, s>>>(w.pb, nch4, 32, grad + L[1].b_off, inv_b, flags, gate);
  }
  if (!use_tensor_cores())
    flip_transpose_kernel<<<blocks(32 * 800), 256, 0, s>>>(P + L[1].w_off, w.wt2, 32, 32, gate);
  DS_CUDA_TRY(cudaGetLastError());
  if (use_tensor_cores())
    DS_TRY((launch_conv5_tc<32, 32, 16>(w.dc2, P + L[1].w_off, true, w.wpk, nullptr, w.dr1, R, false, gate, s)));
  else
    DS_TRY((launch_conv5<32, 32, 16, 16, 2, 2>(w.dc2, w.wt2, nullptr, w.dr1, R, false, gate, s)));
  // relu1 -> pool1 (max) -> conv1 (weights only), one sample per partial
  maxpool_relu_bwd2_kernel<<<blocks(R * 32 * 256), 256, 0, s>>>(w.dr1, w.arg1, w.dc1, R * 32, 16, gate);
  DS_CUDA_TRY(cudaGetLastError());
  if (use_tensor_cores()) {
    DS_TRY((launch_conv5_wgrad_tc<3, 32, 32, 1>(idx ? w.x0 : X, w.dc1, w.part, grad + L[0].w_off, grad + L[0].b_off, R,
                                                inv_b, flags, gate, s)));
  } else {
    DS_TRY((launch_conv5_bwd_w<3, 32, 32, 1>(idx ? w.x0 : X, w.dc1, w.part, w.pb, R, 32, gate, s)));
    reduce_parts_kernel<<<blocks(32 * 75), 256, 0, s>>>(w.part, R, 32 * 75, grad + L[0].w_off, inv_b, flags, gate);
    reduce_parts_kernel<<<1, 32, 0, s>>>(w.pb, R, 32, grad + L[0].b_off, inv_b, flags, gate);
  }
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

int launch_cnn_count_hits(const ModelInfo& m, const float* P, const float* X, const uint32_t* y, uint32_t R,
                          void* ws_base, unsigned long long* hits, uint32_t* pred, cudaStream_t s) {
  CnnWs w = carve(R, m.n_classes, ws_base);
  DS_TRY(cnn_forward(m, P, X, nullptr, R, w, nullptr, s));
  cnn_hits_kernel<<<blocks(R, 128), 128, 0, s>>>(w.z, y, R, m.n_classes, pred, hits);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

}  // namespace dsb
