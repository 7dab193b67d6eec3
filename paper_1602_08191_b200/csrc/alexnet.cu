// alexnet.cu — the AlexNet-shaped convnet of BASELINE config 4 (model kind
// DS_MODEL_ALEXNET; NOT IN THE REFERENCE, f64 oracle in
// oracle/ds_oracle_alex.c). loss_and_grad for R rows.
//
// Every contraction is a tcgen05 GEMM (gemm_tc.cu, tf32 operands, f32 accumulation in
// TMEM). Activations are NHWC ([rows][y][x][c], channels contiguous); the inputs of
// conv2..conv5 live in spatially zero-padded maps (border = the conv's padding), so a
// convolution is an implicit GEMM whose K loop walks the filter taps: tap (ky, kx) reads
// the A tile at the pixel shift (ky-p)*Hp + (kx-p) (a TMA row coordinate), no im2col
// matrix is written. Outputs are computed on the padded grid; the epilogue keeps interior
// rows only. Per conv layer (group g, KK taps):
//   forward  out[o] = sum_t in[o + d_t] . Wp_g[t]^T          (taps accumulate)
//   dgrad    din[i] = sum_t dout[i - d_t] . WpT_g[t]^T       (taps accumulate, ReLU mask)
//   wgrad    dW[t]  = doutT . inT(shifted by d_t)^T           (one output per tap, split-K)
// wgrad contracts over pixels, so it reads transposed (pixel-contiguous) copies of dout and
// the padded input: tf32 MMA operands must be K-major. conv1 (11x11 stride 4 on the CHW
// input) becomes a 3x3 stride-1 convolution by space-to-depth: the input is regrouped into
// 4x4 pixel blocks (48 channels on a ceil(S/4) grid) and the 11x11 kernel zero-extended to
// 12x12 (1.19x the MACs, no im2col). LRN, max-pooling, softmax cross-entropy and the bias
// sums are HBM-bound elementwise kernels. The gradient is the batch mean (scale 1/R in the
// GEMM epilogues), rounded to f32 like the reference's Grad = f32(sum / b). Dropout is
// omitted (deterministic; see the oracle).
#include <algorithm>
#include <initializer_list>

#include "ds_common.cuh"
#include "gemm_tc.cuh"
#include "model.cuh"

namespace dsb {
namespace {

thread_local uint32_t t_launches = 0;  // kernels issued by the last loss_and_grad on this thread

constexpr float kLrnAlpha = 1e-4f, kLrnBeta = 0.75f, kLrnK = 1.f;
constexpr int kLrnN = 5;

inline unsigned nblk(uint64_t n, unsigned t = 256) {
  return static_cast<unsigned>(std::min<uint64_t>((n + t - 1) / t, 148ull * 64));
}
inline uint32_t up4(uint32_t v) { return (v + 3) & ~3u; }

struct Shape {
  uint32_t S, H1, P1, P2, P5, C, Cp;
  uint32_t Hs;        // side of the space-to-depth grid of the input (conv1)
  uint32_t Hp2, Hp3;  // padded sides of the conv2 input (pad 2) and the conv3..5 maps (pad 1)
  uint64_t q5;        // fc6 fan-in
};

Shape shape_of(const ModelInfo& m) {
  Shape s{};
  s.S = m.alex_side;
  s.H1 = (s.S - 11) / 4 + 1;
  auto pooled = [](uint32_t h) { return (h - 2) / 2 + 1; };  // ceil((h-3)/2)+1
  s.P1 = pooled(s.H1);
  s.P2 = pooled(s.P1);
  s.P5 = pooled(s.P2);
  s.C = m.n_classes;
  s.Cp = up4(s.C);
  s.Hs = (s.S + 3) / 4;
  s.Hp2 = s.P1 + 4;
  s.Hp3 = s.P2 + 2;
  s.q5 = 256ull * s.P5 * s.P5;
  return s;
}

// conv2..5 (stride 1, same padding, NHWC)
struct ConvSpec {
  uint32_t Cin, Cout, K, pad, g, H, Hp;
  uint32_t cig() const { return Cin / g; }
  uint32_t cog() const { return Cout / g; }
  uint32_t KK() const { return K * K; }
  uint32_t Kg() const { return K * K * cig(); }
};

// conv1 after space-to-depth: 48 -> 96, 3x3 taps on the Hs grid, outputs at [1, 1 + H1)
ConvSpec conv1_spec(const Shape& s) { return ConvSpec{48, 96, 3, 1, 1, s.H1, s.Hs}; }

ConvSpec conv_spec(const Shape& s, int l) {  // l = 0..3 -> conv2..conv5
  static const ConvSpec kConv[4] = {{96, 256, 5, 2, 2, 0, 0}, {256, 384, 3, 1, 1, 0, 0}, {384, 384, 3, 1, 2, 0, 0},
                                    {384, 256, 3, 1, 2, 0, 0}};
  ConvSpec c = kConv[l];
  c.H = l == 0 ? s.P1 : s.P2;
  c.Hp = l == 0 ? s.Hp2 : s.Hp3;
  return c;
}

// ---- workspace ---------------------------------------------------------------------
struct AlexWs {
  // forward maps (p = spatially padded, zero border)
  float *a1, *p1p, *a2, *p2p, *a3p, *a4p, *a5p, *p5, *h6, *h7, *z, *dz;
  uint8_t *arg1, *arg2, *arg5;
  // backward
  float *dh7, *dh6, *dp5, *dc5p, *dc4p, *dc3p, *dp2p, *dc2p, *dp1, *dc1p;
  float *xs, *trA, *trB, *part, *part2, *wtmp, *bpart;
  float *w1p, *wp[4], *wpT[4], *w6T, *w7T, *w8T, *zT, *h7T, *h6T, *p5T, *dh7T, *dh6T;
  double* loss_rows;
  uint64_t end;
};

constexpr uint64_t kPartFloats = 24ull << 20;  // split-K slabs

// one carve for sizing (base = nullptr) and for the pointers
AlexWs carve_ws(const ModelInfo& m, uint32_t R, void* base) {
  AlexWs ws{};
  uint8_t* b = static_cast<uint8_t*>(base);
  const Shape s = shape_of(m);
  const uint64_t M1 = 1ull * R * s.H1 * s.H1, M2 = 1ull * R * s.P1 * s.P1, M3 = 1ull * R * s.P2 * s.P2;
  const uint64_t G1 = 1ull * R * s.Hs * s.Hs, G2 = 1ull * R * s.Hp2 * s.Hp2, G3 = 1ull * R * s.Hp3 * s.Hp3;
  const uint64_t Q5 = R * s.q5;
  const uint32_t Rp = up4(R);
  uint64_t off = 0;
  auto f = [&](float*& p, uint64_t n) { p = reinterpret_cast<float*>(b + off); off += (n * 4 + 255) & ~255ull; };
  auto u = [&](uint8_t*& p, uint64_t n) { p = b + off; off += (n + 255) & ~255ull; };
  f(ws.a1, M1 * 96), f(ws.p1p, G2 * 96), u(ws.arg1, M2 * 96);
  f(ws.a2, M2 * 256), f(ws.p2p, G3 * 256), u(ws.arg2, M3 * 256);
  f(ws.a3p, G3 * 384), f(ws.a4p, G3 * 384), f(ws.a5p, G3 * 256), f(ws.p5, Q5), u(ws.arg5, Q5);
  f(ws.h6, 4096ull * R), f(ws.h7, 4096ull * R), f(ws.z, 1ull * s.Cp * R), f(ws.dz, 1ull * s.Cp * R);
  f(ws.dh7, 4096ull * R), f(ws.dh6, 4096ull * R), f(ws.dp5, Q5);
  f(ws.dc5p, G3 * 256), f(ws.dc4p, G3 * 384), f(ws.dc3p, G3 * 384), f(ws.dp2p, G3 * 256);
  f(ws.dc2p, G2 * 256), f(ws.dp1, M2 * 96), f(ws.dc1p, G1 * 96);
  f(ws.xs, G1 * 48);
  const uint64_t trA = std::max({384 * (G3 + 8), 256 * (G2 + 8), 96 * (G1 + 8)});
  const uint64_t trB = 4 * std::max({384 * (G3 + 8), 96 * (G2 + 8), 48 * (G1 + 8)});
  f(ws.trA, trA), f(ws.trB, trB), f(ws.part, kPartFloats), f(ws.part2, kPartFloats), f(ws.wtmp, 384ull * 2304);
  f(ws.bpart, 4096ull * 512);
  f(ws.w1p, 96ull * 9 * 48);
  for (int l = 0; l < 4; ++l) {
    const ConvSpec c = conv_spec(s, l);
    f(ws.wp[l], 1ull * c.Cout * c.Kg());
    f(ws.wpT[l], 1ull * c.Cout * c.Kg());
  }
  f(ws.w6T, s.q5 * 4096), f(ws.w7T, 4096ull * 4096), f(ws.w8T, 4096ull * s.Cp);
  f(ws.zT, 1ull * s.Cp * Rp), f(ws.h7T, 4096ull * Rp), f(ws.h6T, 4096ull * Rp), f(ws.p5T, s.q5 * Rp);
  f(ws.dh7T, 4096ull * Rp), f(ws.dh6T, 4096ull * Rp);
  ws.loss_rows = reinterpret_cast<double*>(b + off);
  off += (R * 8ull + 255) & ~255ull;
  ws.end = off;
  return ws;
}

// ---- kernels -------------------------------------------------------------------------
#define GATE \
  if (gate && *gate) return

// space-to-depth of the CHW input rows (row r = X[idx[r]]): xs[r][ys][xs][(dy*4+dx)*3+c] =
// X[c][4ys+dy][4xs+dx] (0 past the image), on the Hs x Hs grid
__global__ void s2d_kernel(const float* __restrict__ X, const uint32_t* __restrict__ idx, uint32_t F, uint32_t S,
                           uint32_t R, uint32_t Hs, float* __restrict__ xs, const uint32_t* gate) {
  GATE;
  const uint32_t HH = Hs * Hs, total = R * HH * 48;
  for (uint32_t i = blockIdx.x * 256 + threadIdx.x; i < total; i += gridDim.x * 256) {
    const uint32_t p = i / 48, ch = i - p * 48;
    const uint32_t r = p / HH, pix = p - r * HH, ys = pix / Hs, xq = pix - ys * Hs;
    const uint32_t blk = ch / 3, c = ch - blk * 3, dy = blk / 4, dx = blk - dy * 4;
    const uint32_t y = ys * 4 + dy, x = xq * 4 + dx;
    float v = 0.f;
    if (y < S && x < S) {
      const uint64_t row = idx ? idx[r] : r;
      v = __ldg(X + row * F + (c * S + y) * S + x);
    }
    xs[i] = v;
  }
}

// conv1 weights [96][3][11][11] -> Wp [96][9 taps (ty,tx)][48 (dy,dx,c)], zero past 11
__global__ void pack_conv1_s2d_kernel(const float* __restrict__ W, float* __restrict__ Wp, const uint32_t* gate) {
  GATE;
  for (uint32_t i = blockIdx.x * 256 + threadIdx.x; i < 96 * 432; i += gridDim.x * 256) {
    const uint32_t co = i / 432, rem = i - co * 432, t = rem / 48, ch = rem - t * 48;
    const uint32_t ty = t / 3, tx = t - ty * 3, blk = ch / 3, c = ch - blk * 3, dy = blk / 4, dx = blk - dy * 4;
    const uint32_t ky = ty * 4 + dy, kx = tx * 4 + dx;
    Wp[i] = (ky < 11 && kx < 11) ? W[((co * 3 + c) * 11 + ky) * 11 + kx] : 0.f;
  }
}

// packed conv1 weight gradient [96][9][48] -> Caffe [96][3][11][11]
__global__ void unpack_conv1_s2d_kernel(const float* __restrict__ dWp, float* __restrict__ grad, uint32_t* flags,
                                        const uint32_t* gate) {
  GATE;
  for (uint32_t i = blockIdx.x * 256 + threadIdx.x; i < 96 * 363; i += gridDim.x * 256) {
    const uint32_t co = i / 363, rem = i - co * 363, c = rem / 121, kyx = rem - c * 121, ky = kyx / 11, kx = kyx - ky * 11;
    const uint32_t t = (ky / 4) * 3 + kx / 4, ch = ((ky % 4) * 4 + kx % 4) * 3 + c;
    const float v = dWp[co * 432 + t * 48 + ch];
    if (!isfinite(v)) atomicOr(flags, DS_FLAG_GRAD_NONFINITE);
    grad[i] = v;
  }
}

// out[c][r] = in[r][c] for a [rows x cols] matrix (ld_in, ld_out), 32x32 tiles, 256 threads:
// float4 loads along c and float4 stores along r (scalar at ragged edges / odd strides)
__global__ void __launch_bounds__(256) transpose_kernel(const float* __restrict__ in, uint64_t rows, uint32_t cols,
                                                        uint64_t ld_in, float* __restrict__ out, uint64_t ld_out,
                                                        const uint32_t* gate) {
  GATE;
  __shared__ float tile[32][33];
  const uint64_t r0 = blockIdx.x * 32ull;
  const uint32_t c0 = blockIdx.y * 32;
  const uint32_t t = threadIdx.x, lr = t / 8, lc = (t % 8) * 4;  // load: row lr, cols lc..lc+3
  const bool vin = (ld_in % 4) == 0 && (reinterpret_cast<uintptr_t>(in) & 15) == 0;
  const uint64_t r = r0 + lr;
  const uint32_t c = c0 + lc;
  if (vin && r < rows && c + 3 < cols) {
    const float4 v = *reinterpret_cast<const float4*>(in + r * ld_in + c);
    tile[lr][lc] = v.x, tile[lr][lc + 1] = v.y, tile[lr][lc + 2] = v.z, tile[lr][lc + 3] = v.w;
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j) tile[lr][lc + j] = (r < rows && c + j < cols) ? in[r * ld_in + c + j] : 0.f;
  }
  __syncthreads();
  const uint32_t sc = t / 8, sr = (t % 8) * 4;  // store: out row c0 + sc, cols r0 + sr .. + 3
  const uint32_t oc = c0 + sc;
  const uint64_t orr = r0 + sr;
  if (oc >= cols) return;
  const bool vout = (ld_out % 4) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  if (vout && orr + 3 < rows) {
    *reinterpret_cast<float4*>(out + oc * ld_out + orr) =
        make_float4(tile[sr][sc], tile[sr + 1][sc], tile[sr + 2][sc], tile[sr + 3][sc]);
  } else {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      if (orr + j < rows) out[oc * ld_out + orr + j] = tile[sr + j][sc];
  }
}

// transpose_kernel fused with the first pass of colsum (the bias gradient) over the same
// matrix: block (x, y) walks row tiles x, x + gridDim.x, ... of column tile y, so the
// gradient map is read once for both; part[x][n] = sum of column n over the block's rows
// (zero-filled beyond `rows`), reduced by colsum_final_kernel.
__global__ void __launch_bounds__(256) transpose_colsum_kernel(const float* __restrict__ in, uint64_t rows,
                                                               uint32_t cols, float* __restrict__ out,
                                                               uint64_t ld_out, float* __restrict__ part,
                                                               const uint32_t* gate) {
  GATE;
  __shared__ float tile[32][33];
  const uint32_t c0 = blockIdx.y * 32;
  const uint32_t t = threadIdx.x, lr = t / 8, lc = (t % 8) * 4;
  const uint32_t sc = t / 8, sr = (t % 8) * 4;
  const uint32_t c = c0 + lc, oc = c0 + sc;
  const bool vin = (cols % 4) == 0 && (reinterpret_cast<uintptr_t>(in) & 15) == 0;
  const bool vout = (ld_out % 4) == 0 && (reinterpret_cast<uintptr_t>(out) & 15) == 0;
  float acc = 0.f;
  for (uint64_t r0 = blockIdx.x * 32ull; r0 < rows; r0 += gridDim.x * 32ull) {
    const uint64_t r = r0 + lr;
    if (vin && r < rows && c + 3 < cols) {
      const float4 v = *reinterpret_cast<const float4*>(in + r * cols + c);
      tile[lr][lc] = v.x, tile[lr][lc + 1] = v.y, tile[lr][lc + 2] = v.z, tile[lr][lc + 3] = v.w;
    } else {
#pragma unroll
      for (int j = 0; j < 4; ++j) tile[lr][lc + j] = (r < rows && c + j < cols) ? in[r * cols + c + j] : 0.f;
    }
    __syncthreads();
    const float a = tile[sr][sc], b = tile[sr + 1][sc], d = tile[sr + 2][sc], e = tile[sr + 3][sc];
    acc += (a + b) + (d + e);
    const uint64_t orr = r0 + sr;
    if (oc < cols) {
      if (vout && orr + 3 < rows) {
        *reinterpret_cast<float4*>(out + oc * ld_out + orr) = make_float4(a, b, d, e);
      } else {
        const float q[4] = {a, b, d, e};
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (orr + j < rows) out[oc * ld_out + orr + j] = q[j];
      }
    }
    __syncthreads();
  }
  acc += __shfl_xor_sync(0xffffffffu, acc, 1);
  acc += __shfl_xor_sync(0xffffffffu, acc, 2);
  acc += __shfl_xor_sync(0xffffffffu, acc, 4);
  if ((t % 8) == 0 && oc < cols) part[1ull * blockIdx.x * cols + oc] = acc;
}

// Four pixel-shifted transposed copies: out[s][c][m] = in[m - s][c] (0 outside the rows),
// m < ldT. TMA needs 16-byte aligned inner coordinates, so a weight-gradient tap with pixel
// shift d reads copy s = (-d mod 4) at the aligned offset d + s: the shifted column is never
// left of the unshifted one, so no needed pixel falls before column 0. 32 m x 32 c per
// block (256 threads), float4 loads along c (cols % 4 == 0) and float4 stores along m.
__global__ void __launch_bounds__(256) transpose_shift4_kernel(const float* __restrict__ in, uint64_t rows,
                                                               uint32_t cols, float* __restrict__ out, uint64_t ldT,
                                                               const uint32_t* gate) {
  GATE;
  __shared__ float tile[36][33];  // rows r0-3 .. r0+32 (35 used)
  const int64_t r0 = blockIdx.x * 32ll;
  const uint32_t c0 = blockIdx.y * 32;
  const uint32_t t = threadIdx.x;
  for (uint32_t i = t; i < 35 * 8; i += 256) {
    const uint32_t lr = i / 8, lc = (i % 8) * 4;
    const int64_t r = r0 - 3 + lr;
    const uint32_t c = c0 + lc;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (r >= 0 && r < static_cast<int64_t>(rows) && c < cols) v = *reinterpret_cast<const float4*>(in + r * cols + c);
    tile[lr][lc] = v.x, tile[lr][lc + 1] = v.y, tile[lr][lc + 2] = v.z, tile[lr][lc + 3] = v.w;
  }
  __syncthreads();
  for (uint32_t i = t; i < 4 * 32 * 8; i += 256) {  // (shift, c, 4-wide m group)
    const uint32_t sft = i / 256, rem = i % 256, sc = rem / 8, sm = (rem % 8) * 4;
    const uint32_t c = c0 + sc;
    const uint64_t m = r0 + sm;
    if (c >= cols || m >= ldT) continue;
    const uint32_t tr = sm + 3 - sft;
    *reinterpret_cast<float4*>(out + (sft * cols + c) * ldT + m) =
        make_float4(tile[tr][sc], tile[tr + 1][sc], tile[tr + 2][sc], tile[tr + 3][sc]);
  }
}

// Caffe conv weight [Cout][cg][K][K] -> Wp [Cout][K*K][cg] and per group WpT_g [K*K][cg][Cout_g]
__global__ void pack_conv_kernel(const float* __restrict__ W, uint32_t Cout, uint32_t cg, uint32_t K, uint32_t g,
                                 float* __restrict__ Wp, float* __restrict__ WpT, const uint32_t* gate) {
  GATE;
  const uint32_t KK = K * K, Kg = KK * cg, cog = Cout / g;
  const uint64_t total = 1ull * Cout * Kg;
  for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < total; i += gridDim.x * 256ull) {
    const uint32_t co = static_cast<uint32_t>(i / Kg), rem = static_cast<uint32_t>(i % Kg);
    const uint32_t c = rem / KK, kk = rem % KK;  // Caffe order (c, ky, kx)
    const float v = W[i];
    const uint32_t k = kk * cg + c;  // packed order (ky, kx, c)
    Wp[1ull * co * Kg + k] = v;
    const uint32_t gi = co / cog, cl = co % cog;
    WpT[1ull * gi * Kg * cog + 1ull * k * cog + cl] = v;
  }
}

// packed weight gradient [Cout][(ky,kx,c)] -> Caffe order [Cout][c][ky][kx]
__global__ void unpack_wgrad_kernel(const float* __restrict__ dWp, uint32_t rows, uint32_t cg, uint32_t K,
                                    float* __restrict__ grad, uint32_t* flags, const uint32_t* gate) {
  GATE;
  const uint32_t KK = K * K, Kg = KK * cg;
  for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < 1ull * rows * Kg; i += gridDim.x * 256ull) {
    const uint32_t co = static_cast<uint32_t>(i / Kg), k = static_cast<uint32_t>(i % Kg);
    const uint32_t kk = k / cg, c = k % cg;
    const float v = dWp[i];
    if (!isfinite(v)) atomicOr(flags, DS_FLAG_GRAD_NONFINITE);
    grad[(1ull * co * cg + c) * KK + kk] = v;
  }
}

// MAX 3x3/2 ceil-mode over an NHWC map (input padded by ipad, output padded by opad, or
// per-row CHW when chw != 0: the fc6 input). arg[r][py][px][c] (unpadded) = window position
// (0..8) of the first maximum in scan order. One warp per pooled pixel (8 per block),
// lanes across channels.
__global__ void __launch_bounds__(256) maxpool_fwd_kernel(const float* __restrict__ in, uint32_t R, uint32_t H,
                                                          uint32_t C, uint32_t Ho, uint32_t ipad, uint32_t opad,
                                                          int chw, float* __restrict__ out,
                                                          uint8_t* __restrict__ arg, const uint32_t* gate) {
  GATE;
  const uint32_t Hi = H + 2 * ipad, Hq = Ho + 2 * opad, HoHo = Ho * Ho;
  const uint32_t p = blockIdx.x * 8 + threadIdx.x / 32, lane = threadIdx.x % 32;
  if (p >= R * HoHo) return;
  const uint32_t r = p / HoHo, pix = p - r * HoHo, py = pix / Ho, px = pix - py * Ho;
  const uint32_t hs = py * 2, ws = px * 2, he = min(hs + 3, H), we = min(ws + 3, H);
  // the window's 9 loads are independent and issued together (clipped taps are predicated
  // off), then scanned in order: first maximum, strict >
  const float* base = in + (static_cast<uint64_t>(r * Hi + hs + ipad) * Hi + ws + ipad) * C;
  const uint32_t nh = he - hs, nw = we - ws, rowC = Hi * C;
  // four channels per lane (C % 4 == 0 at every call site: 96, 256): float4 window loads,
  // uchar4 argmax stores, float4 output stores (scalar into the CHW planes of pool5)
#pragma unroll 2  // two channel groups' window loads in flight per lane
  for (uint32_t c = lane * 4; c < C; c += 128) {
    float4 v[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      const uint32_t dh = k / 3, dw = k % 3;
      v[k] = (dh < nh && dw < nw) ? *reinterpret_cast<const float4*>(base + dh * rowC + dw * C + c)
                                  : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
    }
    float4 best = v[0];
    uchar4 bi = make_uchar4(0, 0, 0, 0);
#pragma unroll
    for (int k = 1; k < 9; ++k) {
      if (v[k].x > best.x) best.x = v[k].x, bi.x = k;
      if (v[k].y > best.y) best.y = v[k].y, bi.y = k;
      if (v[k].z > best.z) best.z = v[k].z, bi.z = k;
      if (v[k].w > best.w) best.w = v[k].w, bi.w = k;
    }
    if (chw) {
      const uint64_t o = (static_cast<uint64_t>(r) * C + c) * HoHo + pix;
      out[o] = best.x, out[o + HoHo] = best.y, out[o + 2 * HoHo] = best.z, out[o + 3 * HoHo] = best.w;
    } else {
      *reinterpret_cast<float4*>(out + (static_cast<uint64_t>(r * Hq + py + opad) * Hq + px + opad) * C + c) = best;
    }
    *reinterpret_cast<uchar4*>(arg + static_cast<uint64_t>(p) * C + c) = bi;
  }
}

// LRN across channels, y = x * (k + a/n sum_{|c'-c|<=2} x_c'^2)^-b, fused into the MAX 3x3/2 ceil-mode pool over its output:
// one warp per pooled pixel, four channels per lane; each window tap's LRN output is
// recomputed from x (channels c-2 .. c+5: float2 + float4 + float2 loads), so the LRN output
// map is never written (the backward recomputes the LRN scale from x and pools by argmax).
// x unpadded NHWC [R][H][H][C]; out padded by opad; arg as maxpool_fwd_kernel.
__global__ void __launch_bounds__(256) lrn_maxpool_fwd_kernel(const float* __restrict__ x, uint32_t R, uint32_t H,
                                                              uint32_t C, uint32_t Ho, uint32_t opad,
                                                              float* __restrict__ out, uint8_t* __restrict__ arg,
                                                              const uint32_t* gate) {
  GATE;
  const uint32_t Hq = Ho + 2 * opad, HoHo = Ho * Ho;
  const uint32_t p = blockIdx.x * 8 + threadIdx.x / 32, lane = threadIdx.x % 32;
  if (p >= R * HoHo) return;
  const uint32_t r = p / HoHo, pix = p - r * HoHo, py = pix / Ho, px = pix - py * Ho;
  const uint32_t hs = py * 2, ws = px * 2, he = min(hs + 3, H), we = min(ws + 3, H);
  const float* base = x + (static_cast<uint64_t>(r * H + hs) * H + ws) * C;
  const uint32_t nh = he - hs, nw = we - ws, rowC = H * C;
  for (uint32_t c = lane * 4; c < C; c += 128) {
    float4 best = make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
    uchar4 bi = make_uchar4(0, 0, 0, 0);
#pragma unroll
    for (int k = 0; k < 9; ++k) {
      const uint32_t dh = k / 3, dw = k % 3;
      float o[4];
      if (dh < nh && dw < nw) {
        const float* q = base + dh * rowC + dw * C + c;
        const float4 m = *reinterpret_cast<const float4*>(q);
        const float2 lo = c >= 2 ? *reinterpret_cast<const float2*>(q - 2) : make_float2(0.f, 0.f);
        const float2 hi = c + 4 < C ? *reinterpret_cast<const float2*>(q + 4) : make_float2(0.f, 0.f);
        const float v[8] = {lo.x, lo.y, m.x, m.y, m.z, m.w, hi.x, hi.y};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const float ss =
              v[j] * v[j] + v[j + 1] * v[j + 1] + v[j + 2] * v[j + 2] + v[j + 3] * v[j + 3] + v[j + 4] * v[j + 4];
          o[j] = v[j + 2] * __powf(kLrnK + kLrnAlpha / kLrnN * ss, -kLrnBeta);
        }
      } else {
        o[0] = o[1] = o[2] = o[3] = -INFINITY;
      }
      if (k == 0) {
        best = make_float4(o[0], o[1], o[2], o[3]);
      } else {  // first maximum in scan order, strict >
        if (o[0] > best.x) best.x = o[0], bi.x = k;
        if (o[1] > best.y) best.y = o[1], bi.y = k;
        if (o[2] > best.z) best.z = o[2], bi.z = k;
        if (o[3] > best.w) best.w = o[3], bi.w = k;
      }
    }
    *reinterpret_cast<float4*>(out + (static_cast<uint64_t>(r * Hq + py + opad) * Hq + px + opad) * C + c) = best;
    *reinterpret_cast<uchar4*>(arg + static_cast<uint64_t>(p) * C + c) = bi;
  }
}

// gather form of the max-pool backward: din[r][y][x][c] = sum of dout over the windows whose
// maximum sat at (y, x). dout: padded by opad (or per-row CHW), din/mask: padded by ipad;
// mask (optional) zeroes din where the pooled map's source was not > 0 (ReLU). One warp
// per input pixel (8 per block), lanes across channels.
__global__ void __launch_bounds__(256) maxpool_bwd_kernel(const float* __restrict__ dout,
                                                          const uint8_t* __restrict__ arg, uint32_t R, uint32_t H,
                                                          uint32_t C, uint32_t Ho, uint32_t opad, int chw,
                                                          uint32_t ipad, const float* __restrict__ mask,
                                                          float* __restrict__ din, const uint32_t* gate) {
  GATE;
  const uint32_t Hi = H + 2 * ipad, Hq = Ho + 2 * opad, HH = H * H;
  const uint32_t p = blockIdx.x * 8 + threadIdx.x / 32, lane = threadIdx.x % 32;
  if (p >= R * HH) return;
  const uint32_t r = p / HH, pix = p - r * HH, y = pix / H, x = pix - y * H;
  const uint32_t py0 = y >= 2 ? (y - 1) / 2 : 0, py1 = min(y / 2, Ho - 1);
  const uint32_t px0 = x >= 2 ? (x - 1) / 2 : 0, px1 = min(x / 2, Ho - 1);
  const uint64_t dbase = (static_cast<uint64_t>(r * Hi + y + ipad) * Hi + x + ipad) * C;
  // up to 2 x 2 windows cover (y, x); their argmax bytes and gradients are loaded
  // independently (no load waits on a comparison), then the matches are summed in window
  // order. Window offsets and expected argmax positions are channel-independent: hoisted.
  const bool two_y = py1 > py0, two_x = px1 > px0;
  // 32-bit offsets: the pooled maps hold < 2^32 elements (the caller bounds the batch)
  const uint8_t* ap[4];
  const float* dp[4];
  uint32_t want[4];
  bool ok[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    const uint32_t py = py0 + (w >> 1), px = px0 + (w & 1);
    ok[w] = ((w >> 1) == 0 || two_y) && ((w & 1) == 0 || two_x);
    ap[w] = arg + ((r * Ho + py) * Ho + px) * C;
    dp[w] = dout + (chw ? r * C * Ho * Ho + py * Ho + px : ((r * Hq + py + opad) * Hq + px + opad) * C);
    want[w] = (y - py * 2) * 3 + (x - px * 2);
  }
  // four channels per lane (C % 4 == 0 at every call site: 96, 256): uchar4 argmax loads,
  // float4 gradient loads (scalar across the CHW planes of pool5) and float4 stores; the
  // per-channel window order of the sum is unchanged
  const uint32_t dstride = chw ? Ho * Ho : 1;  // channel step in dout
  for (uint32_t c = lane * 4; c < C; c += 128) {
    uchar4 av[4];
    float4 dv[4];
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      av[w] = ok[w] ? *reinterpret_cast<const uchar4*>(ap[w] + c) : make_uchar4(255, 255, 255, 255);
      if (!ok[w])
        dv[w] = make_float4(0.f, 0.f, 0.f, 0.f);
      else if (chw)
        dv[w] = make_float4(dp[w][c * dstride], dp[w][(c + 1) * dstride], dp[w][(c + 2) * dstride],
                            dp[w][(c + 3) * dstride]);
      else
        dv[w] = *reinterpret_cast<const float4*>(dp[w] + c);
    }
    float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      if (av[w].x == want[w]) s.x += dv[w].x;
      if (av[w].y == want[w]) s.y += dv[w].y;
      if (av[w].z == want[w]) s.z += dv[w].z;
      if (av[w].w == want[w]) s.w += dv[w].w;
    }
    if (mask) {
      const float4 mk = *reinterpret_cast<const float4*>(mask + dbase + c);
      if (!(mk.x > 0.f)) s.x = 0.f;
      if (!(mk.y > 0.f)) s.y = 0.f;
      if (!(mk.z > 0.f)) s.z = 0.f;
      if (!(mk.w > 0.f)) s.w = 0.f;
    }
    *reinterpret_cast<float4*>(din + dbase + c) = s;
  }
}

// max-pool backward and LRN backward (ReLU-masked) fused, one warp per pixel of the LRN
// input map x (unpadded [R][H][H][C], C % 4 == 0, C <= 256): the warp gathers the pooled
// gradient of every channel of its pixel (maxpool_bwd_kernel's window order) into shared
// memory, then applies the LRN backward across the channel window from there (scale
// recomputed from x, masked by the ReLU that produced x):
//   dx_c = dy_c s_c^-b - (2 a b / n) x_c sum_{|j-c|<=2} dy_j x_j s_j^(-b-1)
// so the LRN output gradient never round-trips through HBM. dout: pooled gradient padded by opad; dx written at pixel
// (y + xpad, x + xpad) of a map of side Hx.
__global__ void __launch_bounds__(256) pool_lrn_bwd_relu_kernel(const float* __restrict__ dout,
                                                                const uint8_t* __restrict__ arg,
                                                                const float* __restrict__ x, uint32_t R, uint32_t H,
                                                                uint32_t C, uint32_t Ho, uint32_t opad, uint32_t xpad,
                                                                uint32_t Hx, float* __restrict__ dx,
                                                                const uint32_t* gate) {
  GATE;
  __shared__ float4 dys[8][66];  // per warp: channels -4 .. C + 3 (zero outside 0 .. C-1)
  __shared__ float4 wts[8][66];  // per warp: LRN window terms, same channel range
  const uint32_t HH = H * H, Hq = Ho + 2 * opad, warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t p = blockIdx.x * 8 + warp;
  if (p >= R * HH) return;
  const uint32_t r = p / HH, pix = p - r * HH, y = pix / H, xx = pix - y * H;
  const uint32_t py0 = y >= 2 ? (y - 1) / 2 : 0, py1 = min(y / 2, Ho - 1);
  const uint32_t px0 = xx >= 2 ? (xx - 1) / 2 : 0, px1 = min(xx / 2, Ho - 1);
  const bool two_y = py1 > py0, two_x = px1 > px0;
  const uint8_t* ap[4];
  const float* dp[4];
  uint32_t want[4];
  bool ok[4];
#pragma unroll
  for (int w = 0; w < 4; ++w) {
    const uint32_t py = py0 + (w >> 1), px = px0 + (w & 1);
    ok[w] = ((w >> 1) == 0 || two_y) && ((w & 1) == 0 || two_x);
    ap[w] = arg + ((r * Ho + py) * Ho + px) * C;
    dp[w] = dout + ((r * Hq + py + opad) * Hq + px + opad) * C;
    want[w] = (y - py * 2) * 3 + (xx - px * 2);
  }
  const uint32_t C4 = C / 4;
  if (lane == 0) dys[warp][0] = make_float4(0.f, 0.f, 0.f, 0.f), dys[warp][C4 + 1] = dys[warp][0];
  for (uint32_t q = lane; q < C4; q += 32) {
    const uint32_t c = q * 4;
    uchar4 av[4];
    float4 dv[4];
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      av[w] = ok[w] ? *reinterpret_cast<const uchar4*>(ap[w] + c) : make_uchar4(255, 255, 255, 255);
      dv[w] = ok[w] ? *reinterpret_cast<const float4*>(dp[w] + c) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    float4 sum = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      if (av[w].x == want[w]) sum.x += dv[w].x;
      if (av[w].y == want[w]) sum.y += dv[w].y;
      if (av[w].z == want[w]) sum.z += dv[w].z;
      if (av[w].w == want[w]) sum.w += dv[w].w;
    }
    dys[warp][q + 1] = sum;
  }
  __syncwarp();
  const float* ds = reinterpret_cast<const float*>(&dys[warp][1]);  // ds[c], c in [-4, C + 4)
  // pass 1: each channel's scale once (one log2, two exp2): s_c^-b in registers and
  // w_c = dy_c x_c s_c^(-b-1) in shared memory; pass 2 sums w over the 5-channel window
  float* wsm = reinterpret_cast<float*>(&wts[warp][1]);  // wsm[c], c in [-4, C + 4)
  if (lane == 0) wts[warp][0] = make_float4(0.f, 0.f, 0.f, 0.f), wts[warp][C4 + 1] = wts[warp][0];
  const float* px = x + static_cast<uint64_t>(p) * C;
  float pwr[2][4], xcr[2][4];
#pragma unroll
  for (int it = 0; it < 2; ++it) {  // C <= 256: at most two channel groups per lane
    const uint32_t q = lane + it * 32;
    if (q >= C4) continue;
    const uint32_t c0 = q * 4;
    float xv[8];  // x[c0-2 .. c0+5]
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int c = static_cast<int>(c0) - 2 + j;
      xv[j] = (c >= 0 && c < static_cast<int>(C)) ? __ldg(px + c) : 0.f;
    }
    float sq[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) sq[j] = xv[j] * xv[j];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const float ss = ((sq[j] + sq[j + 1]) + (sq[j + 2] + sq[j + 3])) + sq[j + 4];
      const float sc = kLrnK + kLrnAlpha / kLrnN * ss;
      const float l2 = __log2f(sc);
      pwr[it][j] = exp2f(-kLrnBeta * l2);
      xcr[it][j] = xv[j + 2];
      wsm[c0 + j] = ds[c0 + j] * xv[j + 2] * exp2f(-(kLrnBeta + 1.f) * l2);
    }
  }
  __syncwarp();
#pragma unroll
  for (int it = 0; it < 2; ++it) {
    const uint32_t q = lane + it * 32;
    if (q >= C4) continue;
    const uint32_t c0 = q * 4;
    float o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = static_cast<int>(c0) + j;  // signed: wsm[c - 2] at c < 2 is the zero guard
      const float xc = xcr[it][j];
      const float acc = wsm[c - 2] + wsm[c - 1] + wsm[c] + wsm[c + 1] + wsm[c + 2];
      o[j] = xc > 0.f ? ds[c] * pwr[it][j] - 2.f * kLrnAlpha * kLrnBeta / kLrnN * xc * acc : 0.f;
    }
    *reinterpret_cast<float4*>(dx + (static_cast<uint64_t>(r * Hx + y + xpad) * Hx + xx + xpad) * C + c0) =
        make_float4(o[0], o[1], o[2], o[3]);
  }
}

// softmax cross-entropy, one warp per row: loss_rows[r], dz[r][c] = softmax - onehot
// (f64 log-sum-exp as the reference's sample_loss_grad, model.cpp:205-214)
__global__ void softmax_ce_warp_kernel(const float* __restrict__ z, uint32_t ldz, const uint32_t* __restrict__ y,
                                       const uint32_t* __restrict__ idx, uint32_t R, uint32_t C,
                                       double* __restrict__ loss_rows, float* __restrict__ dz, uint32_t* flags,
                                       const uint32_t* gate) {
  GATE;
  const uint32_t r = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x % 32;
  if (r >= R) return;
  const float* zr = z + 1ull * r * ldz;
  double zmax = -INFINITY;
  for (uint32_t c = lane; c < C; c += 32) zmax = fmax(zmax, static_cast<double>(zr[c]));
  for (int o = 16; o; o >>= 1) zmax = fmax(zmax, __shfl_xor_sync(0xffffffffu, zmax, o));
  double sum = 0.0;
  for (uint32_t c = lane; c < C; c += 32) sum += exp(static_cast<double>(zr[c]) - zmax);
  for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
  const double lse = zmax + log(sum);
  const uint32_t label = y[idx ? idx[r] : r];
  if (lane == 0) {
    if (label >= C) {
      atomicOr(flags, DS_FLAG_LABEL_RANGE);
      loss_rows[r] = 0.0;
    } else {
      loss_rows[r] = lse - static_cast<double>(zr[label]);
    }
  }
  if (dz)
    for (uint32_t c = lane; c < ldz; c += 32)
      dz[1ull * r * ldz + c] =
          c < C ? static_cast<float>(exp(static_cast<double>(zr[c]) - lse) - (c == label ? 1.0 : 0.0)) : 0.f;
}

__global__ void alex_loss_mean_kernel(const double* __restrict__ loss_rows, uint32_t R, double* loss_out,
                                      uint32_t* flags, const uint32_t* gate) {
  GATE;
  double s = 0.0;
  for (uint32_t r = 0; r < R; ++r) s += loss_rows[r];
  const double l = s / R;
  if (!isfinite(l)) atomicOr(flags, DS_FLAG_LOSS_NONFINITE);
  *loss_out = l;
}

// column sums of d[rows][N] (ld): block (column tile of 32, part) with 8 row lanes per
// column, reduced in shared memory -> part[part][N]; then one warp per column sums the parts
// in a fixed order (deterministic) and scales
__global__ void colsum_part_kernel(const float* __restrict__ d, uint64_t rows, uint32_t N, uint64_t ld,
                                   uint64_t rows_per_part, float* __restrict__ part, const uint32_t* gate) {
  GATE;
  __shared__ float red[8][33];
  const uint32_t n = blockIdx.x * 32 + threadIdx.x;
  const uint64_t r0 = blockIdx.y * rows_per_part, r1 = min(rows, r0 + rows_per_part);
  float s = 0.f;
  if (n < N)
    for (uint64_t r = r0 + threadIdx.y; r < r1; r += 8) s += d[r * ld + n];
  red[threadIdx.y][threadIdx.x] = s;
  __syncthreads();
  if (threadIdx.y == 0 && n < N) {
    float t = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) t += red[j][threadIdx.x];
    part[1ull * blockIdx.y * N + n] = t;
  }
}
__global__ void colsum_final_kernel(const float* __restrict__ part, uint32_t nparts, uint32_t N, float scale,
                                    float* __restrict__ out, uint32_t* flags, const uint32_t* gate) {
  GATE;
  const uint32_t n = blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32, lane = threadIdx.x % 32;
  if (n >= N) return;
  float s = 0.f;
  for (uint32_t p = lane; p < nparts; p += 32) s += part[1ull * p * N + n];
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) {
    const float v = s * scale;
    if (!isfinite(v)) atomicOr(flags, DS_FLAG_GRAD_NONFINITE);
    out[n] = v;
  }
}

// Zero the border of a padded NHWC map [R][Hp][Hp][C] (everything outside rows and columns
// [pad, pad + H)); the interior is rewritten every step, so only the border needs clearing.
// One block per (image, row); interior rows clear only their 2 * pad... edge pixels.
__global__ void zero_border_kernel(float* __restrict__ map, uint32_t Hp, uint32_t pad, uint32_t H, uint32_t C,
                                   const uint32_t* gate) {
  GATE;
  const uint32_t r = blockIdx.x / Hp, yp = blockIdx.x - r * Hp;
  float* row = map + (static_cast<uint64_t>(r) * Hp + yp) * Hp * C;
  const bool full = yp < pad || yp >= pad + H;
  const uint32_t n = full ? Hp * C : (Hp - H) * C;  // the row, or its left + right edges
  for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
    uint32_t e = i;
    if (!full && e >= pad * C) e += H * C;  // skip the interior columns
    row[e] = 0.f;
  }
}

// Several maps' borders in one launch (blocks [first[i], first[i + 1]) clear map i): the
// per-step border clears were 11 launches of ~7 us each, latency not bandwidth
struct BorderMaps {
  float* p[6];
  uint32_t Hp[6], pad[6], H[6], C[6], first[7];
  uint32_t n;
};
__global__ void zero_borders_kernel(const __grid_constant__ BorderMaps bm, const uint32_t* gate) {
  GATE;
  uint32_t i = 0;
  while (i + 1 < bm.n && blockIdx.x >= bm.first[i + 1]) ++i;
  const uint32_t b = blockIdx.x - bm.first[i], Hp = bm.Hp[i], pad = bm.pad[i], H = bm.H[i], C = bm.C[i];
  const uint32_t r = b / Hp, yp = b - r * Hp;
  float* row = bm.p[i] + (static_cast<uint64_t>(r) * Hp + yp) * Hp * C;
  const bool full = yp < pad || yp >= pad + H;
  const uint32_t n = full ? Hp * C : (Hp - H) * C;  // the row, or its left + right edges
  for (uint32_t k = threadIdx.x; k < n; k += blockDim.x) {
    uint32_t e = k;
    if (!full && e >= pad * C) e += H * C;  // skip the interior columns
    row[e] = 0.f;
  }
}

// argmax of the logits (first maximum), hits against labels (predict, model.cpp:303-318)
__global__ void alex_hits_kernel(const float* __restrict__ z, uint32_t ldz, const uint32_t* __restrict__ y, uint32_t R,
                                 uint32_t C, uint32_t* pred, unsigned long long* hits) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= R) return;
  const float* zr = z + 1ull * r * ldz;
  uint32_t best = 0;
  for (uint32_t k = 1; k < C; ++k)
    if (zr[k] > zr[best]) best = k;
  if (pred) pred[r] = best;
  if (hits && y && best == y[r]) atomicAdd(hits, 1ull);
}

// ---- host helpers --------------------------------------------------------------------
// DS_DEBUG_SYNC=1: synchronize and check after every launch of this file (fault isolation)
int debug_sync(cudaStream_t s, int line) {
  static const bool on = [] {
    const char* e = getenv("DS_DEBUG_SYNC");
    return e && e[0] == '1';
  }();
  if (!on) return DS_OK;
  const cudaError_t e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return set_error(DS_E_CUDA, "alexnet.cu:%d: %s", line, cudaGetErrorString(e));
  return DS_OK;
}
#define KDONE(n)                          \
  do {                                    \
    t_launches += (n);                    \
    DS_TRY(debug_sync(s_, __LINE__));     \
  } while (0)

struct Ctx {
  cudaStream_t s;
  const uint32_t* gate;
  float* part;
  uint32_t* flags;
};

// A second stream per device for work that can run beside the main chain (weight-gradient
// GEMMs beside data-gradient GEMMs, FC weight transposes beside the forward). Fork and join
// are event edges, so the pair is captured into the engine's CUDA graph as parallel branches.
struct Side {
  cudaStream_t s = nullptr;
  cudaEvent_t ev[16] = {};
};
int side_stream(Side** out) {
  // per host thread: the fork/join events must not be shared between engines driven from
  // different threads (an interleaved record would retarget another engine's wait)
  thread_local Side sides[64];
  int dev = 0;
  DS_CUDA_TRY(cudaGetDevice(&dev));
  Side& sd = sides[dev & 63];
  if (!sd.s) {
    DS_CUDA_TRY(cudaStreamCreateWithFlags(&sd.s, cudaStreamNonBlocking));
    for (auto& e : sd.ev) DS_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  *out = &sd;
  return DS_OK;
}
int edge(cudaStream_t from, cudaStream_t to, cudaEvent_t ev) {  // `to` waits for `from`'s work so far
  DS_CUDA_TRY(cudaEventRecord(ev, from));
  DS_CUDA_TRY(cudaStreamWaitEvent(to, ev, 0));
  return DS_OK;
}

// splits so that tiles * splits fills ONE wave of co-resident CTAs (148 SMs x the tile
// width's CTAs per SM) without spilling over it — a few CTAs past a full wave run as a
// whole extra CTA duration (conv4's weight gradient was 306 CTAs on 296 slots); each split
// >= 4 k-steps, slabs fit. `bn` = the kernel's tile width (0: gemm_pick_bn(N)); the stacked
// weight-gradient taps run ONE N-wide tile (240 = 5 taps x 48), not N / gemm_pick_bn(N).
uint32_t pick_splits(uint32_t M, uint32_t N, uint64_t K, uint32_t ntaps = 1, uint32_t bn = 0) {
  if (bn == 0) bn = gemm_pick_bn(N);
  const uint64_t tiles = 1ull * ((N + bn - 1) / bn) * ((M + 127) / 128) * ntaps;
  const uint64_t slots = 148ull * gemm_ctas_per_sm(bn);
  if (tiles >= 148) return 1;
  uint32_t sp = static_cast<uint32_t>(std::max<uint64_t>(1, slots / tiles));
  sp = static_cast<uint32_t>(std::min<uint64_t>(sp, std::max<uint64_t>(1, K / 128)));
  while (sp > 1 && 1ull * sp * M * N * ntaps > kPartFloats) --sp;
  return sp;
}

GemmEpilogue epi(const Ctx& c, float* D, uint64_t ldd, float scale, const float* bias_n, bool relu,
                 const float* mask = nullptr, uint64_t ldm = 0) {
  GemmEpilogue ep;
  ep.D = D;
  ep.ldd = ldd;
  ep.scale = scale;
  ep.bias_n = bias_n;
  ep.relu = relu;
  ep.mask = mask;
  ep.ldm = ldm;
  ep.gate = c.gate;
  return ep;
}

int gemm(const Ctx& c, const float* A, uint64_t lda, const float* B, uint64_t ldb, float* D, uint64_t ldd, uint32_t M,
         uint32_t N, uint32_t K, float scale, const float* bias_n, bool relu, const float* mask = nullptr,
         uint64_t ldm = 0) {
  const uint32_t sp = pick_splits(M, N, K);
  DS_TRY(launch_gemm_tf32(A, lda, B, ldb, M, N, K, epi(c, D, ldd, scale, bias_n, relu, mask, ldm), sp, c.part, c.s));
  const cudaStream_t s_ = c.s;
  KDONE(sp > 1 ? 2 : 1);
  return DS_OK;
}

int transpose(const Ctx& c, const float* in, uint64_t rows, uint32_t cols, uint64_t ld_in, float* out, uint64_t ld_out) {
  const cudaStream_t s_ = c.s;
  dim3 grid(static_cast<unsigned>((rows + 31) / 32), (cols + 31) / 32);
  transpose_kernel<<<grid, 256, 0, c.s>>>(in, rows, cols, ld_in, out, ld_out, c.gate);
  KDONE(1);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

int colsum(const Ctx& c, const float* d, uint64_t rows, uint32_t N, uint64_t ld, float scale, float* out, float* bpart) {
  const cudaStream_t s_ = c.s;
  const uint32_t ntile = (N + 31) / 32;
  // about 4 blocks per SM, parts of >= 64 rows; bpart holds 4096 * 512 floats
  uint32_t nparts = static_cast<uint32_t>(std::min<uint64_t>(std::max<uint64_t>(1, 592 / ntile), (rows + 63) / 64));
  nparts = std::min<uint32_t>(nparts, (4096u * 512u) / N);
  const uint64_t rpp = (rows + nparts - 1) / nparts;
  colsum_part_kernel<<<dim3(ntile, nparts), dim3(32, 8), 0, c.s>>>(d, rows, N, ld, rpp, bpart, c.gate);
  colsum_final_kernel<<<(N + 7) / 8, 256, 0, c.s>>>(bpart, nparts, N, scale, out, c.flags, c.gate);
  KDONE(2);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

// transpose (out[c][r] = in[r][c], ld_in = cols) and the bias gradient
// bias[n] = scale * sum_r in[r][n] from one read of `in`
int transpose_colsum(const Ctx& c, const float* in, uint64_t rows, uint32_t cols, float* out, uint64_t ld_out,
                     float scale, float* bias, float* bpart) {
  const cudaStream_t s_ = c.s;
  const uint32_t ntile = (cols + 31) / 32;
  uint64_t gx = std::max<uint32_t>(1, 1184 / ntile);  // ~8 resident blocks per SM
  gx = std::min<uint64_t>(gx, (rows + 31) / 32);
  gx = std::min<uint64_t>(gx, (4096ull * 512ull) / cols);
  transpose_colsum_kernel<<<dim3(static_cast<unsigned>(gx), ntile), 256, 0, c.s>>>(in, rows, cols, out, ld_out, bpart,
                                                                                    c.gate);
  colsum_final_kernel<<<(cols + 7) / 8, 256, 0, c.s>>>(bpart, static_cast<uint32_t>(gx), cols, scale, bias, c.flags,
                                                       c.gate);
  KDONE(2);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

int zero(const Ctx& c, float* p, uint64_t floats) {
  DS_CUDA_TRY(cudaMemsetAsync(p, 0, floats * 4, c.s));
  return DS_OK;
}

struct BorderSpec {
  float* p;
  uint32_t Hp, pad, H, C;
};
// clear only the borders of padded maps (the interiors are fully rewritten before they are read)
int zero_borders(const Ctx& c, uint32_t R, std::initializer_list<BorderSpec> maps) {
  BorderMaps bm{};
  uint32_t blocks = 0;
  for (const BorderSpec& m : maps) {
    if (bm.n == 6) return set_error(DS_E_CONTRACT, "zero_borders: at most 6 maps");
    bm.p[bm.n] = m.p, bm.Hp[bm.n] = m.Hp, bm.pad[bm.n] = m.pad, bm.H[bm.n] = m.H, bm.C[bm.n] = m.C;
    bm.first[bm.n] = blocks;
    blocks += R * m.Hp;
    ++bm.n;
  }
  bm.first[bm.n] = blocks;
  zero_borders_kernel<<<blocks, 256, 0, c.s>>>(bm, c.gate);
  ++t_launches;
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

int zero_border(const Ctx& c, float* p, uint32_t R, uint32_t Hp, uint32_t pad, uint32_t H, uint32_t C) {
  zero_border_kernel<<<R * Hp, 256, 0, c.s>>>(p, Hp, pad, H, C, c.gate);
  ++t_launches;
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

// pixel shift of tap (ky, kx) on the padded grid of side Hp
int32_t shift(const ConvSpec& cs, uint32_t t) {
  return (static_cast<int32_t>(t / cs.K) - static_cast<int32_t>(cs.pad)) * static_cast<int32_t>(cs.Hp) +
         (static_cast<int32_t>(t % cs.K) - static_cast<int32_t>(cs.pad));
}

// conv forward over the padded input `in` ([R*Hp*Hp][Cin]): out = relu(conv + b) at the
// interior rows, unpadded (out_padded = false) or on the same padded grid
int conv_fwd(const Ctx& c, const ConvSpec& cs, uint32_t R, const float* in, const float* Wp, const float* bias,
             float* out, bool out_padded) {
  const cudaStream_t s_ = c.s;
  const uint32_t G = R * cs.Hp * cs.Hp, Kg = cs.Kg(), cog = cs.cog(), cig = cs.cig();
  for (uint32_t gi = 0; gi < cs.g; ++gi) {
    GemmTaps tp;
    tp.n = static_cast<int32_t>(cs.KK());
    tp.kt = cig;
    for (uint32_t t = 0; t < cs.KK(); ++t) {
      tp.a_row[t] = shift(cs, t);
      tp.a_col[t] = static_cast<int32_t>(gi * cig);
      tp.b_row[t] = 0;
      tp.b_col[t] = static_cast<int32_t>(t * cig);
    }
    const GemmOperand A{in, G, cs.Cin, cs.Cin}, B{Wp + 1ull * gi * cog * Kg, cog, Kg, Kg};
    GemmEpilogue ep = epi(c, out + gi * cog, cs.Cout, 1.f, bias + gi * cog, true);
    ep.map_Hp = cs.Hp, ep.map_pad = cs.pad, ep.map_H = cs.H, ep.map_out_padded = out_padded;
    DS_TRY(launch_gemm(A, B, G, cog, 0, &tp, ep, 1, nullptr, c.s));
    KDONE(1);
  }
  return DS_OK;
}

// conv data gradient: din = sum_t dout[i - d_t] . WpT[t]^T (ReLU-masked by `mask`, same
// layout as din), dout on the padded grid with a zero border; din at the interior rows
int conv_dgrad(const Ctx& c, const ConvSpec& cs, uint32_t R, const float* dout, const float* WpT, float* din,
               bool din_padded, const float* mask) {
  const cudaStream_t s_ = c.s;
  const uint32_t G = R * cs.Hp * cs.Hp, Kg = cs.Kg(), cog = cs.cog(), cig = cs.cig();
  for (uint32_t gi = 0; gi < cs.g; ++gi) {
    GemmTaps tp;
    tp.n = static_cast<int32_t>(cs.KK());
    tp.kt = cog;
    for (uint32_t t = 0; t < cs.KK(); ++t) {
      tp.a_row[t] = -shift(cs, t);
      tp.a_col[t] = static_cast<int32_t>(gi * cog);
      tp.b_row[t] = static_cast<int32_t>(t * cig);
      tp.b_col[t] = 0;
    }
    const GemmOperand A{dout, G, cs.Cout, cs.Cout}, B{WpT + 1ull * gi * Kg * cog, Kg, cog, cog};
    GemmEpilogue ep = epi(c, din + gi * cig, cs.Cin, 1.f, nullptr, false, mask ? mask + gi * cig : nullptr, cs.Cin);
    ep.map_Hp = cs.Hp, ep.map_pad = cs.pad, ep.map_H = cs.H, ep.map_out_padded = din_padded;
    DS_TRY(launch_gemm(A, B, G, cig, 0, &tp, ep, 1, nullptr, c.s));
    KDONE(1);
  }
  return DS_OK;
}

// conv weight gradient from pixel-contiguous maps doutT [Cout][ldT] and the four shifted
// copies inT4 [4][Cin][ldT] (padded grid, ldT >= G + 3): packed [Cout][KK][cig] into wtmp,
// then Caffe order into grad
int conv_wgrad(const Ctx& c, const ConvSpec& cs, uint32_t R, const float* doutT, const float* inT4, uint64_t ldT,
               float scale, float* wtmp, float* grad, bool s2d = false) {
  const cudaStream_t s_ = c.s;
  const uint32_t G = R * cs.Hp * cs.Hp, Kg = cs.Kg(), cog = cs.cog(), cig = cs.cig();
  for (uint32_t gi = 0; gi < cs.g; ++gi) {
    GemmTaps tp;
    tp.n = static_cast<int32_t>(cs.KK());
    tp.per_z = 1;
    tp.d_col_step = cig;
    for (uint32_t t = 0; t < cs.KK(); ++t) {
      const int32_t d = shift(cs, t), sft = (((-d) % 4) + 4) % 4;
      tp.a_row[t] = 0;
      tp.a_col[t] = 0;
      tp.b_row[t] = sft * static_cast<int32_t>(cs.Cin) + static_cast<int32_t>(gi * cig);
      tp.b_col[t] = d + sft;
    }
    const GemmOperand A{doutT + 1ull * gi * cog * ldT, cog, G, ldT}, B{inT4, 4ull * cs.Cin, G + 3, ldT};
    // the GEMM stacks up to 256 / cig taps per CTA along N (launch_gemm); size the split-K
    // for the resulting number of tap groups
    uint32_t tpc = std::min<uint32_t>(cs.KK(), 256 / cig);
    if (!(tpc > 1 && (tpc * cig == 192 || tpc * cig == 240 || tpc * cig == 256))) tpc = 1;
    const uint32_t sp = pick_splits(cog, tpc * cig, G, (cs.KK() + tpc - 1) / tpc, tpc > 1 ? tpc * cig : 0);
    GemmEpilogue ep = epi(c, wtmp + 1ull * gi * cog * Kg, Kg, scale, nullptr, false);
    DS_TRY(launch_gemm(A, B, cog, cig, G, &tp, ep, sp, c.part, c.s));
    KDONE(sp > 1 ? 2 : 1);
  }
  if (s2d)
    unpack_conv1_s2d_kernel<<<nblk(96 * 363), 256, 0, c.s>>>(wtmp, grad, c.flags, c.gate);
  else
    unpack_wgrad_kernel<<<nblk(1ull * cs.Cout * Kg), 256, 0, c.s>>>(wtmp, cs.Cout, cig, cs.K, grad, c.flags, c.gate);
  KDONE(1);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

// forward to the logits w.z [R x Cp]
int alex_forward(const ModelInfo& m, const float* P, const float* X, const uint32_t* idx, uint32_t R, AlexWs& w,
                 const Ctx& c) {
  const cudaStream_t s_ = c.s;
  const Shape sh = shape_of(m);
  const auto& L = m.layers;
  const uint32_t F = m.n_features;
  const uint64_t M2 = 1ull * R * sh.P1 * sh.P1;
  const uint64_t G2 = 1ull * R * sh.Hp2 * sh.Hp2, G3 = 1ull * R * sh.Hp3 * sh.Hp3;
  cudaStream_t s = c.s;
  const uint32_t* gate = c.gate;
  pack_conv1_s2d_kernel<<<nblk(96 * 432), 256, 0, s>>>(P + L[0].w_off, w.w1p, gate);
  KDONE(1);
  for (int l = 0; l < 4; ++l) {
    const ConvSpec cs = conv_spec(sh, l);
    pack_conv_kernel<<<nblk(1ull * cs.Cout * cs.Kg()), 256, 0, s>>>(P + L[l + 1].w_off, cs.Cout, cs.cig(), cs.K, cs.g,
                                                                   w.wp[l], w.wpT[l], gate);
    KDONE(1);
  }
  // padded maps: zero borders (interiors are rewritten below)
  DS_TRY(zero_borders(c, R, {{w.p1p, sh.Hp2, 2, sh.P1, 96}, {w.p2p, sh.Hp3, 1, sh.P2, 256},
                             {w.a3p, sh.Hp3, 1, sh.P2, 384}, {w.a4p, sh.Hp3, 1, sh.P2, 384},
                             {w.a5p, sh.Hp3, 1, sh.P2, 256}}));
  // conv1 (space-to-depth, 3x3 taps) + relu, LRN1, pool1 -> p1p (pad 2)
  s2d_kernel<<<nblk(1ull * R * sh.Hs * sh.Hs * 48), 256, 0, s>>>(X, idx, F, sh.S, R, sh.Hs, w.xs, gate);
  KDONE(1);
  DS_TRY(conv_fwd(c, conv1_spec(sh), R, w.xs, w.w1p, P + L[0].b_off, w.a1, false));
  lrn_maxpool_fwd_kernel<<<static_cast<unsigned>((M2 + 7) / 8), 256, 0, s>>>(w.a1, R, sh.H1, 96, sh.P1, 2, w.p1p,
                                                                           w.arg1, gate);
  KDONE(1);
  // conv2 + relu -> a2 (unpadded), LRN2, pool2 -> p2p (pad 1)
  DS_TRY(conv_fwd(c, conv_spec(sh, 0), R, w.p1p, w.wp[0], P + L[1].b_off, w.a2, false));
  lrn_maxpool_fwd_kernel<<<(R * sh.P2 * sh.P2 + 7) / 8, 256, 0, s>>>(w.a2, R, sh.P1, 256, sh.P2, 1, w.p2p, w.arg2,
                                                                    gate);
  KDONE(1);
  // conv3, conv4, conv5 on the pad-1 grid, pool5 -> p5 (per-row CHW)
  DS_TRY(conv_fwd(c, conv_spec(sh, 1), R, w.p2p, w.wp[1], P + L[2].b_off, w.a3p, true));
  DS_TRY(conv_fwd(c, conv_spec(sh, 2), R, w.a3p, w.wp[2], P + L[3].b_off, w.a4p, true));
  DS_TRY(conv_fwd(c, conv_spec(sh, 3), R, w.a4p, w.wp[3], P + L[4].b_off, w.a5p, true));
  maxpool_fwd_kernel<<<(R * sh.P5 * sh.P5 + 7) / 8, 256, 0, s>>>(w.a5p, R, sh.P2, 256, sh.P5, 1, 0, 1, w.p5, w.arg5, gate);
  KDONE(1);
  // fc6, fc7 (+relu), fc8
  DS_TRY(gemm(c, w.p5, sh.q5, P + L[5].w_off, sh.q5, w.h6, 4096, R, 4096, static_cast<uint32_t>(sh.q5), 1.f,
              P + L[5].b_off, true));
  DS_TRY(gemm(c, w.h6, 4096, P + L[6].w_off, 4096, w.h7, 4096, R, 4096, 4096, 1.f, P + L[6].b_off, true));
  DS_TRY(gemm(c, w.h7, 4096, P + L[7].w_off, 4096, w.z, sh.Cp, R, sh.C, 4096, 1.f, P + L[7].b_off, false));
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

}  // namespace

uint64_t alex_workspace_bytes(const ModelInfo& m, uint32_t R) { return carve_ws(m, R, nullptr).end; }
uint32_t alex_last_launches() { return t_launches; }

int launch_alex_count_hits(const ModelInfo& m, const float* P, const float* X, const uint32_t* y, uint32_t R,
                           void* ws_base, unsigned long long* hits, uint32_t* pred, cudaStream_t s) {
  AlexWs w = carve_ws(m, R, ws_base);
  Ctx c{s, nullptr, w.part, nullptr};
  DS_TRY(alex_forward(m, P, X, nullptr, R, w, c));
  const Shape sh = shape_of(m);
  alex_hits_kernel<<<(R + 127) / 128, 128, 0, s>>>(w.z, sh.Cp, y, R, sh.C, pred, hits);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

int launch_alex_loss_and_grad(const ModelInfo& m, const float* P, const float* X, const uint32_t* idx,
                              const uint32_t* y, uint32_t R, float* grad, double* loss_out, void* ws_base,
                              uint32_t* flags, const uint32_t* gate, cudaStream_t s) {
  const cudaStream_t s_ = s;
  const Shape sh = shape_of(m);
  AlexWs w = carve_ws(m, R, ws_base);
  Ctx c{s, gate, w.part, flags};
  const auto& L = m.layers;
  const uint32_t F = m.n_features, Rp = up4(R);
  const uint64_t M1 = 1ull * R * sh.H1 * sh.H1, M2 = 1ull * R * sh.P1 * sh.P1, M3 = 1ull * R * sh.P2 * sh.P2;
  const uint64_t G2 = 1ull * R * sh.Hp2 * sh.Hp2, G3 = 1ull * R * sh.Hp3 * sh.Hp3;
  const float inv_b = 1.f / static_cast<float>(R);
  if (1ull * R * sh.Hs * sh.Hs * 96 >= (1ull << 31))
    return set_error(DS_E_CONTRACT, "alexnet: at most %llu rows per call",
                     static_cast<unsigned long long>((1ull << 31) / (96ull * sh.Hs * sh.Hs)));
  t_launches = 0;
  Side* sd = nullptr;
  DS_TRY(side_stream(&sd));
  Ctx c2{sd->s, gate, w.part2, flags};  // its own split-K slabs
  if (grad) {  // the FC backward's transposed weights depend only on P: build them beside the forward
    DS_TRY(edge(s, c2.s, sd->ev[0]));
    DS_TRY(transpose(c2, P + L[7].w_off, sh.C, 4096, 4096, w.w8T, sh.Cp));
    DS_TRY(transpose(c2, P + L[6].w_off, 4096, 4096, 4096, w.w7T, 4096));
    DS_TRY(transpose(c2, P + L[5].w_off, 4096, static_cast<uint32_t>(sh.q5), sh.q5, w.w6T, 4096));
  }
  DS_TRY(alex_forward(m, P, X, idx, R, w, c));
  softmax_ce_warp_kernel<<<(R + 7) / 8, 256, 0, s>>>(w.z, sh.Cp, y, idx, R, sh.C, w.loss_rows, grad ? w.dz : nullptr,
                                                     flags, gate);
  alex_loss_mean_kernel<<<1, 1, 0, s>>>(w.loss_rows, R, loss_out, flags, gate);
  KDONE(2);
  DS_CUDA_TRY(cudaGetLastError());
  if (!grad) return DS_OK;
  DS_TRY(edge(c2.s, s, sd->ev[1]));  // join: the transposed FC weights are ready

  // ---- fc8, fc7, fc6: dW = dh^T h / R and db on the side stream; dh_prev = dh W (ReLU-masked)
  // on the main stream ---------------------------------------------------------------------
  DS_TRY(edge(s, c2.s, sd->ev[8]));
  DS_TRY(transpose(c2, w.dz, R, sh.Cp, sh.Cp, w.zT, Rp));
  DS_TRY(transpose(c2, w.h7, R, 4096, 4096, w.h7T, Rp));
  DS_TRY(gemm(c2, w.zT, Rp, w.h7T, Rp, grad + L[7].w_off, 4096, sh.C, 4096, R, inv_b, nullptr, false));
  DS_TRY(colsum(c2, w.dz, R, sh.C, sh.Cp, inv_b, grad + L[7].b_off, w.bpart));
  DS_TRY(gemm(c, w.dz, sh.Cp, w.w8T, sh.Cp, w.dh7, 4096, R, 4096, sh.C, 1.f, nullptr, false, w.h7, 4096));
  DS_TRY(edge(s, c2.s, sd->ev[9]));
  DS_TRY(transpose(c2, w.dh7, R, 4096, 4096, w.dh7T, Rp));
  DS_TRY(transpose(c2, w.h6, R, 4096, 4096, w.h6T, Rp));
  DS_TRY(gemm(c2, w.dh7T, Rp, w.h6T, Rp, grad + L[6].w_off, 4096, 4096, 4096, R, inv_b, nullptr, false));
  DS_TRY(colsum(c2, w.dh7, R, 4096, 4096, inv_b, grad + L[6].b_off, w.bpart));
  DS_TRY(gemm(c, w.dh7, 4096, w.w7T, 4096, w.dh6, 4096, R, 4096, 4096, 1.f, nullptr, false, w.h6, 4096));
  DS_TRY(edge(s, c2.s, sd->ev[10]));
  DS_TRY(transpose(c2, w.dh6, R, 4096, 4096, w.dh6T, Rp));
  DS_TRY(transpose(c2, w.p5, R, static_cast<uint32_t>(sh.q5), sh.q5, w.p5T, Rp));
  DS_TRY(gemm(c2, w.dh6T, Rp, w.p5T, Rp, grad + L[5].w_off, sh.q5, 4096, static_cast<uint32_t>(sh.q5), R, inv_b,
              nullptr, false));
  DS_TRY(colsum(c2, w.dh6, R, 4096, 4096, inv_b, grad + L[5].b_off, w.bpart));
  DS_TRY(gemm(c, w.dh6, 4096, w.w6T, 4096, w.dp5, sh.q5, R, static_cast<uint32_t>(sh.q5), 4096, 1.f, nullptr, false));

  // ---- conv5 .. conv2 on the padded grids ------------------------------------------------
  DS_TRY(zero_borders(c, R, {{w.dc5p, sh.Hp3, 1, sh.P2, 256}, {w.dc4p, sh.Hp3, 1, sh.P2, 384},
                             {w.dc3p, sh.Hp3, 1, sh.P2, 384}, {w.dc2p, sh.Hp2, 2, sh.P1, 256},
                             {w.dc1p, sh.Hs, 1, sh.H1, 96}, {w.dp2p, sh.Hp3, 1, sh.P2, 256}}));
  // pool5 backward (per-row CHW pooled map) with the ReLU5 mask (a5p) -> dc5p
  maxpool_bwd_kernel<<<static_cast<unsigned>((M3 + 7) / 8), 256, 0, s>>>(w.dp5, w.arg5, R, sh.P2, 256, sh.P5, 0, 1, 1, w.a5p,
                                                                w.dc5p, gate);
  KDONE(1);
  const float* in_maps[4] = {w.p1p, w.p2p, w.a3p, w.a4p};
  float* dout_maps[4] = {w.dc2p, w.dc3p, w.dc4p, w.dc5p};
  for (int l = 3; l >= 0; --l) {
    const ConvSpec cs = conv_spec(sh, l);
    const uint64_t G = 1ull * R * cs.Hp * cs.Hp, ldT = up4(static_cast<uint32_t>(G + 3));
    float* dout = dout_maps[l];
    // side stream: bias gradient (border rows are zero) and the weight gradient from
    // pixel-contiguous copies, beside the main stream's data gradient of the same layer
    DS_TRY(edge(s, c2.s, sd->ev[2 + l]));
    DS_TRY(transpose_colsum(c2, dout, G, cs.Cout, w.trA, ldT, inv_b, grad + L[l + 1].b_off, w.bpart));
    {
      dim3 grid(static_cast<unsigned>((ldT + 31) / 32), (cs.Cin + 31) / 32);
      transpose_shift4_kernel<<<grid, 256, 0, c2.s>>>(in_maps[l], G, cs.Cin, w.trB, ldT, gate);
      KDONE(1);
    }
    DS_TRY(conv_wgrad(c2, cs, R, w.trA, w.trB, ldT, inv_b, w.wtmp, grad + L[l + 1].w_off));
    // data gradient
    if (l >= 2) {  // into relu(conv3 / conv4): masked, same padded grid
      DS_TRY(conv_dgrad(c, cs, R, dout, w.wpT[l], dout_maps[l - 1], true, in_maps[l]));
    } else if (l == 1) {  // into pool2(LRN2(relu(conv2))): d(p2p), pool2 bwd, LRN2 bwd -> dc2p
      DS_TRY(conv_dgrad(c, cs, R, dout, w.wpT[l], w.dp2p, true, nullptr));
      pool_lrn_bwd_relu_kernel<<<static_cast<unsigned>((M2 + 7) / 8), 256, 0, s>>>(w.dp2p, w.arg2, w.a2, R, sh.P1, 256,
                                                                             sh.P2, 1, 2, sh.Hp2, w.dc2p, gate);
      KDONE(1);
    } else {  // into pool1(LRN1(relu(conv1))): d(p1) unpadded, pool1 bwd, LRN1 bwd -> dc1p
      DS_TRY(conv_dgrad(c, cs, R, dout, w.wpT[l], w.dp1, false, nullptr));
      pool_lrn_bwd_relu_kernel<<<static_cast<unsigned>((M1 + 7) / 8), 256, 0, s>>>(w.dp1, w.arg1, w.a1, R, sh.H1, 96,
                                                                             sh.P1, 0, 1, sh.Hs, w.dc1p, gate);
      KDONE(1);
    }
  }
  // ---- conv1: bias and weight gradients on the space-to-depth grid (no data gradient) ------
  {
    const ConvSpec cs = conv1_spec(sh);
    const uint64_t G1 = 1ull * R * sh.Hs * sh.Hs, ldT = up4(static_cast<uint32_t>(G1 + 3));
    DS_TRY(edge(s, c2.s, sd->ev[6]));
    DS_TRY(transpose_colsum(c2, w.dc1p, G1, 96, w.trA, ldT, inv_b, grad + L[0].b_off, w.bpart));
    dim3 grid(static_cast<unsigned>((ldT + 31) / 32), (48 + 31) / 32);
    transpose_shift4_kernel<<<grid, 256, 0, c2.s>>>(w.xs, G1, 48, w.trB, ldT, gate);
    KDONE(1);
    DS_TRY(conv_wgrad(c2, cs, R, w.trA, w.trB, ldT, inv_b, w.wtmp, grad + L[0].w_off, true));
    DS_TRY(edge(c2.s, s, sd->ev[7]));  // join: every gradient is written when the main stream moves on
  }
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

}  // namespace dsb
