// alexnet.cu — the AlexNet-shaped convnet of BASELINE config 4 (model kind
// DS_MODEL_ALEXNET; NOT IN THE REFERENCE, f64 oracle in
// oracle/ds_oracle_alex.c). loss_and_grad for R rows.
//
// Layout: activations NHWC ([rows][y][x][c], channels contiguous), so every contraction is
// a K-major GEMM on the tcgen05 tensor cores (gemm_tc.cu, tf32 with f32 accumulation):
//   conv forward   col[M = R*Ho*Wo][g][ky][kx][cg] . Wp_g[Cout_g][ky][kx][cg]^T   (im2col)
//   conv dgrad     dc_g[M][Cout_g] . WpT_g[K_g][Cout_g]^T -> dcol, then col2im (gather)
//   conv wgrad     dcT_g[Cout_g][M] . colT_g[K_g][M]^T     (split-K over the pixels)
//   fc forward     h[R][in] . W[out][in]^T ; dgrad dh . WT^T ; wgrad dhT . hT^T
// conv1 reads the CHW input rows directly (k order = Caffe's (c, ky, kx)); conv2-5 use
// (ky, kx, c) and their weights are repacked each step (tiny). LRN, max-pooling, ReLU
// masks, softmax cross-entropy and the bias sums are HBM-bound elementwise kernels.
// The gradient is the batch mean (scale 1/R in the GEMM epilogues), rounded to f32 like
// the reference's Grad = f32(sum / b). Dropout is omitted (deterministic; see the oracle).
#include <algorithm>

#include "ds_common.cuh"
#include "gemm_tc.cuh"
#include "model.cuh"

namespace dsb {
namespace {

constexpr float kLrnAlpha = 1e-4f, kLrnBeta = 0.75f, kLrnK = 1.f;
constexpr int kLrnN = 5;

thread_local uint32_t t_launches = 0;  // kernels issued by the last loss_and_grad on this thread

inline unsigned nblk(uint64_t n, unsigned t = 256) {
  return static_cast<unsigned>(std::min<uint64_t>((n + t - 1) / t, 148ull * 64));
}
inline uint32_t up4(uint32_t v) { return (v + 3) & ~3u; }

struct Shape {
  uint32_t S, H1, P1, P2, P5, C, Cp;
  uint64_t q5;  // fc6 fan-in
};

Shape shape_of(const ModelInfo& m) {
  Shape s{};
  s.S = m.alex_side;
  s.H1 = (s.S - 11) / 4 + 1;
  auto pooled = [](uint32_t h) { return (h - 3 + 1) / 2 + 1; };  // ceil((h-3)/2)+1
  s.P1 = pooled(s.H1);
  s.P2 = pooled(s.P1);
  s.P5 = pooled(s.P2);
  s.C = m.n_classes;
  s.Cp = up4(s.C);
  s.q5 = 256ull * s.P5 * s.P5;
  return s;
}

// one conv layer of conv2..5 (NHWC input)
struct ConvSpec {
  uint32_t Cin, Cout, K, pad, g, H;  // H = input side = output side (stride 1, same padding)
  uint32_t cig() const { return Cin / g; }
  uint32_t cog() const { return Cout / g; }
  uint32_t Kg() const { return K * K * cig(); }
};

// ---- workspace ---------------------------------------------------------------------
struct AlexWs {
  float *a1, *n1, *p1, *a2, *n2, *p2, *a3, *a4, *a5, *p5, *h6, *h7, *z, *dz;
  uint8_t *arg1, *arg2, *arg5;
  float *dh7, *dh6, *dp5, *dA, *dB;  // dA/dB: ping-pong gradient maps (largest layer)
  float *col, *tr, *part, *wtmp, *bpart;
  float *w1p, *wp[4], *wpT[4], *w6T, *w7T, *w8T, *zT, *h7T, *h6T, *p5T, *dh7T, *dh6T;
  double* loss_rows;
};

const ConvSpec kConv[4] = {{96, 256, 5, 2, 2, 0}, {256, 384, 3, 1, 1, 0}, {384, 384, 3, 1, 2, 0}, {384, 256, 3, 1, 2, 0}};

ConvSpec conv_spec(const Shape& s, int l) {  // l = 0..3 -> conv2..conv5
  ConvSpec c = kConv[l];
  c.H = l == 0 ? s.P1 : s.P2;
  return c;
}

constexpr uint64_t kPartFloats = 24ull << 20;  // split-K slabs

// one carve for sizing (base = nullptr) and for the pointers
AlexWs carve_ws(const ModelInfo& m, uint32_t R, void* base) {
  AlexWs ws{};
  uint8_t* b = static_cast<uint8_t*>(base);
  const Shape s = shape_of(m);
  const uint64_t A1 = 1ull * R * s.H1 * s.H1 * 96, Q1 = 1ull * R * s.P1 * s.P1 * 96, A2 = 1ull * R * s.P1 * s.P1 * 256,
                 Q2 = 1ull * R * s.P2 * s.P2 * 256, A3 = 1ull * R * s.P2 * s.P2 * 384, Q5 = R * s.q5;
  const uint64_t M1 = 1ull * R * s.H1 * s.H1, M2 = 1ull * R * s.P1 * s.P1, M3 = 1ull * R * s.P2 * s.P2;
  const uint64_t col = std::max({up4(static_cast<uint32_t>(M1)) * 364ull, up4(static_cast<uint32_t>(M2)) * 2400ull,
                                 up4(static_cast<uint32_t>(M3)) * 3456ull});
  const uint64_t tr = std::max({96 * (M1 + 4), 256 * (M2 + 4), 384 * (M3 + 4)});
  const uint32_t Rp = up4(R);
  uint64_t off = 0;
  auto f = [&](float*& p, uint64_t n) { p = reinterpret_cast<float*>(b + off); off += (n * 4 + 255) & ~255ull; };
  auto u = [&](uint8_t*& p, uint64_t n) { p = b + off; off += (n + 255) & ~255ull; };
  f(ws.a1, A1), f(ws.n1, A1), f(ws.p1, Q1), u(ws.arg1, Q1);
  f(ws.a2, A2), f(ws.n2, A2), f(ws.p2, Q2), u(ws.arg2, Q2);
  f(ws.a3, A3), f(ws.a4, A3), f(ws.a5, Q2), f(ws.p5, Q5), u(ws.arg5, Q5);
  f(ws.h6, 4096ull * R), f(ws.h7, 4096ull * R), f(ws.z, 1ull * s.Cp * R), f(ws.dz, 1ull * s.Cp * R);
  f(ws.dh7, 4096ull * R), f(ws.dh6, 4096ull * R), f(ws.dp5, Q5), f(ws.dA, A1), f(ws.dB, A1);
  f(ws.col, col), f(ws.tr, tr), f(ws.part, kPartFloats), f(ws.wtmp, 384ull * 2304), f(ws.bpart, 4096ull * 512);
  f(ws.w1p, 96ull * 364);
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
  (void)off;
  return ws;
}

uint64_t ws_bytes(const ModelInfo& m, uint32_t R) {
  // size = end offset of carve_ws's last buffer: carve against a null base
  AlexWs w = carve_ws(m, R, nullptr);
  return reinterpret_cast<uint64_t>(w.loss_rows) + ((R * 8ull + 255) & ~255ull);
}

// ---- kernels -------------------------------------------------------------------------
#define GATE \
  if (gate && *gate) return

// conv1 im2col from CHW input rows (row r = X[idx[r]]): col[m][k], k = (c*11+ky)*11+kx,
// ld 364 (k = 363 zero)
__global__ void im2col_conv1_kernel(const float* __restrict__ X, const uint32_t* __restrict__ idx, uint32_t F,
                                    uint32_t S, uint32_t Ho, uint64_t M, float* __restrict__ col, const uint32_t* gate) {
  GATE;
  const uint64_t total = M * 364;
  for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < total; i += gridDim.x * 256ull) {
    const uint64_t m = i / 364;
    const uint32_t k = static_cast<uint32_t>(i % 364);
    float v = 0.f;
    if (k < 363) {
      const uint32_t c = k / 121, ky = (k / 11) % 11, kx = k % 11;
      const uint32_t r = static_cast<uint32_t>(m / (1ull * Ho * Ho)), pix = static_cast<uint32_t>(m % (1ull * Ho * Ho));
      const uint32_t oy = pix / Ho, ox = pix % Ho;
      const uint64_t row = idx ? idx[r] : r;
      v = __ldg(X + row * F + (1ull * c * S + oy * 4 + ky) * S + ox * 4 + kx);
    }
    col[i] = v;
  }
}

// conv1 im2col transposed: colT[k][m] (ld ldT), for the weight gradient
__global__ void im2colT_conv1_kernel(const float* __restrict__ X, const uint32_t* __restrict__ idx, uint32_t F,
                                     uint32_t S, uint32_t Ho, uint64_t M, uint64_t ldT, float* __restrict__ colT,
                                     const uint32_t* gate) {
  GATE;
  const uint64_t total = 363ull * M;
  for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < total; i += gridDim.x * 256ull) {
    const uint32_t k = static_cast<uint32_t>(i / M);
    const uint64_t m = i % M;
    const uint32_t c = k / 121, ky = (k / 11) % 11, kx = k % 11;
    const uint32_t r = static_cast<uint32_t>(m / (1ull * Ho * Ho)), pix = static_cast<uint32_t>(m % (1ull * Ho * Ho));
    const uint32_t oy = pix / Ho, ox = pix % Ho;
    const uint64_t row = idx ? idx[r] : r;
    colT[k * ldT + m] = __ldg(X + row * F + (1ull * c * S + oy * 4 + ky) * S + ox * 4 + kx);
  }
}

// NHWC im2col, stride 1, same padding: col[m][g][ky][kx][cg] (ld = g*K*K*cg); float4 over c
__global__ void im2col_nhwc_kernel(const float* __restrict__ in, uint32_t R, uint32_t H, uint32_t Cin, uint32_t K,
                                   uint32_t pad, uint32_t g, float* __restrict__ col, const uint32_t* gate) {
  GATE;
  const uint32_t cg = Cin / g, cg4 = cg / 4, KK = K * K;
  const uint64_t ld = 1ull * g * KK * cg;
  const uint64_t total = 1ull * R * H * H * g * KK * cg4;
  for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < total; i += gridDim.x * 256ull) {
    const uint32_t c4 = static_cast<uint32_t>(i % cg4);
    uint64_t t = i / cg4;
    const uint32_t kk = static_cast<uint32_t>(t % KK);
    t /= KK;
    const uint32_t gi = static_cast<uint32_t>(t % g);
    const uint64_t m = t / g;
    const uint32_t x = static_cast<uint32_t>(m % H), y = static_cast<uint32_t>((m / H) % H);
    const uint64_t r = m / (1ull * H * H);
    const int iy = static_cast<int>(y + kk / K) - static_cast<int>(pad), ix = static_cast<int>(x + kk % K) - static_cast<int>(pad);
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (iy >= 0 && iy < static_cast<int>(H) && ix >= 0 && ix < static_cast<int>(H))
      v = __ldg(reinterpret_cast<const float4*>(in + ((r * H + iy) * H + ix) * Cin + gi * cg) + c4);
    *reinterpret_cast<float4*>(col + m * ld + (1ull * gi * KK + kk) * cg + c4 * 4) = v;
  }
}

// NHWC im2col transposed for one group: colT[k][m] (k = (ky*K+kx)*cg + c, ld ldT).
// 32x32 smem tile: read along c (coalesced), write along m (coalesced).
__global__ void im2colT_nhwc_kernel(const float* __restrict__ in, uint32_t R, uint32_t H, uint32_t Cin, uint32_t K,
                                    uint32_t pad, uint32_t g, uint32_t gi, uint64_t ldT, float* __restrict__ colT,
                                    const uint32_t* gate) {
  GATE;
  __shared__ float tile[32][33];
  const uint32_t cg = Cin / g, Kg = K * K * cg;
  const uint64_t M = 1ull * R * H * H;
  const uint64_t m0 = blockIdx.x * 32ull;
  const uint32_t k0 = blockIdx.y * 32;
  // load: thread (ty, tx): m = m0 + ty (rows 0..31 in steps of 8), k = k0 + tx
  for (uint32_t ty = threadIdx.y; ty < 32; ty += 8) {
    const uint64_t m = m0 + ty;
    const uint32_t k = k0 + threadIdx.x;
    float v = 0.f;
    if (m < M && k < Kg) {
      const uint32_t c = k % cg, kk = k / cg;
      const uint32_t x = static_cast<uint32_t>(m % H), y = static_cast<uint32_t>((m / H) % H);
      const uint64_t r = m / (1ull * H * H);
      const int iy = static_cast<int>(y + kk / K) - static_cast<int>(pad), ix = static_cast<int>(x + kk % K) - static_cast<int>(pad);
      if (iy >= 0 && iy < static_cast<int>(H) && ix >= 0 && ix < static_cast<int>(H))
        v = __ldg(in + ((r * H + iy) * H + ix) * Cin + gi * cg + c);
    }
    tile[ty][threadIdx.x] = v;
  }
  __syncthreads();
  for (uint32_t ty = threadIdx.y; ty < 32; ty += 8) {
    const uint32_t k = k0 + ty;
    const uint64_t m = m0 + threadIdx.x;
    if (k < Kg && m < M) colT[k * ldT + m] = tile[threadIdx.x][ty];
  }
}

// col2im (gather) for stride-1 same-padding convs: dX[r][y][x][c] = sum over (ky, kx) of
// dcol[(r, y+pad-ky, x+pad-kx)][g][ky][kx][c'] ; optional ReLU mask (forward activation)
__global__ void col2im_nhwc_kernel(const float* __restrict__ dcol, uint32_t R, uint32_t H, uint32_t Cin, uint32_t K,
                                   uint32_t pad, uint32_t g, const float* __restrict__ mask, float* __restrict__ dX,
                                   const uint32_t* gate) {
  GATE;
  const uint32_t cg = Cin / g, KK = K * K;
  const uint64_t ld = 1ull * g * KK * cg;
  const uint64_t total = 1ull * R * H * H * Cin;
  for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < total; i += gridDim.x * 256ull) {
    const uint32_t c = static_cast<uint32_t>(i % Cin);
    const uint64_t p = i / Cin;
    if (mask && !(mask[i] > 0.f)) {
      dX[i] = 0.f;
      continue;
    }
    const uint32_t x = static_cast<uint32_t>(p % H), y = static_cast<uint32_t>((p / H) % H);
    const uint64_t r = p / (1ull * H * H);
    const uint32_t gi = c / cg, cc = c % cg;
    float s = 0.f;
    for (uint32_t ky = 0; ky < K; ++ky) {
      const int oy = static_cast<int>(y + pad) - static_cast<int>(ky);
      if (oy < 0 || oy >= static_cast<int>(H)) continue;
      for (uint32_t kx = 0; kx < K; ++kx) {
        const int ox = static_cast<int>(x + pad) - static_cast<int>(kx);
        if (ox < 0 || ox >= static_cast<int>(H)) continue;
        const uint64_t m = (r * H + oy) * H + ox;
        s += dcol[m * ld + (1ull * gi * KK + ky * K + kx) * cg + cc];
      }
    }
    dX[i] = s;
  }
}

// out[c][r] = in[r][c] for a [rows x cols] matrix (ld_in, ld_out), 32x32 tiles
__global__ void transpose_kernel(const float* __restrict__ in, uint64_t rows, uint32_t cols, uint64_t ld_in,
                                 float* __restrict__ out, uint64_t ld_out, const uint32_t* gate) {
  GATE;
  __shared__ float tile[32][33];
  const uint64_t r0 = blockIdx.x * 32ull;
  const uint32_t c0 = blockIdx.y * 32;
  for (uint32_t ty = threadIdx.y; ty < 32; ty += 8) {
    const uint64_t r = r0 + ty;
    const uint32_t c = c0 + threadIdx.x;
    tile[ty][threadIdx.x] = (r < rows && c < cols) ? in[r * ld_in + c] : 0.f;
  }
  __syncthreads();
  for (uint32_t ty = threadIdx.y; ty < 32; ty += 8) {
    const uint32_t c = c0 + ty;
    const uint64_t r = r0 + threadIdx.x;
    if (c < cols && r < rows) out[c * ld_out + r] = tile[threadIdx.x][ty];
  }
}

// Caffe conv weight [Cout][cg][K][K] -> Wp [Cout][K][K][cg] and per group WpT_g [Kg][Cout_g]
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

// conv1 weights [96][363] -> [96][364] (zero pad)
__global__ void pack_conv1_kernel(const float* __restrict__ W, float* __restrict__ Wp, const uint32_t* gate) {
  GATE;
  for (uint32_t i = blockIdx.x * 256 + threadIdx.x; i < 96 * 364; i += gridDim.x * 256) {
    const uint32_t co = i / 364, k = i % 364;
    Wp[i] = k < 363 ? W[co * 363 + k] : 0.f;
  }
}

// packed weight gradient [Cout_g][(ky,kx,c)] of group gi -> Caffe order in grad
__global__ void unpack_wgrad_kernel(const float* __restrict__ dWp, uint32_t cog, uint32_t cg, uint32_t K, uint32_t gi,
                                    float* __restrict__ grad, const uint32_t* gate) {
  GATE;
  const uint32_t KK = K * K, Kg = KK * cg;
  for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < 1ull * cog * Kg; i += gridDim.x * 256ull) {
    const uint32_t col = static_cast<uint32_t>(i / Kg), k = static_cast<uint32_t>(i % Kg);
    const uint32_t kk = k / cg, c = k % cg;
    grad[(1ull * (gi * cog + col) * cg + c) * KK + kk] = dWp[i];
  }
}

// LRN across channels (NHWC): y = x * (k + a/n sum_{|c'-c|<=2} x_c'^2)^-b
__global__ void lrn_fwd_kernel(const float* __restrict__ x, uint64_t pixels, uint32_t C, float* __restrict__ y,
                               const uint32_t* gate) {
  GATE;
  const uint64_t total = pixels * C;
  for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < total; i += gridDim.x * 256ull) {
    const uint32_t c = static_cast<uint32_t>(i % C);
    const float* px = x + (i - c);
    float ss = 0.f;
    const int lo = max(0, static_cast<int>(c) - kLrnN / 2), hi = min(static_cast<int>(C) - 1, static_cast<int>(c) + kLrnN / 2);
    for (int j = lo; j <= hi; ++j) ss += px[j] * px[j];
    const float sc = kLrnK + kLrnAlpha / kLrnN * ss;
    y[i] = px[c] * __powf(sc, -kLrnBeta);
  }
}

// LRN backward, scale recomputed from x; the result is masked by ReLU (x = relu output > 0)
__global__ void lrn_bwd_relu_kernel(const float* __restrict__ x, const float* __restrict__ dy, uint64_t pixels,
                                    uint32_t C, float* __restrict__ dx, const uint32_t* gate) {
  GATE;
  const uint64_t total = pixels * C;
  for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < total; i += gridDim.x * 256ull) {
    const uint32_t c = static_cast<uint32_t>(i % C);
    const float* px = x + (i - c);
    const float* pd = dy + (i - c);
    if (!(px[c] > 0.f)) {
      dx[i] = 0.f;
      continue;
    }
    float acc = 0.f, own = 0.f;
    const int lo = max(0, static_cast<int>(c) - kLrnN / 2), hi = min(static_cast<int>(C) - 1, static_cast<int>(c) + kLrnN / 2);
    for (int j = lo; j <= hi; ++j) {
      const int l2 = max(0, j - kLrnN / 2), h2 = min(static_cast<int>(C) - 1, j + kLrnN / 2);
      float ss = 0.f;
      for (int t = l2; t <= h2; ++t) ss += px[t] * px[t];
      const float sc = kLrnK + kLrnAlpha / kLrnN * ss;
      const float p = __powf(sc, -kLrnBeta);
      if (j == static_cast<int>(c)) own = p;
      acc += pd[j] * px[j] * p / sc;  // dy_j * y_j / scale_j
    }
    dx[i] = pd[c] * own - 2.f * kLrnAlpha * kLrnBeta / kLrnN * px[c] * acc;
  }
}

// MAX 3x3/2 ceil-mode (NHWC in); out NHWC, or per-row CHW when chw != 0 (fc6 input).
// arg = window position (0..8) of the first maximum in scan order.
__global__ void maxpool_fwd_kernel(const float* __restrict__ in, uint32_t R, uint32_t H, uint32_t C, uint32_t Ho,
                                   int chw, float* __restrict__ out, uint8_t* __restrict__ arg, const uint32_t* gate) {
  GATE;
  const uint64_t total = 1ull * R * Ho * Ho * C;
  for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < total; i += gridDim.x * 256ull) {
    const uint32_t c = static_cast<uint32_t>(i % C);
    const uint64_t p = i / C;
    const uint32_t px = static_cast<uint32_t>(p % Ho), py = static_cast<uint32_t>((p / Ho) % Ho);
    const uint64_t r = p / (1ull * Ho * Ho);
    const uint32_t hs = py * 2, ws = px * 2, he = min(hs + 3, H), we = min(ws + 3, H);
    float best = -INFINITY;
    uint32_t bi = 0;
    for (uint32_t h = hs; h < he; ++h)
      for (uint32_t w = ws; w < we; ++w) {
        const float v = in[((r * H + h) * H + w) * C + c];
        if (v > best) best = v, bi = (h - hs) * 3 + (w - ws);
      }
    const uint64_t o = chw ? (r * C + c) * Ho * Ho + py * Ho + px : i;
    out[o] = best;
    arg[o] = static_cast<uint8_t>(bi);
  }
}

// gather form of the max-pool backward: din[r][y][x][c] = sum of dout over the windows
// whose maximum sat at (y, x); optional ReLU mask (x > 0 of the pooled map's source)
__global__ void maxpool_bwd_kernel(const float* __restrict__ dout, const uint8_t* __restrict__ arg, uint32_t R,
                                   uint32_t H, uint32_t C, uint32_t Ho, int chw, const float* __restrict__ mask,
                                   float* __restrict__ din, const uint32_t* gate) {
  GATE;
  const uint64_t total = 1ull * R * H * H * C;
  for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < total; i += gridDim.x * 256ull) {
    const uint32_t c = static_cast<uint32_t>(i % C);
    const uint64_t p = i / C;
    const uint32_t x = static_cast<uint32_t>(p % H), y = static_cast<uint32_t>((p / H) % H);
    const uint64_t r = p / (1ull * H * H);
    float s = 0.f;
    if (!mask || mask[i] > 0.f) {
      const uint32_t py0 = y >= 2 ? (y - 1) / 2 : 0, py1 = min(y / 2, Ho - 1);
      const uint32_t px0 = x >= 2 ? (x - 1) / 2 : 0, px1 = min(x / 2, Ho - 1);
      for (uint32_t py = py0; py <= py1; ++py)
        for (uint32_t px = px0; px <= px1; ++px) {
          const uint64_t o = chw ? (r * C + c) * Ho * Ho + py * Ho + px : ((r * Ho + py) * Ho + px) * C + c;
          if (arg[o] == (y - py * 2) * 3 + (x - px * 2)) s += dout[o];
        }
    }
    din[i] = s;
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

// column sums of d[rows][N] (ld) -> part[block][N]; then fixed-order final sum * scale
__global__ void colsum_part_kernel(const float* __restrict__ d, uint64_t rows, uint32_t N, uint64_t ld,
                                   uint64_t rows_per_block, float* __restrict__ part, const uint32_t* gate) {
  GATE;
  const uint64_t r0 = blockIdx.y * rows_per_block, r1 = min(rows, r0 + rows_per_block);
  for (uint32_t n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x) {
    float s = 0.f;
    for (uint64_t r = r0; r < r1; ++r) s += d[r * ld + n];
    part[1ull * blockIdx.y * N + n] = s;
  }
}
__global__ void colsum_final_kernel(const float* __restrict__ part, uint32_t nparts, uint32_t N, float scale,
                                    float* __restrict__ out, uint32_t* flags, const uint32_t* gate) {
  GATE;
  for (uint32_t n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x) {
    float s = 0.f;
    for (uint32_t p = 0; p < nparts; ++p) s += part[1ull * p * N + n];
    const float v = s * scale;
    if (!isfinite(v)) atomicOr(flags, DS_FLAG_GRAD_NONFINITE);
    out[n] = v;
  }
}

// ---- host helpers --------------------------------------------------------------------
struct Ctx {
  cudaStream_t s;
  const uint32_t* gate;
  float* part;
  uint32_t* flags;
};

// splits so that tiles * splits covers the SMs, each split >= 4 k-steps, slabs fit `part`
uint32_t pick_splits(uint32_t M, uint32_t N, uint32_t K) {
  const uint32_t bn = gemm_pick_bn(N);
  const uint64_t tiles = 1ull * ((N + bn - 1) / bn) * ((M + 127) / 128);
  if (tiles >= 148) return 1;
  uint32_t sp = static_cast<uint32_t>((148 + tiles - 1) / tiles);
  sp = std::min<uint32_t>(sp, std::max<uint32_t>(1, K / 128));
  while (sp > 1 && 1ull * sp * M * N > kPartFloats) --sp;
  return sp;
}

int gemm(const Ctx& c, const float* A, uint64_t lda, const float* B, uint64_t ldb, float* D, uint64_t ldd, uint32_t M,
         uint32_t N, uint32_t K, float scale, const float* bias_n, bool relu, const float* mask = nullptr,
         uint64_t ldm = 0, bool allow_split = true) {
  GemmEpilogue ep;
  ep.D = D;
  ep.ldd = ldd;
  ep.scale = scale;
  ep.bias_n = bias_n;
  ep.relu = relu;
  ep.mask = mask;
  ep.ldm = ldm;
  ep.gate = c.gate;
  const uint32_t sp = allow_split ? pick_splits(M, N, K) : 1;
  t_launches += sp > 1 ? 2 : 1;
  return launch_gemm_tf32(A, lda, B, ldb, M, N, K, ep, sp, c.part, c.s);
}

int transpose(const Ctx& c, const float* in, uint64_t rows, uint32_t cols, uint64_t ld_in, float* out, uint64_t ld_out) {
  dim3 grid(static_cast<unsigned>((rows + 31) / 32), (cols + 31) / 32);
  transpose_kernel<<<grid, dim3(32, 8), 0, c.s>>>(in, rows, cols, ld_in, out, ld_out, c.gate); ++t_launches;
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

int colsum(const Ctx& c, const float* d, uint64_t rows, uint32_t N, uint64_t ld, float scale, float* out, float* bpart) {
  const uint32_t nparts = static_cast<uint32_t>(std::min<uint64_t>(512, std::max<uint64_t>(1, rows / 64)));
  const uint64_t rpb = (rows + nparts - 1) / nparts;
  dim3 grid((N + 127) / 128, nparts);
  colsum_part_kernel<<<grid, 128, 0, c.s>>>(d, rows, N, ld, rpb, bpart, c.gate); ++t_launches;
  colsum_final_kernel<<<(N + 127) / 128, 128, 0, c.s>>>(bpart, nparts, N, scale, out, c.flags, c.gate); ++t_launches;
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

}  // namespace

uint64_t alex_workspace_bytes(const ModelInfo& m, uint32_t R) { return ws_bytes(m, R); }
uint32_t alex_last_launches() { return t_launches; }

namespace {

// forward to the logits w.z [R x Cp]
int alex_forward(const ModelInfo& m, const float* P, const float* X, const uint32_t* idx, uint32_t R, AlexWs& w,
                 const Ctx& c) {
  const Shape sh = shape_of(m);
  const auto& L = m.layers;
  const uint32_t F = m.n_features;
  const uint64_t M1 = 1ull * R * sh.H1 * sh.H1, M2 = 1ull * R * sh.P1 * sh.P1, M3 = 1ull * R * sh.P2 * sh.P2;
  cudaStream_t s = c.s;
  const uint32_t* gate = c.gate;
  pack_conv1_kernel<<<nblk(96 * 364), 256, 0, s>>>(P + L[0].w_off, w.w1p, gate); ++t_launches;
  for (int l = 0; l < 4; ++l) {
    const ConvSpec cs = conv_spec(sh, l);
    pack_conv_kernel<<<nblk(1ull * cs.Cout * cs.Kg()), 256, 0, s>>>(P + L[l + 1].w_off, cs.Cout, cs.cig(), cs.K, cs.g,
                                                                   w.wp[l], w.wpT[l], gate); ++t_launches;
  }
  // conv1 + relu
  im2col_conv1_kernel<<<nblk(M1 * 364), 256, 0, s>>>(X, idx, F, sh.S, sh.H1, M1, w.col, gate); ++t_launches;
  DS_TRY(gemm(c, w.col, 364, w.w1p, 364, w.a1, 96, static_cast<uint32_t>(M1), 96, 364, 1.f, P + L[0].b_off, true));
  lrn_fwd_kernel<<<nblk(M1 * 96), 256, 0, s>>>(w.a1, M1, 96, w.n1, gate); ++t_launches;
  maxpool_fwd_kernel<<<nblk(M2 * 96), 256, 0, s>>>(w.n1, R, sh.H1, 96, sh.P1, 0, w.p1, w.arg1, gate); ++t_launches;
  // conv2..5
  const float* in_act[4] = {w.p1, w.p2, w.a3, w.a4};
  float* out_act[4] = {w.a2, w.a3, w.a4, w.a5};
  for (int l = 0; l < 4; ++l) {
    const ConvSpec cs = conv_spec(sh, l);
    const uint64_t Mx = l == 0 ? M2 : M3;
    const uint32_t Kg = cs.Kg(), ldc = Kg * cs.g;
    im2col_nhwc_kernel<<<nblk(Mx * ldc / 4), 256, 0, s>>>(in_act[l], R, cs.H, cs.Cin, cs.K, cs.pad, cs.g, w.col, gate); ++t_launches;
    for (uint32_t gi = 0; gi < cs.g; ++gi)
      DS_TRY(gemm(c, w.col + gi * Kg, ldc, w.wp[l] + 1ull * gi * cs.cog() * Kg, Kg, out_act[l] + gi * cs.cog(), cs.Cout,
                  static_cast<uint32_t>(Mx), cs.cog(), Kg, 1.f, P + L[l + 1].b_off + gi * cs.cog(), true));
    if (l == 0) {
      lrn_fwd_kernel<<<nblk(M2 * 256), 256, 0, s>>>(w.a2, M2, 256, w.n2, gate); ++t_launches;
      maxpool_fwd_kernel<<<nblk(M3 * 256), 256, 0, s>>>(w.n2, R, sh.P1, 256, sh.P2, 0, w.p2, w.arg2, gate); ++t_launches;
    }
  }
  maxpool_fwd_kernel<<<nblk(R * sh.q5), 256, 0, s>>>(w.a5, R, sh.P2, 256, sh.P5, 1, w.p5, w.arg5, gate); ++t_launches;
  // fc6, fc7 (+relu), fc8
  DS_TRY(gemm(c, w.p5, sh.q5, P + L[5].w_off, sh.q5, w.h6, 4096, R, 4096, static_cast<uint32_t>(sh.q5), 1.f,
              P + L[5].b_off, true));
  DS_TRY(gemm(c, w.h6, 4096, P + L[6].w_off, 4096, w.h7, 4096, R, 4096, 4096, 1.f, P + L[6].b_off, true));
  DS_TRY(gemm(c, w.h7, 4096, P + L[7].w_off, 4096, w.z, sh.Cp, R, sh.C, 4096, 1.f, P + L[7].b_off, false, nullptr, 0,
              sh.Cp == sh.C));
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

// predict() (model.cpp:303-318): first maximal logit, hits against labels
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

}  // namespace

int launch_alex_count_hits(const ModelInfo& m, const float* P, const float* X, const uint32_t* y, uint32_t R,
                           void* ws_base, unsigned long long* hits, uint32_t* pred, cudaStream_t s) {
  AlexWs w = carve_ws(m, R, ws_base);
  Ctx c{s, nullptr, w.part, nullptr};
  DS_TRY(alex_forward(m, P, X, nullptr, R, w, c));
  const Shape sh = shape_of(m);
  alex_hits_kernel<<<(R + 127) / 128, 128, 0, s>>>(w.z, sh.Cp, y, R, sh.C, pred, hits); ++t_launches;
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

int launch_alex_loss_and_grad(const ModelInfo& m, const float* P, const float* X, const uint32_t* idx,
                              const uint32_t* y, uint32_t R, float* grad, double* loss_out, void* ws_base,
                              uint32_t* flags, const uint32_t* gate, cudaStream_t s) {
  const Shape sh = shape_of(m);
  AlexWs w = carve_ws(m, R, ws_base);
  Ctx c{s, gate, w.part, flags};
  const auto& L = m.layers;
  const uint32_t F = m.n_features, Rp = up4(R);
  const uint64_t M1 = 1ull * R * sh.H1 * sh.H1, M2 = 1ull * R * sh.P1 * sh.P1, M3 = 1ull * R * sh.P2 * sh.P2;
  const float inv_b = 1.f / static_cast<float>(R);
  t_launches = 0;
  DS_TRY(alex_forward(m, P, X, idx, R, w, c));
  softmax_ce_warp_kernel<<<(R + 7) / 8, 256, 0, s>>>(w.z, sh.Cp, y, idx, R, sh.C, w.loss_rows, grad ? w.dz : nullptr,
                                                     flags, gate); ++t_launches;
  alex_loss_mean_kernel<<<1, 1, 0, s>>>(w.loss_rows, R, loss_out, flags, gate); ++t_launches;
  DS_CUDA_TRY(cudaGetLastError());
  if (!grad) return DS_OK;

  // ---------------- backward ----------------
  // fc8: dW8 = dz^T h7 / R ; db8 ; dh7 = dz W8, masked by h7 > 0
  DS_TRY(transpose(c, w.dz, R, sh.Cp, sh.Cp, w.zT, Rp));
  DS_TRY(transpose(c, w.h7, R, 4096, 4096, w.h7T, Rp));
  DS_TRY(gemm(c, w.zT, Rp, w.h7T, Rp, grad + L[7].w_off, 4096, sh.C, 4096, R, inv_b, nullptr, false));
  DS_TRY(colsum(c, w.dz, R, sh.C, sh.Cp, inv_b, grad + L[7].b_off, w.bpart));
  DS_TRY(transpose(c, P + L[7].w_off, sh.C, 4096, 4096, w.w8T, sh.Cp));
  DS_TRY(gemm(c, w.dz, sh.Cp, w.w8T, sh.Cp, w.dh7, 4096, R, 4096, sh.C, 1.f, nullptr, false, w.h7, 4096));
  // fc7
  DS_TRY(transpose(c, w.dh7, R, 4096, 4096, w.dh7T, Rp));
  DS_TRY(transpose(c, w.h6, R, 4096, 4096, w.h6T, Rp));
  DS_TRY(gemm(c, w.dh7T, Rp, w.h6T, Rp, grad + L[6].w_off, 4096, 4096, 4096, R, inv_b, nullptr, false));
  DS_TRY(colsum(c, w.dh7, R, 4096, 4096, inv_b, grad + L[6].b_off, w.bpart));
  DS_TRY(transpose(c, P + L[6].w_off, 4096, 4096, 4096, w.w7T, 4096));
  DS_TRY(gemm(c, w.dh7, 4096, w.w7T, 4096, w.dh6, 4096, R, 4096, 4096, 1.f, nullptr, false, w.h6, 4096));
  // fc6
  DS_TRY(transpose(c, w.dh6, R, 4096, 4096, w.dh6T, Rp));
  DS_TRY(transpose(c, w.p5, R, static_cast<uint32_t>(sh.q5), sh.q5, w.p5T, Rp));
  DS_TRY(gemm(c, w.dh6T, Rp, w.p5T, Rp, grad + L[5].w_off, sh.q5, 4096, static_cast<uint32_t>(sh.q5), R, inv_b,
              nullptr, false));
  DS_TRY(colsum(c, w.dh6, R, 4096, 4096, inv_b, grad + L[5].b_off, w.bpart));
  DS_TRY(transpose(c, P + L[5].w_off, 4096, static_cast<uint32_t>(sh.q5), sh.q5, w.w6T, 4096));
  DS_TRY(gemm(c, w.dh6, 4096, w.w6T, 4096, w.dp5, sh.q5, R, static_cast<uint32_t>(sh.q5), 4096, 1.f, nullptr, false));
  // pool5 backward (CHW pooled map), masked by a5 > 0 -> dc5 (NHWC)
  float* dcur = w.dA;
  float* dnext = w.dB;
  maxpool_bwd_kernel<<<nblk(M3 * 256), 256, 0, s>>>(w.dp5, w.arg5, R, sh.P2, 256, sh.P5, 1, w.a5, dcur, gate); ++t_launches;
  // conv5, conv4, conv3, conv2
  const float* in_act[4] = {w.p1, w.p2, w.a3, w.a4};
  const float* fwd_out[4] = {w.a2, w.a3, w.a4, w.a5};
  for (int l = 3; l >= 0; --l) {
    const ConvSpec cs = conv_spec(sh, l);
    const uint64_t Mx = l == 0 ? M2 : M3;
    const uint32_t Kg = cs.Kg(), cog = cs.cog(), Mp = up4(static_cast<uint32_t>(Mx));
    // bias gradient: column sums of dc
    DS_TRY(colsum(c, dcur, Mx, cs.Cout, cs.Cout, inv_b, grad + L[l + 1].b_off, w.bpart));
    // weight gradient per group: dcT_g [cog x M] . colT_g [Kg x M]^T
    DS_TRY(transpose(c, dcur, Mx, cs.Cout, cs.Cout, w.tr, Mp));
    for (uint32_t gi = 0; gi < cs.g; ++gi) {
      dim3 grid(static_cast<unsigned>((Mx + 31) / 32), (Kg + 31) / 32);
      im2colT_nhwc_kernel<<<grid, dim3(32, 8), 0, s>>>(in_act[l], R, cs.H, cs.Cin, cs.K, cs.pad, cs.g, gi, Mp, w.col,
                                                       gate); ++t_launches;
      DS_TRY(gemm(c, w.tr + 1ull * gi * cog * Mp, Mp, w.col, Mp, w.wtmp, Kg, cog, Kg, static_cast<uint32_t>(Mx), inv_b,
                  nullptr, false));
      unpack_wgrad_kernel<<<nblk(1ull * cog * Kg), 256, 0, s>>>(w.wtmp, cog, cs.cig(), cs.K, gi, grad + L[l + 1].w_off,
                                                               gate); ++t_launches;
    }
    // data gradient: dcol = dc_g . WpT_g^T, then col2im (+ ReLU mask of the input for conv3..5)
    const uint32_t ldc = Kg * cs.g;
    for (uint32_t gi = 0; gi < cs.g; ++gi)
      DS_TRY(gemm(c, dcur + gi * cog, cs.Cout, w.wpT[l] + 1ull * gi * Kg * cog, cog, w.col + gi * Kg, ldc,
                  static_cast<uint32_t>(Mx), Kg, cog, 1.f, nullptr, false));
    if (l >= 2) {  // input of conv4/conv5 is relu(conv3/conv4): mask, stay in NHWC
      col2im_nhwc_kernel<<<nblk(Mx * cs.Cin), 256, 0, s>>>(w.col, R, cs.H, cs.Cin, cs.K, cs.pad, cs.g, fwd_out[l - 1],
                                                           dnext, gate); ++t_launches;
      std::swap(dcur, dnext);
    } else if (l == 1) {  // input of conv3 is pool2(LRN2(relu(conv2)))
      col2im_nhwc_kernel<<<nblk(Mx * cs.Cin), 256, 0, s>>>(w.col, R, cs.H, cs.Cin, cs.K, cs.pad, cs.g, nullptr, dnext,
                                                           gate); ++t_launches;
      maxpool_bwd_kernel<<<nblk(M2 * 256), 256, 0, s>>>(dnext, w.arg2, R, sh.P1, 256, sh.P2, 0, nullptr, dcur, gate); ++t_launches;
      lrn_bwd_relu_kernel<<<nblk(M2 * 256), 256, 0, s>>>(w.a2, dcur, M2, 256, dnext, gate); ++t_launches;
      std::swap(dcur, dnext);
    } else {  // input of conv2 is pool1(LRN1(relu(conv1)))
      col2im_nhwc_kernel<<<nblk(Mx * cs.Cin), 256, 0, s>>>(w.col, R, cs.H, cs.Cin, cs.K, cs.pad, cs.g, nullptr, dnext,
                                                           gate); ++t_launches;
      maxpool_bwd_kernel<<<nblk(M1 * 96), 256, 0, s>>>(dnext, w.arg1, R, sh.H1, 96, sh.P1, 0, nullptr, dcur, gate); ++t_launches;
      lrn_bwd_relu_kernel<<<nblk(M1 * 96), 256, 0, s>>>(w.a1, dcur, M1, 96, dnext, gate); ++t_launches;
      std::swap(dcur, dnext);
    }
  }
  // conv1: bias and weight gradients (no data gradient)
  DS_TRY(colsum(c, dcur, M1, 96, 96, inv_b, grad + L[0].b_off, w.bpart));
  const uint32_t M1p = up4(static_cast<uint32_t>(M1));
  DS_TRY(transpose(c, dcur, M1, 96, 96, w.tr, M1p));
  im2colT_conv1_kernel<<<nblk(363 * M1), 256, 0, s>>>(X, idx, F, sh.S, sh.H1, M1, M1p, w.col, gate); ++t_launches;
  DS_TRY(gemm(c, w.tr, M1p, w.col, M1p, grad + L[0].w_off, 363, 96, 363, static_cast<uint32_t>(M1), inv_b, nullptr,
              false));
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

}  // namespace dsb
