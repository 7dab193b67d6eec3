/* ds_oracle_cnn.c — TEST INFRASTRUCTURE ONLY: f64 restatement of cifar10_quick (model
 * kind 2) for the CPU oracle. See ds_oracle_cnn.h for the network and conventions. */
#include "ds_oracle_cnn.h"

#include <math.h>
#include <string.h>

void dso_cnn_layers(uint32_t n_classes, dso_cnn_layer out[5]) {
  const uint32_t in[5] = {3 * 25, 32 * 25, 32 * 25, 1024, 64};
  const uint32_t o[5] = {32, 32, 64, 64, n_classes};
  uint64_t off = 0;
  for (int l = 0; l < 5; ++l) {
    out[l].w_off = off;
    off += (uint64_t)o[l] * in[l];
    out[l].b_off = off;
    off += o[l];
    out[l].in_dim = in[l];
    out[l].out_dim = o[l];
  }
}

/* activation/gradient buffer sizes (doubles) */
enum {
  X0 = 3 * 32 * 32, C1 = 32 * 32 * 32, P1 = 32 * 16 * 16, C2 = 32 * 16 * 16, P2 = 32 * 8 * 8, C3 = 64 * 8 * 8,
  P3 = 64 * 4 * 4, H1 = 64
};

uint64_t dso_cnn_ws_doubles(uint32_t n_classes) {
  /* forward: x0 c1 p1(+arg) r1 c2 p2 c3 p3 h1 z ; backward: same shapes again */
  return 2ull * (X0 + C1 + 2 * P1 + P1 + C2 + P2 + C3 + P3 + H1 + n_classes + 64);
}

/* out[co][h][w] = b[co] + sum_ci,kh,kw W[co][ci][kh][kw] in[ci][h+kh-2][w+kw-2] */
static void conv5_fwd(const double* in, uint32_t Cin, uint32_t H, const float* W, const float* b, uint32_t Cout,
                      double* out) {
  for (uint32_t co = 0; co < Cout; ++co)
    for (uint32_t h = 0; h < H; ++h)
      for (uint32_t w = 0; w < H; ++w) {
        double z = (double)b[co];
        for (uint32_t ci = 0; ci < Cin; ++ci)
          for (int kh = 0; kh < 5; ++kh) {
            const int y = (int)h + kh - 2;
            if (y < 0 || y >= (int)H) continue;
            for (int kw = 0; kw < 5; ++kw) {
              const int x = (int)w + kw - 2;
              if (x < 0 || x >= (int)H) continue;
              z += (double)W[((co * Cin + ci) * 5 + kh) * 5 + kw] * in[(ci * H + y) * H + x];
            }
          }
        out[(co * H + h) * H + w] = z;
      }
}

/* gW/gb += dL/dW, dL/db; din (may be NULL) = dL/din */
static void conv5_bwd(const double* in, uint32_t Cin, uint32_t H, const float* W, uint32_t Cout, const double* dout,
                      double* gW, double* gb, double* din) {
  if (din) memset(din, 0, sizeof(double) * Cin * H * H);
  for (uint32_t co = 0; co < Cout; ++co)
    for (uint32_t h = 0; h < H; ++h)
      for (uint32_t w = 0; w < H; ++w) {
        const double d = dout[(co * H + h) * H + w];
        gb[co] += d;
        for (uint32_t ci = 0; ci < Cin; ++ci)
          for (int kh = 0; kh < 5; ++kh) {
            const int y = (int)h + kh - 2;
            if (y < 0 || y >= (int)H) continue;
            for (int kw = 0; kw < 5; ++kw) {
              const int x = (int)w + kw - 2;
              if (x < 0 || x >= (int)H) continue;
              const uint64_t wi = ((co * Cin + ci) * 5 + kh) * 5 + kw;
              const uint64_t ii = (ci * H + y) * H + x;
              gW[wi] += d * in[ii];
              if (din) din[ii] += d * (double)W[wi];
            }
          }
      }
}

static uint32_t pooled(uint32_t H) { return (uint32_t)ceil((double)(H - 3) / 2.0) + 1; }

/* MAX 3x3/2, ceil mode, pad 0; first maximum in scan order (Caffe strict >) */
static void maxpool_fwd(const double* in, uint32_t C, uint32_t H, double* out, double* arg) {
  const uint32_t Ho = pooled(H);
  for (uint32_t c = 0; c < C; ++c)
    for (uint32_t ph = 0; ph < Ho; ++ph)
      for (uint32_t pw = 0; pw < Ho; ++pw) {
        const uint32_t hs = ph * 2, ws = pw * 2, he = hs + 3 < H ? hs + 3 : H, we = ws + 3 < H ? ws + 3 : H;
        double best = -INFINITY;
        uint32_t bi = 0;
        for (uint32_t h = hs; h < he; ++h)
          for (uint32_t w = ws; w < we; ++w) {
            const uint32_t i = (c * H + h) * H + w;
            if (in[i] > best) best = in[i], bi = i;
          }
        out[(c * Ho + ph) * Ho + pw] = best;
        arg[(c * Ho + ph) * Ho + pw] = (double)bi;
      }
}

/* AVE 3x3/2, ceil mode, pad 0: divisor = window clipped to the image */
static void avepool_fwd(const double* in, uint32_t C, uint32_t H, double* out) {
  const uint32_t Ho = pooled(H);
  for (uint32_t c = 0; c < C; ++c)
    for (uint32_t ph = 0; ph < Ho; ++ph)
      for (uint32_t pw = 0; pw < Ho; ++pw) {
        const uint32_t hs = ph * 2, ws = pw * 2, he = hs + 3 < H ? hs + 3 : H, we = ws + 3 < H ? ws + 3 : H;
        double s = 0.0;
        for (uint32_t h = hs; h < he; ++h)
          for (uint32_t w = ws; w < we; ++w) s += in[(c * H + h) * H + w];
        out[(c * Ho + ph) * Ho + pw] = s / (double)((he - hs) * (we - ws));
      }
}

static void avepool_bwd(const double* dout, uint32_t C, uint32_t H, double* din) {
  const uint32_t Ho = pooled(H);
  memset(din, 0, sizeof(double) * C * H * H);
  for (uint32_t c = 0; c < C; ++c)
    for (uint32_t ph = 0; ph < Ho; ++ph)
      for (uint32_t pw = 0; pw < Ho; ++pw) {
        const uint32_t hs = ph * 2, ws = pw * 2, he = hs + 3 < H ? hs + 3 : H, we = ws + 3 < H ? ws + 3 : H;
        const double d = dout[(c * Ho + ph) * Ho + pw] / (double)((he - hs) * (we - ws));
        for (uint32_t h = hs; h < he; ++h)
          for (uint32_t w = ws; w < we; ++w) din[(c * H + h) * H + w] += d;
      }
}

double dso_cnn_sample(const float* P, uint32_t C, const float* xin, uint32_t label, double* g, double* ws,
                      uint32_t* pred) {
  dso_cnn_layer L[5];
  dso_cnn_layers(C, L);
  double* x0 = ws;
  double* c1 = x0 + X0;
  double* p1 = c1 + C1;
  double* a1 = p1 + P1;
  double* r1 = a1 + P1;
  double* c2 = r1 + P1;
  double* p2 = c2 + C2;
  double* c3 = p2 + P2;
  double* p3 = c3 + C3;
  double* h1 = p3 + P3;
  double* z = h1 + H1;
  for (uint32_t i = 0; i < X0; ++i) x0[i] = (double)xin[i];
  conv5_fwd(x0, 3, 32, P + L[0].w_off, P + L[0].b_off, 32, c1);
  maxpool_fwd(c1, 32, 32, p1, a1);
  for (uint32_t i = 0; i < P1; ++i) r1[i] = p1[i] > 0.0 ? p1[i] : 0.0;
  conv5_fwd(r1, 32, 16, P + L[1].w_off, P + L[1].b_off, 32, c2);
  for (uint32_t i = 0; i < C2; ++i) c2[i] = c2[i] > 0.0 ? c2[i] : 0.0;
  avepool_fwd(c2, 32, 16, p2);
  conv5_fwd(p2, 32, 8, P + L[2].w_off, P + L[2].b_off, 64, c3);
  for (uint32_t i = 0; i < C3; ++i) c3[i] = c3[i] > 0.0 ? c3[i] : 0.0;
  avepool_fwd(c3, 64, 8, p3);
  for (uint32_t o = 0; o < 64; ++o) {
    double s = (double)P[L[3].b_off + o];
    for (uint32_t i = 0; i < 1024; ++i) s += (double)P[L[3].w_off + (uint64_t)o * 1024 + i] * p3[i];
    h1[o] = s;
  }
  for (uint32_t o = 0; o < C; ++o) {
    double s = (double)P[L[4].b_off + o];
    for (uint32_t i = 0; i < 64; ++i) s += (double)P[L[4].w_off + (uint64_t)o * 64 + i] * h1[i];
    z[o] = s;
  }
  double zmax = z[0];
  uint32_t best = 0;
  for (uint32_t c = 1; c < C; ++c)
    if (z[c] > zmax) zmax = z[c], best = c;
  if (pred) *pred = best;
  double sum = 0.0;
  for (uint32_t c = 0; c < C; ++c) sum += exp(z[c] - zmax);
  const double lse = zmax + log(sum);
  const double loss = label < C ? lse - z[label] : NAN;
  if (!g) return loss;

  double* dz = z + C;
  double* dh1 = dz + C;
  double* dp3 = dh1 + H1;
  double* dc3 = dp3 + P3;
  double* dp2 = dc3 + C3;
  double* dc2 = dp2 + P2;
  double* dr1 = dc2 + C2;
  double* dc1 = dr1 + P1;
  for (uint32_t c = 0; c < C; ++c) dz[c] = exp(z[c] - lse) - (c == label ? 1.0 : 0.0);
  /* ip2 */
  for (uint32_t i = 0; i < 64; ++i) dh1[i] = 0.0;
  for (uint32_t o = 0; o < C; ++o) {
    g[L[4].b_off + o] += dz[o];
    for (uint32_t i = 0; i < 64; ++i) {
      g[L[4].w_off + (uint64_t)o * 64 + i] += dz[o] * h1[i];
      dh1[i] += dz[o] * (double)P[L[4].w_off + (uint64_t)o * 64 + i];
    }
  }
  /* ip1 */
  for (uint32_t i = 0; i < 1024; ++i) dp3[i] = 0.0;
  for (uint32_t o = 0; o < 64; ++o) {
    g[L[3].b_off + o] += dh1[o];
    for (uint32_t i = 0; i < 1024; ++i) {
      g[L[3].w_off + (uint64_t)o * 1024 + i] += dh1[o] * p3[i];
      dp3[i] += dh1[o] * (double)P[L[3].w_off + (uint64_t)o * 1024 + i];
    }
  }
  /* pool3, relu3, conv3 */
  avepool_bwd(dp3, 64, 8, dc3);
  for (uint32_t i = 0; i < C3; ++i)
    if (!(c3[i] > 0.0)) dc3[i] = 0.0;
  conv5_bwd(p2, 32, 8, P + L[2].w_off, 64, dc3, g + L[2].w_off, g + L[2].b_off, dp2);
  /* pool2, relu2, conv2 */
  avepool_bwd(dp2, 32, 16, dc2);
  for (uint32_t i = 0; i < C2; ++i)
    if (!(c2[i] > 0.0)) dc2[i] = 0.0;
  conv5_bwd(r1, 32, 16, P + L[1].w_off, 32, dc2, g + L[1].w_off, g + L[1].b_off, dr1);
  /* relu1, pool1 (max), conv1 */
  for (uint32_t i = 0; i < P1; ++i)
    if (!(p1[i] > 0.0)) dr1[i] = 0.0;
  memset(dc1, 0, sizeof(double) * C1);
  for (uint32_t i = 0; i < P1; ++i) dc1[(uint32_t)a1[i]] += dr1[i];
  conv5_bwd(x0, 3, 32, P + L[0].w_off, 32, dc1, g + L[0].w_off, g + L[0].b_off, NULL);
  return loss;
}
