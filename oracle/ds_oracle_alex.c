/* ds_oracle_alex.c — TEST INFRASTRUCTURE ONLY: f64 restatement of the AlexNet-shaped
 * convnet (model kind 3). See ds_oracle_alex.h for the network and conventions. */
#include "ds_oracle_alex.h"

#include <math.h>
#include <string.h>

#define LRN_N 5
#define LRN_ALPHA 1e-4
#define LRN_BETA 0.75
#define LRN_K 1.0

static uint32_t conv_out(uint32_t H, uint32_t k, uint32_t s, uint32_t p) { return (H + 2 * p - k) / s + 1; }
static uint32_t pooled(uint32_t H) { return (uint32_t)ceil((double)(H - 3) / 2.0) + 1; }

typedef struct {
  uint32_t S, H1, P1, P2, P5, C;
} dims;

static dims shape(uint32_t side, uint32_t C) {
  dims d;
  d.S = side;
  d.H1 = conv_out(side, 11, 4, 0);
  d.P1 = pooled(d.H1);
  d.P2 = pooled(d.P1);
  d.P5 = pooled(d.P2);
  d.C = C;
  return d;
}

uint32_t dso_alex_side(uint32_t n_features) {
  if (n_features % 3) return 0;
  const uint32_t s = (uint32_t)llround(sqrt((double)(n_features / 3)));
  if (3ull * s * s != n_features || s < 55) return 0;
  return s;
}

void dso_alex_layers(uint32_t side, uint32_t n_classes, dso_alex_layer out[DSO_ALEX_LAYERS]) {
  const dims d = shape(side, n_classes);
  const uint32_t in[DSO_ALEX_LAYERS] = {3 * 121, 48 * 25, 256 * 9, 192 * 9, 192 * 9, 256 * d.P5 * d.P5, 4096, 4096};
  const uint32_t o[DSO_ALEX_LAYERS] = {96, 256, 384, 384, 256, 4096, 4096, n_classes};
  uint64_t off = 0;
  for (int l = 0; l < DSO_ALEX_LAYERS; ++l) {
    out[l].w_off = off;
    off += (uint64_t)o[l] * in[l];
    out[l].b_off = off;
    off += o[l];
    out[l].in_dim = in[l];
    out[l].out_dim = o[l];
  }
}

uint64_t dso_alex_ws_doubles(uint32_t side, uint32_t n_classes) {
  const dims d = shape(side, n_classes);
  const uint64_t a1 = 96ull * d.H1 * d.H1, q1 = 96ull * d.P1 * d.P1, a2 = 256ull * d.P1 * d.P1,
                 q2 = 256ull * d.P2 * d.P2, a3 = 384ull * d.P2 * d.P2, q5 = 256ull * d.P5 * d.P5;
  const uint64_t fwd = 3ull * d.S * d.S + 3 * a1 + 2 * q1 + 3 * a2 + 2 * q2 + 2 * a3 + q2 + 2 * q5 + 8192 + n_classes;
  return 2 * fwd + 64;
}

/* out[co][y][x] = b[co] + sum over the group's ci, kh, kw of W[co][ci'][kh][kw] in[ci][y*s+kh-p][x*s+kw-p] */
static void conv_fwd(const double* in, uint32_t Cin, uint32_t H, uint32_t K, uint32_t s, uint32_t p, uint32_t g,
                     const float* W, const float* b, uint32_t Cout, double* out, uint32_t Ho) {
  const uint32_t cig = Cin / g, cog = Cout / g;
  for (uint32_t co = 0; co < Cout; ++co) {
    const uint32_t c0 = (co / cog) * cig;
    for (uint32_t oy = 0; oy < Ho; ++oy)
      for (uint32_t ox = 0; ox < Ho; ++ox) {
        double z = (double)b[co];
        for (uint32_t ci = 0; ci < cig; ++ci)
          for (uint32_t kh = 0; kh < K; ++kh) {
            const int y = (int)(oy * s + kh) - (int)p;
            if (y < 0 || y >= (int)H) continue;
            for (uint32_t kw = 0; kw < K; ++kw) {
              const int x = (int)(ox * s + kw) - (int)p;
              if (x < 0 || x >= (int)H) continue;
              z += (double)W[(((uint64_t)co * cig + ci) * K + kh) * K + kw] * in[((uint64_t)(c0 + ci) * H + y) * H + x];
            }
          }
        out[((uint64_t)co * Ho + oy) * Ho + ox] = z;
      }
  }
}

static void conv_bwd(const double* in, uint32_t Cin, uint32_t H, uint32_t K, uint32_t s, uint32_t p, uint32_t g,
                     const float* W, uint32_t Cout, uint32_t Ho, const double* dout, double* gW, double* gb,
                     double* din) {
  const uint32_t cig = Cin / g, cog = Cout / g;
  if (din) memset(din, 0, sizeof(double) * Cin * H * H);
  for (uint32_t co = 0; co < Cout; ++co) {
    const uint32_t c0 = (co / cog) * cig;
    for (uint32_t oy = 0; oy < Ho; ++oy)
      for (uint32_t ox = 0; ox < Ho; ++ox) {
        const double d = dout[((uint64_t)co * Ho + oy) * Ho + ox];
        if (d == 0.0) continue;
        gb[co] += d;
        for (uint32_t ci = 0; ci < cig; ++ci)
          for (uint32_t kh = 0; kh < K; ++kh) {
            const int y = (int)(oy * s + kh) - (int)p;
            if (y < 0 || y >= (int)H) continue;
            for (uint32_t kw = 0; kw < K; ++kw) {
              const int x = (int)(ox * s + kw) - (int)p;
              if (x < 0 || x >= (int)H) continue;
              const uint64_t wi = (((uint64_t)co * cig + ci) * K + kh) * K + kw;
              const uint64_t ii = ((uint64_t)(c0 + ci) * H + y) * H + x;
              gW[wi] += d * in[ii];
              if (din) din[ii] += d * (double)W[wi];
            }
          }
      }
  }
}

static void relu(double* v, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i) v[i] = v[i] > 0.0 ? v[i] : 0.0;
}
static void relu_bwd(const double* post, double* d, uint64_t n) {
  for (uint64_t i = 0; i < n; ++i)
    if (!(post[i] > 0.0)) d[i] = 0.0;
}

static void lrn_fwd(const double* in, uint32_t C, uint64_t HW, double* out, double* scale) {
  for (uint32_t c = 0; c < C; ++c) {
    const int lo = (int)c - LRN_N / 2 < 0 ? 0 : (int)c - LRN_N / 2;
    const int hi = (int)c + LRN_N / 2 >= (int)C ? (int)C - 1 : (int)c + LRN_N / 2;
    for (uint64_t i = 0; i < HW; ++i) {
      double ss = 0.0;
      for (int j = lo; j <= hi; ++j) ss += in[(uint64_t)j * HW + i] * in[(uint64_t)j * HW + i];
      const double sc = LRN_K + LRN_ALPHA / LRN_N * ss;
      scale[(uint64_t)c * HW + i] = sc;
      out[(uint64_t)c * HW + i] = in[(uint64_t)c * HW + i] * pow(sc, -LRN_BETA);
    }
  }
}

/* dx_c = dy_c scale_c^-b - (2 a b / n) x_c sum_{|c'-c|<=2} dy_c' y_c' / scale_c' */
static void lrn_bwd(const double* in, const double* out, const double* scale, const double* dout, uint32_t C,
                    uint64_t HW, double* din) {
  for (uint32_t c = 0; c < C; ++c) {
    const int lo = (int)c - LRN_N / 2 < 0 ? 0 : (int)c - LRN_N / 2;
    const int hi = (int)c + LRN_N / 2 >= (int)C ? (int)C - 1 : (int)c + LRN_N / 2;
    for (uint64_t i = 0; i < HW; ++i) {
      double acc = 0.0;
      for (int j = lo; j <= hi; ++j) {
        const uint64_t k = (uint64_t)j * HW + i;
        acc += dout[k] * out[k] / scale[k];
      }
      const uint64_t k = (uint64_t)c * HW + i;
      din[k] = dout[k] * pow(scale[k], -LRN_BETA) - 2.0 * LRN_ALPHA * LRN_BETA / LRN_N * in[k] * acc;
    }
  }
}

static void maxpool_fwd(const double* in, uint32_t C, uint32_t H, double* out, double* arg) {
  const uint32_t Ho = pooled(H);
  for (uint32_t c = 0; c < C; ++c)
    for (uint32_t ph = 0; ph < Ho; ++ph)
      for (uint32_t pw = 0; pw < Ho; ++pw) {
        const uint32_t hs = ph * 2, ws = pw * 2, he = hs + 3 < H ? hs + 3 : H, we = ws + 3 < H ? ws + 3 : H;
        double best = -INFINITY;
        uint64_t bi = 0;
        for (uint32_t h = hs; h < he; ++h)
          for (uint32_t w = ws; w < we; ++w) {
            const uint64_t i = ((uint64_t)c * H + h) * H + w;
            if (in[i] > best) best = in[i], bi = i;
          }
        out[((uint64_t)c * Ho + ph) * Ho + pw] = best;
        arg[((uint64_t)c * Ho + ph) * Ho + pw] = (double)bi;
      }
}

static void maxpool_bwd(const double* dout, const double* arg, uint64_t n_out, double* din, uint64_t n_in) {
  memset(din, 0, sizeof(double) * n_in);
  for (uint64_t i = 0; i < n_out; ++i) din[(uint64_t)arg[i]] += dout[i];
}

static void fc_fwd(const double* in, uint32_t I, const float* W, const float* b, uint32_t O, double* out) {
  for (uint32_t o = 0; o < O; ++o) {
    double s = (double)b[o];
    for (uint32_t i = 0; i < I; ++i) s += (double)W[(uint64_t)o * I + i] * in[i];
    out[o] = s;
  }
}

static void fc_bwd(const double* in, uint32_t I, const float* W, uint32_t O, const double* dout, double* gW,
                   double* gb, double* din) {
  if (din) memset(din, 0, sizeof(double) * I);
  for (uint32_t o = 0; o < O; ++o) {
    const double d = dout[o];
    gb[o] += d;
    if (d == 0.0) continue;
    for (uint32_t i = 0; i < I; ++i) {
      gW[(uint64_t)o * I + i] += d * in[i];
      if (din) din[i] += d * (double)W[(uint64_t)o * I + i];
    }
  }
}

double dso_alex_sample(const float* P, uint32_t side, uint32_t C, const float* xin, uint32_t label, double* g,
                       double* ws, uint32_t* pred) {
  const dims d = shape(side, C);
  dso_alex_layer L[DSO_ALEX_LAYERS];
  dso_alex_layers(side, C, L);
  const uint64_t nx = 3ull * d.S * d.S, a1 = 96ull * d.H1 * d.H1, q1 = 96ull * d.P1 * d.P1,
                 a2 = 256ull * d.P1 * d.P1, q2 = 256ull * d.P2 * d.P2, a3 = 384ull * d.P2 * d.P2,
                 q5 = 256ull * d.P5 * d.P5;
  double* x0 = ws;
  double* c1 = x0 + nx;    /* conv1 + relu */
  double* n1 = c1 + a1;    /* LRN out */
  double* s1 = n1 + a1;    /* LRN scale */
  double* p1 = s1 + a1;    /* pool1 */
  double* m1 = p1 + q1;    /* pool1 argmax */
  double* c2 = m1 + q1;
  double* n2 = c2 + a2;
  double* s2 = n2 + a2;
  double* p2 = s2 + a2;
  double* m2 = p2 + q2;
  double* c3 = m2 + q2;
  double* c4 = c3 + a3;
  double* c5 = c4 + a3;
  double* p5 = c5 + q2;
  double* m5 = p5 + q5;
  double* h6 = m5 + q5;
  double* h7 = h6 + 4096;
  double* z = h7 + 4096;
  for (uint64_t i = 0; i < nx; ++i) x0[i] = (double)xin[i];
  conv_fwd(x0, 3, d.S, 11, 4, 0, 1, P + L[0].w_off, P + L[0].b_off, 96, c1, d.H1);
  relu(c1, a1);
  lrn_fwd(c1, 96, (uint64_t)d.H1 * d.H1, n1, s1);
  maxpool_fwd(n1, 96, d.H1, p1, m1);
  conv_fwd(p1, 96, d.P1, 5, 1, 2, 2, P + L[1].w_off, P + L[1].b_off, 256, c2, d.P1);
  relu(c2, a2);
  lrn_fwd(c2, 256, (uint64_t)d.P1 * d.P1, n2, s2);
  maxpool_fwd(n2, 256, d.P1, p2, m2);
  conv_fwd(p2, 256, d.P2, 3, 1, 1, 1, P + L[2].w_off, P + L[2].b_off, 384, c3, d.P2);
  relu(c3, a3);
  conv_fwd(c3, 384, d.P2, 3, 1, 1, 2, P + L[3].w_off, P + L[3].b_off, 384, c4, d.P2);
  relu(c4, a3);
  conv_fwd(c4, 384, d.P2, 3, 1, 1, 2, P + L[4].w_off, P + L[4].b_off, 256, c5, d.P2);
  relu(c5, q2);
  maxpool_fwd(c5, 256, d.P2, p5, m5);
  fc_fwd(p5, (uint32_t)q5, P + L[5].w_off, P + L[5].b_off, 4096, h6);
  relu(h6, 4096);
  fc_fwd(h6, 4096, P + L[6].w_off, P + L[6].b_off, 4096, h7);
  relu(h7, 4096);
  fc_fwd(h7, 4096, P + L[7].w_off, P + L[7].b_off, C, z);
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
  double* dh7 = dz + C;
  double* dh6 = dh7 + 4096;
  double* dp5 = dh6 + 4096;
  double* dc5 = dp5 + q5;
  double* dc4 = dc5 + q2;
  double* dc3 = dc4 + a3;
  double* dp2 = dc3 + a3;
  double* dn2 = dp2 + q2;
  double* dc2 = dn2 + a2;
  double* dp1 = dc2 + a2;
  double* dn1 = dp1 + q1;
  double* dc1 = dn1 + a1;
  for (uint32_t c = 0; c < C; ++c) dz[c] = exp(z[c] - lse) - (c == label ? 1.0 : 0.0);
  fc_bwd(h7, 4096, P + L[7].w_off, C, dz, g + L[7].w_off, g + L[7].b_off, dh7);
  relu_bwd(h7, dh7, 4096);
  fc_bwd(h6, 4096, P + L[6].w_off, 4096, dh7, g + L[6].w_off, g + L[6].b_off, dh6);
  relu_bwd(h6, dh6, 4096);
  fc_bwd(p5, (uint32_t)q5, P + L[5].w_off, 4096, dh6, g + L[5].w_off, g + L[5].b_off, dp5);
  maxpool_bwd(dp5, m5, q5, dc5, q2);
  relu_bwd(c5, dc5, q2);
  conv_bwd(c4, 384, d.P2, 3, 1, 1, 2, P + L[4].w_off, 256, d.P2, dc5, g + L[4].w_off, g + L[4].b_off, dc4);
  relu_bwd(c4, dc4, a3);
  conv_bwd(c3, 384, d.P2, 3, 1, 1, 2, P + L[3].w_off, 384, d.P2, dc4, g + L[3].w_off, g + L[3].b_off, dc3);
  relu_bwd(c3, dc3, a3);
  conv_bwd(p2, 256, d.P2, 3, 1, 1, 1, P + L[2].w_off, 384, d.P2, dc3, g + L[2].w_off, g + L[2].b_off, dp2);
  maxpool_bwd(dp2, m2, q2, dn2, a2);
  lrn_bwd(c2, n2, s2, dn2, 256, (uint64_t)d.P1 * d.P1, dc2);
  relu_bwd(c2, dc2, a2);
  conv_bwd(p1, 96, d.P1, 5, 1, 2, 2, P + L[1].w_off, 256, d.P1, dc2, g + L[1].w_off, g + L[1].b_off, dp1);
  maxpool_bwd(dp1, m1, q1, dn1, a1);
  lrn_bwd(c1, n1, s1, dn1, 96, (uint64_t)d.H1 * d.H1, dc1);
  relu_bwd(c1, dc1, a1);
  conv_bwd(x0, 3, d.S, 11, 4, 0, 1, P + L[0].w_off, 96, d.H1, dc1, g + L[0].w_off, g + L[0].b_off, NULL);
  return loss;
}
