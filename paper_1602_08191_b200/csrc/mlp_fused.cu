// mlp_fused.cu — one persistent kernel runs many SGD iterations of a softmax
// regression or a one-hidden-layer tanh MLP, with the ExchangePolicy and the elastic
// exchange folded in (engine.cpp:72-111 + exchanger.cpp:76-92 in one launch).
//
// Work split (MLP F-H-C, batch R): CTA j owns hidden units [u0, u0+U) — the rows
// W1[u,:] and b1[u], the columns W2[:,u] — and is the only writer of those parameters
// and of their slice of the center. Per iteration:
//
//   A  stage the batch rows of X and own W1 rows into shared memory; forward own
//      units a[r,u] = tanh(b1[u] + sum_i W1[u,i] x[r,i]) -> global act[par]
//   -- grid barrier (the only one per iteration) --
//   B  every CTA loads all a[r,:] and computes the logits, softmax-CE, per-row deltas
//      and the batch loss redundantly (identical everywhere, so no second barrier)
//   C  own backward: delta1, gradients of own W1 rows / b1 / W2 columns (+ b2 on
//      CTA 0), f32 rounding, L2 fold, SGD -> params[cur^1] (ping-pong buffers)
//   D  policy on every CTA (same loss -> same decision); if it fires, each CTA
//      elastic-updates its own parameter slice against the center in place, over
//      NVLink when the slice lives on a peer (LockFree: plain ld/st; Locked and
//      deterministic: per-shard tickets, exchanger order preserved)
//
// Numerics are the reference's (model.cpp:185-263): every dot product and every
// batch sum is one thread's sequential f64 chain with separate roundings, the gradient
// is rounded to f32 once, and the update rounds like param_vector.cpp:33.
#include <cooperative_groups.h>

#include "ds_common.cuh"
#include "engine.cuh"

namespace dsb {
namespace {

constexpr int kFT = 256;

__device__ __forceinline__ void grid_barrier(unsigned int* bar, unsigned int G) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned int* gen = bar + 1;
    const unsigned int g = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == G - 1) {
      bar[0] = 0;
      __threadfence();
      atomicExch(bar + 1, g + 1);
    } else {
      while (*gen == g) __nanosleep(32);
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ float ldcg(const float* p) { return __ldcg(p); }
__device__ __forceinline__ double ldcg(const double* p) { return __ldcg(p); }

// f32 gradient -> L2 fold -> SGD, with the reference's checks (param_vector.cpp:21-39).
__device__ __forceinline__ float sgd_apply(double acc, double inv_b, float x, float eta, float wd, uint32_t& bad) {
  const double g = dmul(acc, inv_b);
  if (!isfinite(g)) bad |= DS_FLAG_GRAD_NONFINITE;
  float gf = static_cast<float>(g);
  if (!isfinite(x)) bad |= DS_FLAG_X_NONFINITE;
  if (wd > 0.0f) gf = fadd(gf, fmul(wd, x));
  if (!isfinite(gf)) bad |= DS_FLAG_G_NONFINITE;
  const float o = fsub(x, fmul(eta, gf));
  if (!isfinite(o)) bad |= DS_FLAG_OUT_NONFINITE;
  return o;
}

// The global parameter indices a CTA owns: up to 4 row-major blocks, element j of
// block k is lo + (j / cols) * row_stride + (j % cols).
struct Slice {
  uint64_t lo[4], row_stride[4];
  uint32_t rows[4], cols[4];
  int n;
};

__device__ __forceinline__ void slice_add(Slice& s, uint64_t lo, uint32_t rows, uint32_t cols, uint64_t rs) {
  if (!rows || !cols) return;
  s.lo[s.n] = lo;
  s.rows[s.n] = rows;
  s.cols[s.n] = cols;
  s.row_stride[s.n] = rs;
  ++s.n;
}

// Elastic update of element g (params[nxt][g] vs center) for the shard containing g.
// The center is read/written through L2 (.cg): it is shared with other CTAs/GPUs.
__device__ __forceinline__ void exchange_elem(float* p, const ShardTable& t, int s, uint64_t g, float a) {
  float* m = t.ptr[s] + (g - t.begin[s]);
  float wo, mo;
  elastic_elem(p[g], __ldcg(m), a, wo, mo);
  p[g] = wo;
  __stcg(m, mo);
}

// All of this CTA's elements that fall into shard s.
__device__ void exchange_shard(float* p, const ShardTable& t, int s, const Slice& sl, float a) {
  const uint64_t b0 = t.begin[s], b1 = t.begin[s + 1];
  for (int k = 0; k < sl.n; ++k) {
    const uint32_t n = sl.rows[k] * sl.cols[k];
    for (uint32_t j = threadIdx.x; j < n; j += kFT) {
      const uint32_t r = j / sl.cols[k];
      const uint64_t g = sl.lo[k] + r * sl.row_stride[k] + (j - r * sl.cols[k]);
      if (g >= b0 && g < b1) exchange_elem(p, t, s, g, a);
    }
  }
}

__device__ void do_exchange(const FusedArgs& A, float* p, const Slice& sl, uint64_t ticket, unsigned int G) {
  const ShardTable& t = A.table;
  const bool ordered = ticket != kNoTicket;
  for (int s = 0; s < t.n; ++s) {
    if (ordered) {
      if (threadIdx.x == 0)
        while (ld_acquire_sys(reinterpret_cast<const uint64_t*>(&t.flags[s]->seq)) != ticket) nanosleep_ns(64);
      __syncthreads();
    }
    exchange_shard(p, t, s, sl, A.alpha);
    __syncthreads();
    if (threadIdx.x == 0) {
      if (ordered) {
        __threadfence_system();
        const unsigned long long old = atomicAdd_system(&t.flags[s]->done, 1ull);
        if (old == G - 1) {
          t.flags[s]->done = 0;
          if (s == 0) t.flags[0]->exchanges += 1;
          __threadfence_system();
          st_release_sys(reinterpret_cast<uint64_t*>(&t.flags[s]->seq), ticket + 1);
        }
      } else if (s == 0 && blockIdx.x == 0) {
        atomicAdd_system(&t.flags[0]->exchanges, 1ull);
      }
    }
  }
}

struct PolicyLocal {
  double cum;
  uint32_t since;
  uint32_t fire, period;
};

__device__ __forceinline__ void policy_update(PolicyLocal& pl, double loss, const DevState* st) {
  pl.cum = dadd(pl.cum, loss);
  pl.since += 1;
  const bool fire = st->adaptive ? (pl.cum > st->cut) : (pl.since == st->tau);
  pl.period = fire ? pl.since : 0u;
  pl.fire = fire ? 1u : 0u;
  if (fire) {
    pl.cum = 0.0;
    pl.since = 0;
  }
}

template <bool kHidden>
__global__ void __launch_bounds__(kFT, 1) fused_kernel(FusedArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const unsigned int G = gridDim.x;
  const uint32_t F = A.F, H = A.H, C = A.C, B = A.B;
  const uint32_t Fp = F | 1u;                      // odd row stride: conflict-free column walks
  const uint32_t U = kHidden ? (H + G - 1) / G : 0;  // units per CTA
  const uint32_t u0 = kHidden ? blockIdx.x * U : 0;
  const uint32_t Uo = kHidden ? (u0 < H ? (u0 + U <= H ? U : H - u0) : 0) : 0;  // owned here
  const uint32_t Hp = H + 1;
  const uint32_t O = kHidden ? H : C;              // width feeding the logits (unused for softmax)
  (void)O;

  // shared memory carve-up
  float* Xs = reinterpret_cast<float*>(smem_raw);                 // B x Fp
  float* Ws = Xs + static_cast<size_t>(B) * Fp;                   // own W1 rows (U x F) | softmax: C x F
  float* W2s = Ws + static_cast<size_t>(kHidden ? U : C) * F;     // C x H (MLP)
  size_t off = reinterpret_cast<unsigned char*>(W2s + (kHidden ? static_cast<size_t>(C) * H : 0)) - smem_raw;
  off = (off + 15) & ~static_cast<size_t>(15);
  double* As = reinterpret_cast<double*>(smem_raw + off);         // B x Hp (MLP)
  double* Z = As + (kHidden ? static_cast<size_t>(B) * Hp : 0);   // B x C logits / deltas
  double* D1 = Z + static_cast<size_t>(B) * C;                     // B x U
  double* Lr = D1 + (kHidden ? static_cast<size_t>(B) * U : 0);   // B row losses
  __shared__ double s_loss;
  __shared__ uint32_t s_bad, s_stop;
  __shared__ PolicyLocal s_pol;
  __shared__ unsigned long long s_ticket;

  // parameter layout (Model::layers, model.cpp:103-121)
  const uint64_t w1 = 0, b1 = kHidden ? static_cast<uint64_t>(H) * F : static_cast<uint64_t>(C) * F;
  const uint64_t w2 = kHidden ? b1 + H : 0, b2 = kHidden ? w2 + static_cast<uint64_t>(C) * H : b1;

  Slice sl;
  sl.n = 0;
  if constexpr (kHidden) {
    slice_add(sl, w1 + static_cast<uint64_t>(u0) * F, 1, Uo * F, 0);  // own W1 rows
    slice_add(sl, b1 + u0, 1, Uo, 0);                                  // own b1
    slice_add(sl, w2 + u0, C, Uo, H);                                  // own W2 columns
    if (blockIdx.x == 0) slice_add(sl, b2, 1, C, 0);                   // b2
  } else if (blockIdx.x == 0) {
    slice_add(sl, 0, 1, static_cast<uint32_t>(A.P), 0);
  }

  DevState* st = A.st;
  if (threadIdx.x == 0) {
    s_pol.cum = st->cum;
    s_pol.since = st->since;
    s_pol.fire = 0;
    s_pol.period = 0;
    s_stop = st->err ? 1u : 0u;
  }
  __syncthreads();
  if (s_stop) return;
  int cur = A.cur;
  uint64_t xcount = 0;  // exchanges performed in this launch
  const unsigned long long it0 = st->iter;

  for (uint64_t step = 0; step < A.steps; ++step) {
    const uint32_t R = A.plan_rows[step];
    const uint32_t* idx = A.plan + step * B;
    const float* P = A.params[cur];
    float* Pn = A.params[cur ^ 1];
    const double inv_b = 1.0 / static_cast<double>(R);
    if (threadIdx.x == 0) s_bad = 0;

    // ---- A: stage X rows and own weights -----------------------------------------
    for (uint32_t e = threadIdx.x; e < R * F; e += kFT) {
      const uint32_t r = e / F, i = e - r * F;
      Xs[r * Fp + i] = __ldg(A.X + static_cast<uint64_t>(idx[r]) * F + i);
    }
    if constexpr (kHidden) {
      for (uint32_t e = threadIdx.x; e < Uo * F; e += kFT) Ws[e] = ldcg(P + w1 + static_cast<uint64_t>(u0) * F + e);
    } else if (blockIdx.x == 0) {
      for (uint32_t e = threadIdx.x; e < C * F; e += kFT) Ws[e] = ldcg(P + e);
    }
    __syncthreads();

    if constexpr (kHidden) {
      double* act = A.act + static_cast<size_t>(step & 1) * B * H;
      for (uint32_t t = threadIdx.x; t < R * Uo; t += kFT) {
        const uint32_t r = t / Uo, uu = t - r * Uo, u = u0 + uu;
        const float* w = Ws + uu * F;
        const float* x = Xs + r * Fp;
        double z = static_cast<double>(ldcg(P + b1 + u));
#pragma unroll 8
        for (uint32_t i = 0; i < F; ++i) z = dadd(z, dmul(static_cast<double>(w[i]), static_cast<double>(x[i])));
        act[static_cast<size_t>(r) * H + u] = tanh(z);
      }
      grid_barrier(A.bar, G);
      const uint32_t fl = *reinterpret_cast<volatile uint32_t*>(&st->flags);
      if (fl) {  // some CTA failed in the previous iteration: every CTA stops here
        if (blockIdx.x == 0 && threadIdx.x == 0) {
          st->err = fl;
          st->bad_iter = it0 + step;  // 1-based number of the failing iteration (step-1)
        }
        return;
      }
      // ---- B: all activations, logits, softmax-CE (redundant per CTA) ----------------
      for (uint32_t e = threadIdx.x; e < R * H; e += kFT) {
        const uint32_t r = e / H, u = e - r * H;
        As[r * Hp + u] = ldcg(act + e);
      }
      for (uint32_t e = threadIdx.x; e < C * H; e += kFT) W2s[e] = ldcg(P + w2 + e);
      __syncthreads();
      for (uint32_t t = threadIdx.x; t < R * C; t += kFT) {
        const uint32_t r = t / C, c = t - r * C;
        const float* w = W2s + static_cast<size_t>(c) * H;
        const double* a = As + r * Hp;
        double z = static_cast<double>(ldcg(P + b2 + c));
#pragma unroll 8
        for (uint32_t u = 0; u < H; ++u) z = dadd(z, dmul(static_cast<double>(w[u]), a[u]));
        Z[t] = z;
      }
    } else {
      if (blockIdx.x == 0) {
        for (uint32_t t = threadIdx.x; t < R * C; t += kFT) {
          const uint32_t r = t / C, c = t - r * C;
          const float* w = Ws + static_cast<size_t>(c) * F;
          const float* x = Xs + r * Fp;
          double z = static_cast<double>(ldcg(P + b1 + c));
#pragma unroll 8
          for (uint32_t i = 0; i < F; ++i) z = dadd(z, dmul(static_cast<double>(w[i]), static_cast<double>(x[i])));
          Z[t] = z;
        }
      }
    }
    __syncthreads();
    // softmax-CE per row (model.cpp:202-214), delta overwrites the logits in place
    for (uint32_t r = threadIdx.x; r < R; r += kFT) {
      const uint32_t label = A.y[idx[r]];
      double* z = Z + static_cast<size_t>(r) * C;
      if (label >= C) {
        atomicOr(&s_bad, DS_FLAG_LABEL_RANGE);
        Lr[r] = 0.0;
        continue;
      }
      double zmax = z[0];
      for (uint32_t c = 1; c < C; ++c) zmax = z[c] > zmax ? z[c] : zmax;
      double sum = 0.0;
      for (uint32_t c = 0; c < C; ++c) sum = dadd(sum, exp(dsub(z[c], zmax)));
      const double lse = dadd(zmax, log(sum));
      Lr[r] = dsub(lse, z[label]);
      for (uint32_t c = 0; c < C; ++c) z[c] = dsub(exp(dsub(z[c], lse)), c == label ? 1.0 : 0.0);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      double s = 0.0;
      for (uint32_t r = 0; r < R; ++r) s = dadd(s, Lr[r]);
      s_loss = dmul(s, inv_b);
      if (!isfinite(s_loss)) atomicOr(&s_bad, DS_FLAG_LOSS_NONFINITE);
    }
    // ---- C: own backward + update ------------------------------------------------------
    uint32_t bad = 0;
    if constexpr (kHidden) {
      for (uint32_t t = threadIdx.x; t < R * Uo; t += kFT) {  // delta1 (model.cpp:225-233)
        const uint32_t r = t / Uo, uu = t - r * Uo, u = u0 + uu;
        const double* d = Z + static_cast<size_t>(r) * C;
        double p = 0.0;
        for (uint32_t c = 0; c < C; ++c) p = dadd(p, dmul(d[c], static_cast<double>(W2s[static_cast<size_t>(c) * H + u])));
        const double a = As[r * Hp + u];
        D1[r * U + uu] = dmul(p, dsub(1.0, dmul(a, a)));
      }
      __syncthreads();
      // own W1 rows and b1
      for (uint32_t e = threadIdx.x; e < Uo * (F + 1); e += kFT) {
        const uint32_t uu = e / (F + 1), i = e - uu * (F + 1), u = u0 + uu;
        double acc = 0.0;
        if (i == F) {
          for (uint32_t r = 0; r < R; ++r) acc = dadd(acc, D1[r * U + uu]);
          const uint64_t g = b1 + u;
          Pn[g] = sgd_apply(acc, inv_b, ldcg(P + g), A.eta, A.wd, bad);
        } else {
          for (uint32_t r = 0; r < R; ++r) acc = dadd(acc, dmul(D1[r * U + uu], static_cast<double>(Xs[r * Fp + i])));
          const uint64_t g = w1 + static_cast<uint64_t>(u) * F + i;
          Pn[g] = sgd_apply(acc, inv_b, Ws[uu * F + i], A.eta, A.wd, bad);
        }
      }
      // own W2 columns
      for (uint32_t e = threadIdx.x; e < C * Uo; e += kFT) {
        const uint32_t c = e / Uo, uu = e - c * Uo, u = u0 + uu;
        double acc = 0.0;
        for (uint32_t r = 0; r < R; ++r) acc = dadd(acc, dmul(Z[static_cast<size_t>(r) * C + c], As[r * Hp + u]));
        const uint64_t g = w2 + static_cast<uint64_t>(c) * H + u;
        Pn[g] = sgd_apply(acc, inv_b, W2s[static_cast<size_t>(c) * H + u], A.eta, A.wd, bad);
      }
      if (blockIdx.x == 0) {
        for (uint32_t c = threadIdx.x; c < C; c += kFT) {
          double acc = 0.0;
          for (uint32_t r = 0; r < R; ++r) acc = dadd(acc, Z[static_cast<size_t>(r) * C + c]);
          const uint64_t g = b2 + c;
          Pn[g] = sgd_apply(acc, inv_b, ldcg(P + g), A.eta, A.wd, bad);
        }
      }
    } else if (blockIdx.x == 0) {
      for (uint32_t e = threadIdx.x; e < C * (F + 1); e += kFT) {
        const uint32_t c = e / (F + 1), i = e - c * (F + 1);
        double acc = 0.0;
        if (i == F) {
          for (uint32_t r = 0; r < R; ++r) acc = dadd(acc, Z[static_cast<size_t>(r) * C + c]);
          const uint64_t g = b1 + c;
          Pn[g] = sgd_apply(acc, inv_b, ldcg(P + g), A.eta, A.wd, bad);
        } else {
          for (uint32_t r = 0; r < R; ++r) acc = dadd(acc, dmul(Z[static_cast<size_t>(r) * C + c], static_cast<double>(Xs[r * Fp + i])));
          const uint64_t g = static_cast<uint64_t>(c) * F + i;
          Pn[g] = sgd_apply(acc, inv_b, Ws[static_cast<size_t>(c) * F + i], A.eta, A.wd, bad);
        }
      }
    }
    bad = __reduce_or_sync(0xffffffffu, bad);
    if (bad && (threadIdx.x & 31) == 0) atomicOr(&s_bad, bad);
    __syncthreads();
    // ---- D: policy + exchange ------------------------------------------------------------
    if (s_bad) {
      // Publish; with a hidden layer every CTA (this one included) stops after the next
      // barrier, so no CTA ever skips a barrier another CTA waits on.
      if (threadIdx.x == 0) atomicOr(&st->flags, s_bad);
      if (!kHidden) {
        if (threadIdx.x == 0) {
          st->err = s_bad;
          st->bad_iter = it0 + step + 1;
        }
        return;
      }
    }
    if (threadIdx.x == 0) {
      policy_update(s_pol, s_loss, st);
      if (blockIdx.x == 0) {
        const unsigned long long row = it0 + step;
        if (row < A.log.cap) {
          A.log.loss[row] = s_loss;
          A.log.cum[row] = s_pol.cum;
          A.log.exchanged[row] = static_cast<uint8_t>(s_pol.fire);
          A.log.period[row] = s_pol.period;
        }
      }
    }
    __syncthreads();
    if (s_pol.fire && A.has_master && (kHidden || blockIdx.x == 0)) {
      uint64_t tk = kNoTicket;
      if (A.tickets) {
        tk = A.tickets[xcount];
      } else if (A.ticket_src) {
        // Locked: take the next global ticket once, share it through the barrier
        unsigned long long* slot = reinterpret_cast<unsigned long long*>(A.bar + 4);
        if (blockIdx.x == 0 && threadIdx.x == 0) *slot = atomicAdd_system(A.ticket_src, 1ull);
        if (kHidden) grid_barrier(A.bar, G);
        else __syncthreads();
        if (threadIdx.x == 0) s_ticket = __ldcg(slot);
        __syncthreads();
        tk = s_ticket;
      }
      do_exchange(A, Pn, sl, tk, kHidden ? G : 1u);
      ++xcount;
    }
    cur ^= 1;
    __syncthreads();
  }
  if constexpr (kHidden) {
    grid_barrier(A.bar, G);  // failures of the last iteration become visible here
    const uint32_t fl = *reinterpret_cast<volatile uint32_t*>(&st->flags);
    if (fl) {
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        st->err = fl;
        st->bad_iter = it0 + A.steps;
      }
      return;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    st->cum = s_pol.cum;
    st->since = s_pol.since;
    st->fire = s_pol.fire;
    st->period = s_pol.period;
    st->loss = s_loss;
    st->iter = it0 + A.steps;
    st->exchanges += xcount;
  }
}

size_t smem_bytes(uint32_t F, uint32_t H, uint32_t C, uint32_t B, uint32_t G) {
  const uint32_t Fp = F | 1u;
  const bool hidden = H > 0;
  const uint32_t U = hidden ? (H + G - 1) / G : 0;
  size_t f = static_cast<size_t>(B) * Fp + static_cast<size_t>(hidden ? U : C) * F + (hidden ? static_cast<size_t>(C) * H : 0);
  size_t bytes = ((f * sizeof(float)) + 15) & ~static_cast<size_t>(15);
  size_t d = (hidden ? static_cast<size_t>(B) * (H + 1) : 0) + static_cast<size_t>(B) * C + (hidden ? static_cast<size_t>(B) * U : 0) + B;
  return bytes + d * sizeof(double);
}

int grid_for(const ModelInfo& m, int device) {
  if (m.hidden.empty()) return 1;
  const uint32_t H = m.hidden[0];
  const uint32_t sms = static_cast<uint32_t>(sm_count(device));
  const uint32_t cap = H < sms ? H : sms;
  const uint32_t U = (H + cap - 1) / cap;
  return static_cast<int>((H + U - 1) / U);
}

}  // namespace

int fused_grid(const ModelInfo& m, int device) { return grid_for(m, device); }

size_t fused_smem_bytes(const ModelInfo& m, uint32_t batch) {
  const uint32_t H = m.hidden.empty() ? 0 : m.hidden[0];
  return smem_bytes(m.n_features, H, m.n_classes, batch, static_cast<uint32_t>(grid_for(m, 0)));
}

int fused_supported(const ModelInfo& m, uint32_t batch, int device, const char** why) {
  if (m.hidden.size() > 1) {
    if (why) *why = "more than one hidden layer";
    return DS_E_CONTRACT;
  }
  const uint32_t H = m.hidden.empty() ? 0 : m.hidden[0];
  const size_t need = smem_bytes(m.n_features, H, m.n_classes, batch, static_cast<uint32_t>(grid_for(m, device)));
  int optin = 0;
  if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device) != cudaSuccess) optin = 227 * 1024;
  if (need + 1024 > static_cast<size_t>(optin)) {
    if (why) *why = "batch x features does not fit in shared memory";
    return DS_E_CONTRACT;
  }
  int coop = 0;
  cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device);
  if (!coop) {
    if (why) *why = "device lacks cooperative launch";
    return DS_E_CONTRACT;
  }
  return DS_OK;
}

int launch_fused(const FusedArgs& a, int grid, cudaStream_t s) {
  const size_t smem = smem_bytes(a.F, a.H, a.C, a.B, static_cast<uint32_t>(grid));
  void* args[] = {const_cast<FusedArgs*>(&a)};
  if (a.H > 0) {
    DS_CUDA_TRY(cudaFuncSetAttribute(fused_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    DS_CUDA_TRY(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(fused_kernel<true>), dim3(grid), dim3(kFT), args, smem, s));
  } else {
    DS_CUDA_TRY(cudaFuncSetAttribute(fused_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    DS_CUDA_TRY(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(fused_kernel<false>), dim3(1), dim3(kFT), args, smem, s));
  }
  return DS_OK;
}

}  // namespace dsb
