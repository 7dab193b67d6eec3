// mlp_fused.cu — one persistent kernel runs many SGD iterations of a softmax
// regression or a one-hidden-layer tanh MLP, with the ExchangePolicy and the elastic
// exchange folded in (engine.cpp:72-111 + exchanger.cpp:76-92 in one launch).
//
// Work split (MLP F-H-C, batch R): CTA j owns hidden units [u0, u0+U) — the rows
// W1[u,:] (kept resident in shared memory for the whole launch) and b1[u], the columns
// W2[:,u] — and is the only writer of those parameters and of their slice of the
// center. Per iteration:
//
//   A  the batch rows of X land in shared memory by TMA bulk copies (cp.async.bulk,
//      one per row, completing on an mbarrier; the next batch is prefetched into L2
//      at the same time); forward own units a[r,u] = tanh(b1[u] + sum_i W1[u,i] x[r,i])
//      -> global act[par]
//   -- grid barrier (the only one per iteration) --
//   B  every CTA bulk-copies all a[r,:], loads W2 transposed, and computes the logits,
//      softmax-CE, per-row deltas and the batch loss redundantly (identical on every CTA,
//      so no second barrier)
//   C  own backward: delta1, gradients of own W1 rows / b1 / W2 columns (+ b2 on CTA 0),
//      f32 rounding, L2 fold, SGD -> shared W1 rows and params[cur^1] (ping-pong)
//   D  policy on every CTA (same loss -> same decision); if it fires, each CTA
//      elastic-updates its own parameter slice against the center in place, over NVLink
//      when the slice lives on a peer (LockFree: plain ld/st; Locked and deterministic:
//      per-shard tickets, exchanger order preserved)
//
// Numerics are the reference's (model.cpp:185-263): every dot product and every batch
// sum is one thread's sequential f64 chain with separate roundings, the gradient is
// rounded to f32 once, and the update rounds like param_vector.cpp:33. The chains are
// what bounds this kernel (latency, not bandwidth): 784 dependent DADDs per hidden
// unit, 256 per logit.
#include "ds_common.cuh"
#include "engine.cuh"

namespace dsb {
namespace {

constexpr int kFT = 384;  // >= R*C logit chains of the default config (32 x 10)

// ---------------------------------------------------------------------------------------
// PTX helpers: mbarrier + TMA bulk copies (sm_90+ async proxy)
// ---------------------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async;" ::: "memory"); }

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
      while (*gen == g) __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
}

__device__ __forceinline__ float ldcg(const float* p) { return __ldcg(p); }

// Optional phase timestamps (CTA 0, thread 0) for DS_FUSED_PROFILE runs.
__device__ __forceinline__ void stamp(unsigned long long* prof, uint64_t step, int slot) {
  if (prof && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    prof[step * kProfSlots + slot] = t;
  }
}

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

// Shared-memory plan (bytes), shared by host sizing and the kernel carve-up.
struct SmemPlan {
  uint32_t Fs;     // X row stride (floats): 16-byte multiple when bulk copies apply
  uint32_t Hs;     // activation row stride (doubles)
  uint32_t H2;     // W2 row stride (doubles)
  bool bulk_x;     // X rows by TMA bulk copies and 128-bit loads (F % 4 == 0)
  bool bulk_a;     // activation rows by TMA bulk copies (H % 2 == 0)
  size_t x, w, w2, as, z, e, d1, lr, rs, bars, total;
};

__host__ __device__ inline SmemPlan make_plan(uint32_t F, uint32_t H, uint32_t C, uint32_t B, uint32_t G) {
  SmemPlan p{};
  const bool hidden = H > 0;
  const uint32_t U = hidden ? (H + G - 1) / G : 0;
  p.bulk_x = (F % 4) == 0;
  p.Fs = p.bulk_x ? F + 4 : (F | 1u);
  p.bulk_a = hidden && (H % 2) == 0;
  p.Hs = hidden ? (p.bulk_a ? H + 2 : (H | 1u)) : 0;
  p.H2 = hidden ? ((H % 2) == 0 ? H + 2 : H + 1) : 0;
  auto al = [](size_t v) { return (v + 127) & ~static_cast<size_t>(127); };
  size_t off = 0;
  p.x = off;   off = al(off + static_cast<size_t>(B) * p.Fs * 4);
  p.w = off;   off = al(off + static_cast<size_t>(hidden ? U : C) * F * 4);
  p.w2 = off;  off = al(off + (hidden ? static_cast<size_t>(C) * p.H2 * 8 : 0));
  p.as = off;  off = al(off + (hidden ? static_cast<size_t>(B) * p.Hs * 8 : 0));
  p.z = off;   off = al(off + static_cast<size_t>(B) * C * 8);
  p.e = off;   off = al(off + static_cast<size_t>(B) * C * 8);
  p.d1 = off;  off = al(off + (hidden ? static_cast<size_t>(B) * U * 8 : 0));
  p.lr = off;  off = al(off + static_cast<size_t>(B) * 8);
  p.rs = off;  off = al(off + static_cast<size_t>(B) * 8 * 2 + static_cast<size_t>(B) * 4 * 2);
  p.bars = off; off = al(off + 4 * 8);
  p.total = off;
  return p;
}

// One reference-order dot product b + sum_i w[i]*x[i] over f32 operands (f64 products,
// exact), blocked by 16 so the loads and products of a block are issued ahead of its
// 16-long DADD chain (the chain is the only serial part).
//
// GPUs issue in order: a DADD that waits for the DMUL (and F2F, LDS) feeding it stalls
// everything behind it, so the products of block b+1 are formed BEFORE the DADD chain
// of block b (explicit software pipelining); the chain then runs at DADD latency.
__device__ __forceinline__ void products16(const float4* w4, const float4* x4, uint32_t blk, double (&p)[16]) {
  float4 wv[4], xv[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    wv[k] = w4[4 * blk + k];
    xv[k] = x4[4 * blk + k];
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    p[4 * k + 0] = dmul(static_cast<double>(wv[k].x), static_cast<double>(xv[k].x));
    p[4 * k + 1] = dmul(static_cast<double>(wv[k].y), static_cast<double>(xv[k].y));
    p[4 * k + 2] = dmul(static_cast<double>(wv[k].z), static_cast<double>(xv[k].z));
    p[4 * k + 3] = dmul(static_cast<double>(wv[k].w), static_cast<double>(xv[k].w));
  }
}

__device__ __forceinline__ double dot_f32_exact(double z, const float* __restrict__ w, const float* __restrict__ x,
                                                uint32_t n, bool vec) {
  uint32_t i = 0;
  if (vec && n >= 16) {
    const float4* w4 = reinterpret_cast<const float4*>(w);
    const float4* x4 = reinterpret_cast<const float4*>(x);
    const uint32_t nb = n / 16;
    double p[16], q[16];
    products16(w4, x4, 0, p);
    for (uint32_t b = 1; b < nb; ++b) {
      products16(w4, x4, b, q);  // next block's loads and products first ...
#pragma unroll
      for (int k = 0; k < 16; ++k) z = dadd(z, p[k]);  // ... then this block's chain
#pragma unroll
      for (int k = 0; k < 16; ++k) p[k] = q[k];
    }
#pragma unroll
    for (int k = 0; k < 16; ++k) z = dadd(z, p[k]);
    i = nb * 16;
  }
  for (; i < n; ++i) z = dadd(z, dmul(static_cast<double>(w[i]), static_cast<double>(x[i])));
  return z;
}

__device__ __forceinline__ void products8(const double2* w2, const double2* a2, uint32_t blk, double (&p)[8]) {
  double2 wv[4], av[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    wv[k] = w2[4 * blk + k];
    av[k] = a2[4 * blk + k];
  }
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    p[2 * k] = dmul(wv[k].x, av[k].x);
    p[2 * k + 1] = dmul(wv[k].y, av[k].y);
  }
}

// b + sum_u w[u]*a[u] over f64 operands (rounded products), pipelined blocks of 8.
__device__ __forceinline__ double dot_f64_exact(double z, const double* __restrict__ w, const double* __restrict__ a,
                                                uint32_t n, bool vec) {
  uint32_t u = 0;
  if (vec && n >= 8) {
    const double2* w2 = reinterpret_cast<const double2*>(w);
    const double2* a2 = reinterpret_cast<const double2*>(a);
    const uint32_t nb = n / 8;
    double p[8], q[8];
    products8(w2, a2, 0, p);
    for (uint32_t b = 1; b < nb; ++b) {
      products8(w2, a2, b, q);
#pragma unroll
      for (int k = 0; k < 8; ++k) z = dadd(z, p[k]);
#pragma unroll
      for (int k = 0; k < 8; ++k) p[k] = q[k];
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) z = dadd(z, p[k]);
    u = nb * 8;
  }
  for (; u < n; ++u) z = dadd(z, dmul(w[u], a[u]));
  return z;
}

template <bool kHidden>
__global__ void __launch_bounds__(kFT, 1) fused_kernel(FusedArgs A) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const unsigned int G = gridDim.x;
  const uint32_t F = A.F, H = A.H, C = A.C, B = A.B;
  const SmemPlan sp = make_plan(F, H, C, B, G);
  const uint32_t Fs = sp.Fs, Hs = sp.Hs, H2 = sp.H2;
  const uint32_t U = kHidden ? (H + G - 1) / G : 0;  // units per CTA
  const uint32_t u0 = kHidden ? blockIdx.x * U : 0;
  const uint32_t Uo = kHidden ? (u0 < H ? (u0 + U <= H ? U : H - u0) : 0) : 0;  // owned here
  const uint32_t tid = threadIdx.x;

  float* Xs = reinterpret_cast<float*>(smem_raw + sp.x);     // B x Fs batch rows
  float* Ws = reinterpret_cast<float*>(smem_raw + sp.w);     // own W1 rows (U x F) | softmax W (C x F)
  double* W2d = reinterpret_cast<double*>(smem_raw + sp.w2); // C x H2, W2 as f64 (exact)
  double* As = reinterpret_cast<double*>(smem_raw + sp.as);  // B x Hs activations
  double* Z = reinterpret_cast<double*>(smem_raw + sp.z);    // B x C logits, then deltas
  double* E = reinterpret_cast<double*>(smem_raw + sp.e);    // B x C exp(z - zmax)
  double* D1 = reinterpret_cast<double*>(smem_raw + sp.d1);  // B x U hidden deltas
  double* Lr = reinterpret_cast<double*>(smem_raw + sp.lr);  // B row losses
  double* Zmax = reinterpret_cast<double*>(smem_raw + sp.rs);
  double* Lse = Zmax + B;
  uint32_t* Lab = reinterpret_cast<uint32_t*>(Lse + B);
  uint32_t* Idx = Lab + B;
  uint64_t* bar_x = reinterpret_cast<uint64_t*>(smem_raw + sp.bars);
  uint64_t* bar_a = bar_x + 1;
  __shared__ double s_loss;
  __shared__ uint32_t s_bad, s_stop, s_flags;
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
  if (tid == 0) {
    s_pol.cum = st->cum;
    s_pol.since = st->since;
    s_pol.fire = 0;
    s_pol.period = 0;
    s_stop = st->err ? 1u : 0u;
    mbar_init(bar_x, 1);
    mbar_init(bar_a, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (s_stop) return;
  int cur = A.cur;
  uint64_t xcount = 0;
  uint32_t phase_x = 0, phase_a = 0;
  const unsigned long long it0 = st->iter;
  const bool own_any = kHidden ? (Uo > 0) : (blockIdx.x == 0);

  // W1 rows (softmax: W) are owned here: stage once, keep resident, updated in place.
  {
    const float* P0 = A.params[cur];
    const uint32_t nW = kHidden ? Uo * F : (blockIdx.x == 0 ? C * F : 0);
    const float* src = P0 + (kHidden ? w1 + static_cast<uint64_t>(u0) * F : 0);
    for (uint32_t e = tid; e < nW; e += kFT) Ws[e] = ldcg(src + e);
  }
  // L2 prefetch of the first batch's rows
  if (tid < B && A.steps > 0 && sp.bulk_x) {
    if (tid < A.plan_rows[0]) prefetch_l2(A.X + static_cast<uint64_t>(A.plan[tid]) * F, F * 4);
  }
  __syncthreads();

  for (uint64_t step = 0; step < A.steps; ++step) {
    const uint32_t R = A.plan_rows[step];
    const uint32_t* idx = A.plan + step * B;
    const float* P = A.params[cur];
    float* Pn = A.params[cur ^ 1];
    const double inv_b = 1.0 / static_cast<double>(R);
    stamp(A.prof, step, 0);
    if (tid == 0) s_bad = 0;
    if (tid < R) {
      const uint32_t row = idx[tid];
      Idx[tid] = row;
      Lab[tid] = A.y[row];
    }

    // ---- A: batch rows -> shared (TMA), next batch -> L2; forward own units ----------
    if (own_any) {
      if (sp.bulk_x) {
        if (tid == 0) {
          fence_proxy_async();  // last iteration's generic reads of Xs before the async writes
          mbar_arrive_expect_tx(bar_x, R * F * 4);
          for (uint32_t r = 0; r < R; ++r)
            bulk_g2s(Xs + static_cast<size_t>(r) * Fs, A.X + static_cast<uint64_t>(idx[r]) * F, F * 4, bar_x);
        }
        if (step + 1 < A.steps && tid >= 32 && tid < 32 + B) {
          const uint32_t r = tid - 32;
          if (r < A.plan_rows[step + 1])
            prefetch_l2(A.X + static_cast<uint64_t>(A.plan[(step + 1) * B + r]) * F, F * 4);
        }
        mbar_wait(bar_x, phase_x);
        phase_x ^= 1;
        stamp(A.prof, step, 1);
      } else {
        __syncthreads();
        for (uint32_t e = tid; e < R * F; e += kFT) {
          const uint32_t r = e / F, i = e - r * F;
          Xs[r * Fs + i] = __ldg(A.X + static_cast<uint64_t>(Idx[r]) * F + i);
        }
        __syncthreads();
      }
    }

    if constexpr (kHidden) {
      double* act = A.act + static_cast<size_t>(step & 1) * B * H;
      for (uint32_t t = tid; t < R * Uo; t += kFT) {
        const uint32_t r = t / Uo, uu = t - r * Uo, u = u0 + uu;
        const double z = dot_f32_exact(static_cast<double>(ldcg(P + b1 + u)), Ws + uu * F, Xs + r * Fs, F, sp.bulk_x);
        act[static_cast<size_t>(r) * H + u] = tanh(z);
      }
      stamp(A.prof, step, 2);
      // grid barrier; thread 0 also samples the failure flags of the previous iteration
      __syncthreads();
      if (tid == 0) {
        volatile unsigned int* gen = A.bar + 1;
        const unsigned int g = *gen;
        __threadfence();
        if (atomicAdd(A.bar, 1u) == G - 1) {
          A.bar[0] = 0;
          __threadfence();
          atomicExch(A.bar + 1, g + 1);
        } else {
          while (*gen == g) __nanosleep(20);
        }
        __threadfence();
        s_flags = *reinterpret_cast<volatile uint32_t*>(&st->flags);
        fence_proxy_async();  // other CTAs' generic writes (act, W2) before our async reads
        if (sp.bulk_a && !s_flags) {
          mbar_arrive_expect_tx(bar_a, R * H * 8);
          for (uint32_t r = 0; r < R; ++r)
            bulk_g2s(As + static_cast<size_t>(r) * Hs, act + static_cast<size_t>(r) * H, H * 8, bar_a);
        }
      }
      __syncthreads();
      stamp(A.prof, step, 3);
      if (s_flags) {  // some CTA failed in the previous iteration: every CTA stops here
        if (blockIdx.x == 0 && tid == 0) {
          st->err = s_flags;
          st->bad_iter = it0 + step;  // 1-based number of the failing iteration (step-1)
        }
        return;
      }
      // ---- B: activations (TMA), W2 as f64, logits, softmax-CE ---------------------------
      if (!sp.bulk_a) {
        for (uint32_t e = tid; e < R * H; e += kFT) {
          const uint32_t r = e / H, u = e - r * H;
          As[static_cast<size_t>(r) * Hs + u] = __ldcg(act + e);
        }
      }
      for (uint32_t e0 = tid; e0 < C * H; e0 += 4 * kFT) {
        float v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) v[k] = (e0 + k * kFT < C * H) ? ldcg(P + w2 + e0 + k * kFT) : 0.0f;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t e = e0 + k * kFT;
          if (e < C * H) {
            const uint32_t c = e / H, u = e - c * H;
            W2d[static_cast<size_t>(c) * H2 + u] = static_cast<double>(v[k]);
          }
        }
      }
      if (sp.bulk_a) {
        mbar_wait(bar_a, phase_a);
        phase_a ^= 1;
      }
      __syncthreads();
      stamp(A.prof, step, 4);
      const bool v2 = (H % 2) == 0;
      for (uint32_t t = tid; t < R * C; t += kFT) {
        const uint32_t r = t / C, c = t - r * C;
        Z[t] = dot_f64_exact(static_cast<double>(ldcg(P + b2 + c)), W2d + static_cast<size_t>(c) * H2,
                             As + static_cast<size_t>(r) * Hs, H, v2);
      }
    } else {
      if (blockIdx.x == 0) {
        for (uint32_t t = tid; t < R * C; t += kFT) {
          const uint32_t r = t / C, c = t - r * C;
          Z[t] = dot_f32_exact(static_cast<double>(ldcg(P + b1 + c)), Ws + static_cast<size_t>(c) * F, Xs + r * Fs,
                               F, sp.bulk_x);
        }
      }
    }
    __syncthreads();
    stamp(A.prof, step, 5);
    // softmax-CE (model.cpp:202-214): row max, exps in parallel, per-row sums in class
    // order, then delta = exp(z - lse) - onehot in parallel; the batch loss sum runs in
    // row order on the last thread while the deltas are formed.
    for (uint32_t r = tid; r < R; r += kFT) {
      const double* z = Z + static_cast<size_t>(r) * C;
      double zmax = z[0];
      for (uint32_t c = 1; c < C; ++c) zmax = z[c] > zmax ? z[c] : zmax;
      Zmax[r] = zmax;
    }
    __syncthreads();
    for (uint32_t t = tid; t < R * C; t += kFT) E[t] = exp(dsub(Z[t], Zmax[t / C]));
    __syncthreads();
    for (uint32_t r = tid; r < R; r += kFT) {
      const double* e = E + static_cast<size_t>(r) * C;
      double sum = 0.0;
      for (uint32_t c = 0; c < C; ++c) sum = dadd(sum, e[c]);
      const double lse = dadd(Zmax[r], log(sum));
      Lse[r] = lse;
      const uint32_t label = Lab[r];
      if (label >= C) {
        atomicOr(&s_bad, DS_FLAG_LABEL_RANGE);
        Lr[r] = 0.0;
      } else {
        Lr[r] = dsub(lse, Z[static_cast<size_t>(r) * C + label]);
      }
    }
    __syncthreads();
    if (tid == kFT - 1) {
      double s = 0.0;
      for (uint32_t r = 0; r < R; ++r) s = dadd(s, Lr[r]);
      s_loss = dmul(s, inv_b);
      if (!isfinite(s_loss)) atomicOr(&s_bad, DS_FLAG_LOSS_NONFINITE);
    }
    for (uint32_t t = tid; t < R * C; t += kFT) {
      const uint32_t r = t / C, c = t - r * C;
      Z[t] = dsub(exp(dsub(Z[t], Lse[r])), c == Lab[r] ? 1.0 : 0.0);
    }
    __syncthreads();
    // ---- C: own backward + update ------------------------------------------------------
    stamp(A.prof, step, 6);
    uint32_t bad = 0;
    if constexpr (kHidden) {
      for (uint32_t t = tid; t < R * Uo; t += kFT) {  // delta1 (model.cpp:225-233)
        const uint32_t r = t / Uo, uu = t - r * Uo, u = u0 + uu;
        const double* d = Z + static_cast<size_t>(r) * C;
        double p = 0.0;
        for (uint32_t c = 0; c < C; ++c) p = dadd(p, dmul(d[c], W2d[static_cast<size_t>(c) * H2 + u]));
        const double a = As[static_cast<size_t>(r) * Hs + u];
        D1[r * U + uu] = dmul(p, dsub(1.0, dmul(a, a)));
      }
      __syncthreads();
      // own W1 rows and b1 (the bias is the column x == 1: dmul(d, 1.0) == d exactly),
      // four independent batch chains per thread for ILP
      const uint32_t nOut = Uo * (F + 1);
      for (uint32_t e0 = tid; e0 < nOut; e0 += 4 * kFT) {
        uint32_t uu[4], ii[4];
        bool ok[4];
        double acc[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t e = e0 + k * kFT;
          ok[k] = e < nOut;
          uu[k] = ok[k] ? e / (F + 1) : 0;
          ii[k] = ok[k] ? e - uu[k] * (F + 1) : 0;
          acc[k] = 0.0;
        }
        // pipelined: the products of row r+1 are formed before row r's adds
        double pc[4], pn[4];
#pragma unroll
        for (int k = 0; k < 4; ++k)
          pc[k] = dmul(D1[uu[k]], ii[k] == F ? 1.0 : static_cast<double>(Xs[ii[k]]));
        for (uint32_t r = 1; r < R; ++r) {
#pragma unroll
          for (int k = 0; k < 4; ++k)
            pn[k] = dmul(D1[r * U + uu[k]], ii[k] == F ? 1.0 : static_cast<double>(Xs[r * Fs + ii[k]]));
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            acc[k] = dadd(acc[k], pc[k]);
            pc[k] = pn[k];
          }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) acc[k] = dadd(acc[k], pc[k]);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (!ok[k]) continue;
          const uint32_t u = u0 + uu[k];
          if (ii[k] == F) {
            const uint64_t g = b1 + u;
            Pn[g] = sgd_apply(acc[k], inv_b, ldcg(P + g), A.eta, A.wd, bad);
          } else {
            const float o = sgd_apply(acc[k], inv_b, Ws[uu[k] * F + ii[k]], A.eta, A.wd, bad);
            Ws[uu[k] * F + ii[k]] = o;
            Pn[w1 + static_cast<uint64_t>(u) * F + ii[k]] = o;
          }
        }
      }
      // own W2 columns
      for (uint32_t e = tid; e < C * Uo; e += kFT) {
        const uint32_t c = e / Uo, uu = e - c * Uo, u = u0 + uu;
        double acc = 0.0;
        for (uint32_t r = 0; r < R; ++r)
          acc = dadd(acc, dmul(Z[static_cast<size_t>(r) * C + c], As[static_cast<size_t>(r) * Hs + u]));
        const uint64_t g = w2 + static_cast<uint64_t>(c) * H + u;
        Pn[g] = sgd_apply(acc, inv_b, static_cast<float>(W2d[static_cast<size_t>(c) * H2 + u]), A.eta, A.wd, bad);
      }
      if (blockIdx.x == 0) {
        for (uint32_t c = tid; c < C; c += kFT) {
          double acc = 0.0;
          for (uint32_t r = 0; r < R; ++r) acc = dadd(acc, Z[static_cast<size_t>(r) * C + c]);
          const uint64_t g = b2 + c;
          Pn[g] = sgd_apply(acc, inv_b, ldcg(P + g), A.eta, A.wd, bad);
        }
      }
    } else if (blockIdx.x == 0) {
      const uint32_t nOut = C * (F + 1);
      for (uint32_t e0 = tid; e0 < nOut; e0 += 4 * kFT) {
        uint32_t cc[4], ii[4];
        bool ok[4];
        double acc[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t e = e0 + k * kFT;
          ok[k] = e < nOut;
          cc[k] = ok[k] ? e / (F + 1) : 0;
          ii[k] = ok[k] ? e - cc[k] * (F + 1) : 0;
          acc[k] = 0.0;
        }
        for (uint32_t r = 0; r < R; ++r) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const double x = ii[k] == F ? 1.0 : static_cast<double>(Xs[r * Fs + ii[k]]);
            acc[k] = dadd(acc[k], dmul(Z[static_cast<size_t>(r) * C + cc[k]], x));
          }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if (!ok[k]) continue;
          if (ii[k] == F) {
            const uint64_t g = b1 + cc[k];
            Pn[g] = sgd_apply(acc[k], inv_b, ldcg(P + g), A.eta, A.wd, bad);
          } else {
            const float o = sgd_apply(acc[k], inv_b, Ws[static_cast<size_t>(cc[k]) * F + ii[k]], A.eta, A.wd, bad);
            Ws[static_cast<size_t>(cc[k]) * F + ii[k]] = o;
            Pn[static_cast<uint64_t>(cc[k]) * F + ii[k]] = o;
          }
        }
      }
    }
    bad = __reduce_or_sync(0xffffffffu, bad);
    if (bad && (tid & 31) == 0) atomicOr(&s_bad, bad);
    __syncthreads();
    // ---- D: policy + exchange ------------------------------------------------------------
    stamp(A.prof, step, 7);
    if (s_bad) {
      // Publish; with a hidden layer every CTA (this one included) stops after the next
      // barrier, so no CTA ever skips a barrier another CTA waits on.
      if (tid == 0) atomicOr(&st->flags, s_bad);
      if (!kHidden) {
        if (tid == 0) {
          st->err = s_bad;
          st->bad_iter = it0 + step + 1;
        }
        return;
      }
    }
    if (tid == 0) {
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
        if (blockIdx.x == 0 && tid == 0) *slot = atomicAdd_system(A.ticket_src, 1ull);
        if (kHidden) grid_barrier(A.bar, G);
        else __syncthreads();
        if (tid == 0) s_ticket = __ldcg(slot);
        __syncthreads();
        tk = s_ticket;
      }
      do_exchange(A, Pn, sl, tk, kHidden ? G : 1u);
      // the exchange moved the resident rows too: refresh them from params[cur^1]
      const uint32_t nW = kHidden ? Uo * F : C * F;
      const float* src = Pn + (kHidden ? w1 + static_cast<uint64_t>(u0) * F : 0);
      for (uint32_t e = tid; e < nW; e += kFT) Ws[e] = src[e];
      ++xcount;
    }
    cur ^= 1;
    __syncthreads();
    stamp(A.prof, step, 8);
  }
  if constexpr (kHidden) {
    grid_barrier(A.bar, G);  // failures of the last iteration become visible here
    const uint32_t fl = *reinterpret_cast<volatile uint32_t*>(&st->flags);
    if (fl) {
      if (blockIdx.x == 0 && tid == 0) {
        st->err = fl;
        st->bad_iter = it0 + A.steps;
      }
      return;
    }
  }
  if (blockIdx.x == 0 && tid == 0) {
    st->cum = s_pol.cum;
    st->since = s_pol.since;
    st->fire = s_pol.fire;
    st->period = s_pol.period;
    st->loss = s_loss;
    st->iter = it0 + A.steps;
    st->exchanges += xcount;
  }
}

int grid_for(const ModelInfo& m, int device) {
  if (m.hidden.empty()) return 1;
  const uint32_t H = m.hidden[0];
  const uint32_t sms = static_cast<uint32_t>(sm_count(device));
  const uint32_t cap = H < sms ? H : sms;
  const uint32_t U = (H + cap - 1) / cap;
  return static_cast<int>((H + U - 1) / U);
}

size_t smem_for(uint32_t F, uint32_t H, uint32_t C, uint32_t B, uint32_t G) {
  return make_plan(F, H, C, B, G).total;
}

}  // namespace

int fused_grid(const ModelInfo& m, int device) { return grid_for(m, device); }

size_t fused_smem_bytes(const ModelInfo& m, uint32_t batch) {
  const uint32_t H = m.hidden.empty() ? 0 : m.hidden[0];
  return smem_for(m.n_features, H, m.n_classes, batch, static_cast<uint32_t>(grid_for(m, 0)));
}

int fused_supported(const ModelInfo& m, uint32_t batch, int device, const char** why) {
  if (m.hidden.size() > 1) {
    if (why) *why = "more than one hidden layer";
    return DS_E_CONTRACT;
  }
  if (batch > 1024) {
    if (why) *why = "batch_size above 1024";
    return DS_E_CONTRACT;
  }
  const uint32_t H = m.hidden.empty() ? 0 : m.hidden[0];
  const size_t need = smem_for(m.n_features, H, m.n_classes, batch, static_cast<uint32_t>(grid_for(m, device)));
  int optin = 0;
  if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device) != cudaSuccess) optin = 227 * 1024;
  if (need + 8192 > static_cast<size_t>(optin)) {  // + static shared (indices, policy)
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
  const size_t smem = smem_for(a.F, a.H, a.C, a.B, static_cast<uint32_t>(grid));
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
