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
#include <algorithm>
#include <cstdlib>

#include <map>
#include <mutex>
#include <tuple>

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
// 16-byte LDGSTS (no register staging) and its completion hook on an mbarrier: the
// arrive fires when every cp.async this thread issued so far has landed (.noinc: the
// barrier's expected count already includes these arrivals).
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_arrive(uint64_t* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Grid-wide barrier over a monotonic arrival counter (zeroed before each launch, see
// launch_fused): the k-th barrier of a launch completes when the counter reaches k*G.
// One release-add per CTA after the CTA barrier (cumulative over the CTA's writes) and
// acquire polling; no reset, no generation flag, no full fences. `nbar` is the calling
// kernel's __shared__ barrier count (touched by thread 0 only).
constexpr int kBarCounter = 32;  // word of A.bar holding the counter (own 128-byte line)
__device__ __forceinline__ void grid_arrive_wait(unsigned int* bar, unsigned int& nbar, unsigned int G) {
  unsigned int* ctr = bar + kBarCounter;
  const unsigned int target = (++nbar) * G;
  asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
  unsigned int v;
  do {
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
  } while (static_cast<int>(v - target) < 0);
}
__device__ __forceinline__ void grid_barrier(unsigned int* bar, unsigned int& nbar, unsigned int G) {
  __syncthreads();
  if (threadIdx.x == 0) grid_arrive_wait(bar, nbar, G);
  __syncthreads();
}

__device__ __forceinline__ float ldcg(const float* p) { return __ldcg(p); }

// Optional phase timestamps (CTA 0, thread 0) for DS_FUSED_PROFILE runs.
__device__ __forceinline__ void stamp_cta(unsigned long long* prof_cta, uint64_t step, int slot) {
  if (prof_cta && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    prof_cta[(step * gridDim.x + blockIdx.x) * 2 + slot] = t;
  }
}
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
      __shared__ int s_timeout;
      if (threadIdx.x == 0) {
        s_timeout = !wait_seq_eq(reinterpret_cast<const uint64_t*>(&t.flags[s]->seq), ticket, 64);
        if (s_timeout) {
          atomicAdd_system(&t.flags[s]->timeouts, 1ull);
          atomicOr(&A.st->flags, DS_FLAG_TICKET_TIMEOUT);
        }
      }
      __syncthreads();
      if (s_timeout) return;
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

// mlp_kernel's exchange: as do_exchange, but the CTA's own W1 rows (slice 0, contiguous,
// 16-byte aligned) go four elements per thread with their loads issued up front, and the
// updated values are written straight into the resident copies (Ws f32, Wd f64) instead of
// re-reading the rows afterwards. The other slices (b1, W2 columns, b2) are tiny.
__device__ void exchange_shard_mlp(float* p, const ShardTable& t, int s, const Slice& sl, float a, float* Ws,
                                   double* Wd, uint32_t F, uint32_t Fd) {
  const uint64_t b0 = t.begin[s], b1 = t.begin[s + 1];
  const uint64_t lo = sl.lo[0];
  const uint32_t n = sl.cols[0];  // Uo * F, one row
  float* m0 = t.ptr[s] - b0;      // m0[g] = center element g
  for (uint32_t j = threadIdx.x * 4; j < n; j += kFT * 4) {
    const uint64_t g = lo + j;
    float w[4], m[4], wo[4], mo[4];
    bool in[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) in[q] = g + q >= b0 && g + q < b1 && j + q < n;
    if (in[0] && in[3] && ((g - b0) & 3) == 0 && (g & 3) == 0) {
      const float4 wv = *reinterpret_cast<const float4*>(p + g);
      const float4 mv = __ldcg(reinterpret_cast<const float4*>(m0 + g));
      w[0] = wv.x, w[1] = wv.y, w[2] = wv.z, w[3] = wv.w;
      m[0] = mv.x, m[1] = mv.y, m[2] = mv.z, m[3] = mv.w;
#pragma unroll
      for (int q = 0; q < 4; ++q) elastic_elem(w[q], m[q], a, wo[q], mo[q]);
      *reinterpret_cast<float4*>(p + g) = make_float4(wo[0], wo[1], wo[2], wo[3]);
      __stcg(reinterpret_cast<float4*>(m0 + g), make_float4(mo[0], mo[1], mo[2], mo[3]));
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (!in[q]) continue;
        elastic_elem(p[g + q], __ldcg(m0 + g + q), a, wo[q], mo[q]);
        p[g + q] = wo[q];
        __stcg(m0 + g + q, mo[q]);
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (!in[q]) continue;
      const uint32_t local = j + q, uu = local / F, i = local - uu * F;
      Ws[local] = wo[q];
      Wd[uu * Fd + i] = static_cast<double>(wo[q]);
    }
  }
  for (int k = 1; k < sl.n; ++k) {
    const uint32_t nk = sl.rows[k] * sl.cols[k];
    for (uint32_t j = threadIdx.x; j < nk; j += kFT) {
      const uint32_t r = j / sl.cols[k];
      const uint64_t g = sl.lo[k] + r * sl.row_stride[k] + (j - r * sl.cols[k]);
      if (g >= b0 && g < b1) exchange_elem(p, t, s, g, a);
    }
  }
}

// Unordered (LockFree) exchange of the whole slice in one pass: every element goes to the
// shard that holds it (no per-shard pass and barrier), so the remote loads of all shards
// are in flight together.
__device__ __forceinline__ int shard_of(const ShardTable& t, uint64_t g) {
  int s = 0;
  while (s + 1 < t.n && g >= t.begin[s + 1]) ++s;
  return s;
}

__device__ void exchange_all_mlp(float* p, const ShardTable& t, const Slice& sl, float a, float* Ws, double* Wd,
                                 uint32_t F, uint32_t Fd) {
  const uint64_t lo = sl.lo[0];
  const uint32_t n = sl.cols[0];  // own W1 rows: Uo * F, one row, 16-byte aligned
  for (uint32_t j = threadIdx.x * 4; j < n; j += kFT * 4) {
    const uint64_t g = lo + j;
    bool in[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) in[q] = j + q < n;  // n % 4 != 0: the last group is partial
    const int s0 = shard_of(t, g), s3 = shard_of(t, g + 3);
    float wo[4], mo[4];
    if (in[3] && s0 == s3 && ((g - t.begin[s0]) & 3) == 0 && (g & 3) == 0) {
      float* m = t.ptr[s0] + (g - t.begin[s0]);
      const float4 wv = *reinterpret_cast<const float4*>(p + g);
      const float4 mv = __ldcg(reinterpret_cast<const float4*>(m));
      const float w[4] = {wv.x, wv.y, wv.z, wv.w}, mm[4] = {mv.x, mv.y, mv.z, mv.w};
#pragma unroll
      for (int q = 0; q < 4; ++q) elastic_elem(w[q], mm[q], a, wo[q], mo[q]);
      *reinterpret_cast<float4*>(p + g) = make_float4(wo[0], wo[1], wo[2], wo[3]);
      __stcg(reinterpret_cast<float4*>(m), make_float4(mo[0], mo[1], mo[2], mo[3]));
    } else {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (!in[q]) continue;
        const int sq = shard_of(t, g + q);
        float* m = t.ptr[sq] + (g + q - t.begin[sq]);
        elastic_elem(p[g + q], __ldcg(m), a, wo[q], mo[q]);
        p[g + q] = wo[q];
        __stcg(m, mo[q]);
      }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (!in[q]) continue;
      const uint32_t local = j + q, uu = local / F, i = local - uu * F;
      Ws[local] = wo[q];
      Wd[uu * Fd + i] = static_cast<double>(wo[q]);
    }
  }
  for (int k = 1; k < sl.n; ++k) {
    const uint32_t nk = sl.rows[k] * sl.cols[k];
    for (uint32_t j = threadIdx.x; j < nk; j += kFT) {
      const uint32_t r = j / sl.cols[k];
      const uint64_t g = sl.lo[k] + r * sl.row_stride[k] + (j - r * sl.cols[k]);
      exchange_elem(p, t, shard_of(t, g), g, a);
    }
  }
}

__device__ void do_exchange_mlp(const FusedArgs& A, float* p, const Slice& sl, uint64_t ticket, unsigned int G,
                                float* Ws, double* Wd, uint32_t F, uint32_t Fd) {
  const ShardTable& t = A.table;
  const bool ordered = ticket != kNoTicket;
  if (!ordered) {
    exchange_all_mlp(p, t, sl, A.alpha, Ws, Wd, F, Fd);
    __syncthreads();
    if (threadIdx.x == 0 && blockIdx.x == 0) atomicAdd_system(&t.flags[0]->exchanges, 1ull);
    return;
  }
  for (int s = 0; s < t.n; ++s) {
    if (ordered) {
      __shared__ int s_timeout;
      if (threadIdx.x == 0) {
        s_timeout = !wait_seq_eq(reinterpret_cast<const uint64_t*>(&t.flags[s]->seq), ticket, 64);
        if (s_timeout) {
          atomicAdd_system(&t.flags[s]->timeouts, 1ull);
          atomicOr(&A.st->flags, DS_FLAG_TICKET_TIMEOUT);
        }
      }
      __syncthreads();
      if (s_timeout) return;
    }
    exchange_shard_mlp(p, t, s, sl, A.alpha, Ws, Wd, F, Fd);
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
  double cut;       // launch constants (DevState), cached so the per-step update
  uint32_t tau;     // touches no global memory
  int32_t adaptive;
  uint32_t since;
  uint32_t fire, period;
};

__device__ __forceinline__ void policy_update(PolicyLocal& pl, double loss) {
  pl.cum = dadd(pl.cum, loss);
  pl.since += 1;
  const bool fire = pl.adaptive ? (pl.cum > pl.cut) : (pl.since == pl.tau);
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
  uint32_t CW;     // X columns per f64 chunk (converted once per element, see below)
  uint32_t CWs;    // f64 chunk row stride (doubles)
  bool bulk_x;     // X rows by TMA bulk copies and 128-bit loads (F % 4 == 0)
  bool bulk_a;     // activation rows by TMA bulk copies (H % 2 == 0)
  // Region `un` is time-shared: f64 X chunks during the forward and the dW1 phase,
  // activations (as) + W2 in f64 (w2) in between.
  size_t x, w, wd, un, w2, as, z, e, d1, lr, rs, bars, total;
};

__host__ __device__ inline SmemPlan make_plan(uint32_t F, uint32_t H, uint32_t C, uint32_t B, uint32_t G) {
  SmemPlan p{};
  const bool hidden = H > 0;
  const uint32_t U = hidden ? (H + G - 1) / G : 0;
  p.bulk_x = (F % 4) == 0;
  p.Fs = p.bulk_x ? F + 4 : (F | 1u);
  // activations are unit-major [H][B] in global and shared memory: one contiguous
  // block (TMA), and lane == row reads are conflict-free in the logits
  p.bulk_a = hidden && (static_cast<size_t>(H) * B) % 2 == 0;
  p.Hs = B;
  p.H2 = hidden ? ((H % 2) == 0 ? H + 2 : H + 1) : 0;
  auto al = [](size_t v) { return (v + 127) & ~static_cast<size_t>(127); };
  const size_t as_bytes = hidden ? al(static_cast<size_t>(H) * B * 8) : 0;
  const size_t w2_bytes = hidden ? al(static_cast<size_t>(C) * p.H2 * 8) : 0;
  // widest chunk (multiple of 16 columns, <= 256) that fits where as + w2 live
  uint32_t cw = 256;
  if (hidden) {
    while (cw > 16 && static_cast<size_t>(B) * (cw + 2) * 8 > as_bytes + w2_bytes) cw -= 16;
  }
  p.CW = cw;
  p.CWs = cw + 2;
  const size_t chunk_bytes = al(static_cast<size_t>(B) * p.CWs * 8);
  size_t off = 0;
  p.x = off;   off = al(off + static_cast<size_t>(B) * p.Fs * 4);
  p.w = off;   off = al(off + static_cast<size_t>(hidden ? U : C) * F * 4);
  p.wd = off;  off = al(off + (hidden ? static_cast<size_t>(U) * F * 8 : 0));
  p.un = off;
  p.as = off;
  p.w2 = off + as_bytes;
  off = al(off + (hidden ? (as_bytes + w2_bytes > chunk_bytes ? as_bytes + w2_bytes : chunk_bytes) : 0));
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

// Xd[r, 0:cw] = (double) Xs[r, c0:c0+cw] for r < R: one warp per row, float4 -> 2 x
// double2 (no per-element index arithmetic; F2F is the only real cost).
__device__ __forceinline__ void convert_chunk(double* Xd, uint32_t CWs, const float* Xs, uint32_t Fs, uint32_t R,
                                              uint32_t c0, uint32_t cw, bool vec) {
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = kFT / 32;
  for (uint32_t r = warp; r < R; r += nwarps) {
    const float* src = Xs + static_cast<size_t>(r) * Fs + c0;
    double* dst = Xd + static_cast<size_t>(r) * CWs;
    if (vec) {
      const float4* s4 = reinterpret_cast<const float4*>(src);
      double2* d2 = reinterpret_cast<double2*>(dst);
      for (uint32_t q = lane; q < cw / 4; q += 32) {
        const float4 v = s4[q];
        d2[2 * q] = make_double2(static_cast<double>(v.x), static_cast<double>(v.y));
        d2[2 * q + 1] = make_double2(static_cast<double>(v.z), static_cast<double>(v.w));
      }
    } else {
      for (uint32_t j = lane; j < cw; j += 32) dst[j] = static_cast<double>(src[j]);
    }
  }
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
  double* Wd = reinterpret_cast<double*>(smem_raw + sp.wd);  // own W1 rows as f64 (exact copy of Ws)
  double* Xd = reinterpret_cast<double*>(smem_raw + sp.un);  // B x CWs f64 chunk of X (time-shared)
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
  __shared__ unsigned int s_nbar;
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
    s_nbar = 0;
    s_pol.cum = st->cum;
    s_pol.cut = st->cut;
    s_pol.tau = st->tau;
    s_pol.adaptive = st->adaptive;
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
    for (uint32_t e = tid; e < nW; e += kFT) {
      const float v = ldcg(src + e);
      Ws[e] = v;
      if constexpr (kHidden) Wd[e] = static_cast<double>(v);
    }
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
      // Forward in f64 chunks of CW columns: every X element is converted to f64 once
      // (F2F runs at a quarter of the FP64 rate on B200) by all threads, then the chain
      // threads (one per (row, unit), R*Uo <= kFT) continue their reference-order sums.
      const uint32_t t_ch = tid;
      const bool chain = t_ch < R * Uo;
      const uint32_t cr = chain ? t_ch / Uo : 0, cuu = chain ? t_ch - cr * Uo : 0;
      double zc = chain ? static_cast<double>(ldcg(P + b1 + u0 + cuu)) : 0.0;
      for (uint32_t c0 = 0; c0 < F; c0 += sp.CW) {
        const uint32_t cw = F - c0 < sp.CW ? F - c0 : sp.CW;
        __syncthreads();  // previous chunk consumed
        convert_chunk(Xd, sp.CWs, Xs, Fs, R, c0, cw, sp.bulk_x && (cw % 4) == 0);
        __syncthreads();
        if (chain) zc = dot_f64_exact(zc, Wd + cuu * F + c0, Xd + cr * sp.CWs, cw, (cw % 2) == 0 && (F % 2) == 0);
      }
      if (chain) act[static_cast<size_t>(u0 + cuu) * B + cr] = tanh(zc);
      stamp(A.prof, step, 2);
      // grid barrier; thread 0 also samples the failure flags of the previous iteration
      __syncthreads();
      if (tid == 0) {
        grid_arrive_wait(A.bar, s_nbar, G);
        s_flags = *reinterpret_cast<volatile uint32_t*>(&st->flags);
        fence_proxy_async();  // other CTAs' generic writes (act, W2) before our async reads
        if (sp.bulk_a && !s_flags) {
          const uint32_t total = H * B * 8;  // [H][B] block, rows >= R unused
          mbar_arrive_expect_tx(bar_a, total);
          for (uint32_t off = 0; off < total; off += 32768)
            bulk_g2s(reinterpret_cast<unsigned char*>(As) + off, reinterpret_cast<const unsigned char*>(act) + off,
                     total - off < 32768 ? total - off : 32768, bar_a);
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
        for (uint32_t e = tid; e < H * B; e += kFT) As[e] = __ldcg(act + e);
      }
      {  // W2 -> f64 rows: one warp per class row, coalesced, all loads issued first
        const uint32_t warp = tid >> 5, lane = tid & 31;
        for (uint32_t c = warp; c < C; c += kFT / 32) {
          const float* src = P + w2 + static_cast<size_t>(c) * H;
          double* dst = W2d + static_cast<size_t>(c) * H2;
          for (uint32_t u0c = 0; u0c < H; u0c += 8 * 32) {
            float v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const uint32_t u = u0c + k * 32 + lane;
              v[k] = u < H ? ldcg(src + u) : 0.0f;
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
              const uint32_t u = u0c + k * 32 + lane;
              if (u < H) dst[u] = static_cast<double>(v[k]);
            }
          }
        }
      }
      if (sp.bulk_a) {
        mbar_wait(bar_a, phase_a);
        phase_a ^= 1;
      }
      __syncthreads();
      stamp(A.prof, step, 4);
      // Logits, lane == batch row, each warp two classes (two interleaved chains): the
      // activation loads are conflict-free ([H][B] layout) and shared by both chains,
      // the W2 loads are warp broadcasts. Reference order: b2[c] + sum_u in u order.
      {
        const uint32_t warp = tid >> 5, lane = tid & 31;
        const uint32_t nwl = (C + 1) / 2 < kFT / 32 ? (C + 1) / 2 : kFT / 32;
        for (uint32_t r0 = 0; r0 < R; r0 += 32) {
          const uint32_t r = r0 + lane;
          if (warp >= nwl || r >= R) continue;
          for (uint32_t c = warp; c < C; c += 2 * nwl) {
            const uint32_t c2 = c + nwl;
            const bool has2 = c2 < C;
            const double* wa = W2d + static_cast<size_t>(c) * H2;
            const double* wb = W2d + static_cast<size_t>(has2 ? c2 : c) * H2;
            const double* a = As + r;
            double za = static_cast<double>(ldcg(P + b2 + c));
            double zb = has2 ? static_cast<double>(ldcg(P + b2 + c2)) : 0.0;
            double pa[8], pb[8], qa[8], qb[8];
            const uint32_t nb = H / 8;
            auto prod = [&](uint32_t blk, double (&xa)[8], double (&xb)[8]) {
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                const double av = a[static_cast<size_t>(blk * 8 + k) * B];
                xa[k] = dmul(wa[blk * 8 + k], av);
                xb[k] = dmul(wb[blk * 8 + k], av);
              }
            };
            if (nb) {
              prod(0, pa, pb);
              for (uint32_t blk = 1; blk < nb; ++blk) {
                prod(blk, qa, qb);
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                  za = dadd(za, pa[k]);
                  zb = dadd(zb, pb[k]);
                  pa[k] = qa[k];
                  pb[k] = qb[k];
                }
              }
#pragma unroll
              for (int k = 0; k < 8; ++k) {
                za = dadd(za, pa[k]);
                zb = dadd(zb, pb[k]);
              }
            }
            for (uint32_t u = nb * 8; u < H; ++u) {
              const double av = a[static_cast<size_t>(u) * B];
              za = dadd(za, dmul(wa[u], av));
              zb = dadd(zb, dmul(wb[u], av));
            }
            Z[static_cast<size_t>(r) * C + c] = za;
            if (has2) Z[static_cast<size_t>(r) * C + c2] = zb;
          }
        }
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
        const double a = As[static_cast<size_t>(u) * Hs + r];
        D1[r * U + uu] = dmul(p, dsub(1.0, dmul(a, a)));
      }
      __syncthreads();
      // own W2 columns and b2 first: they read As / W2d, whose shared region the f64
      // X chunks of the dW1 phase reuse next
      for (uint32_t e = tid; e < C * Uo; e += kFT) {
        const uint32_t c = e / Uo, uu = e - c * Uo, u = u0 + uu;
        double acc = 0.0;
        for (uint32_t r = 0; r < R; ++r)
          acc = dadd(acc, dmul(Z[static_cast<size_t>(r) * C + c], As[static_cast<size_t>(u) * Hs + r]));
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
      // own b1: row-order sums of delta1 (model.cpp:218)
      for (uint32_t uu = tid; uu < Uo; uu += kFT) {
        double acc = 0.0;
        for (uint32_t r = 0; r < R; ++r) acc = dadd(acc, D1[r * U + uu]);
        const uint64_t g = b1 + u0 + uu;
        Pn[g] = sgd_apply(acc, inv_b, ldcg(P + g), A.eta, A.wd, bad);
      }
      stamp(A.prof, step, 9);
      // own W1 rows, f64 X chunks again: dW1[u,i] = sum_r delta1[r,u] * x[r,i] in row
      // order (model.cpp:219-221), four independent chains per thread, products of row
      // r+1 formed before the adds of row r
      for (uint32_t c0 = 0; c0 < F; c0 += sp.CW) {
        const uint32_t cw = F - c0 < sp.CW ? F - c0 : sp.CW;
        __syncthreads();
        convert_chunk(Xd, sp.CWs, Xs, Fs, R, c0, cw, sp.bulk_x && (cw % 4) == 0);
        __syncthreads();
        // one thread per column j: one Xd load feeds the chains of every owned unit
        // (up to kMaxU interleaved), products of row r+1 formed before row r's adds
        constexpr uint32_t kMaxU = 4;
        for (uint32_t j = tid; j < cw; j += kFT) {
          for (uint32_t ub = 0; ub < Uo; ub += kMaxU) {
            const uint32_t nu = Uo - ub < kMaxU ? Uo - ub : kMaxU;
            double acc[kMaxU], pc[kMaxU], pn[kMaxU];
#pragma unroll
            for (uint32_t k = 0; k < kMaxU; ++k) {
              acc[k] = 0.0;
              pc[k] = k < nu ? dmul(D1[ub + k], Xd[j]) : 0.0;
            }
            for (uint32_t r = 1; r < R; ++r) {
              const double x = Xd[r * sp.CWs + j];
#pragma unroll
              for (uint32_t k = 0; k < kMaxU; ++k) pn[k] = k < nu ? dmul(D1[r * U + ub + k], x) : 0.0;
#pragma unroll
              for (uint32_t k = 0; k < kMaxU; ++k) {
                acc[k] = dadd(acc[k], pc[k]);
                pc[k] = pn[k];
              }
            }
#pragma unroll
            for (uint32_t k = 0; k < kMaxU; ++k) {
              if (k >= nu) continue;
              acc[k] = dadd(acc[k], pc[k]);
              const uint32_t uu = ub + k, i = c0 + j;
              const float o = sgd_apply(acc[k], inv_b, Ws[uu * F + i], A.eta, A.wd, bad);
              Ws[uu * F + i] = o;
              Wd[uu * F + i] = static_cast<double>(o);
              Pn[w1 + static_cast<uint64_t>(u0 + uu) * F + i] = o;
            }
          }
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
      policy_update(s_pol, s_loss);
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
        if (kHidden) grid_barrier(A.bar, s_nbar, G);
        else __syncthreads();
        if (tid == 0) s_ticket = __ldcg(slot);
        __syncthreads();
        tk = s_ticket;
      }
      do_exchange(A, Pn, sl, tk, kHidden ? G : 1u);
      // the exchange moved the resident rows too: refresh them from params[cur^1]
      const uint32_t nW = kHidden ? Uo * F : C * F;
      const float* src = Pn + (kHidden ? w1 + static_cast<uint64_t>(u0) * F : 0);
      for (uint32_t e = tid; e < nW; e += kFT) {
        const float v = src[e];
        Ws[e] = v;
        if constexpr (kHidden) Wd[e] = static_cast<double>(v);
      }
      ++xcount;
    }
    cur ^= 1;
    __syncthreads();
    stamp(A.prof, step, 8);
  }
  if constexpr (kHidden) {
    grid_barrier(A.bar, s_nbar, G);  // failures of the last iteration become visible here
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


// ======================================================================================
// One-hidden-layer MLP: the persistent step kernel.
//
// Per iteration the batch rows land once in shared memory as f32 (TMA bulk copies, the
// next batch prefetched into L2). Both passes that need X in f64 — the forward dot
// products and dW1 — run as producer/consumer pipelines inside the CTA: producer warps
// convert 128-column chunks to f64 (F2F.F64.F32 is quarter-rate on B200, so each
// element is converted once per pass, off the consumers' critical path) into a double
// buffer while consumer warps run the reference-order chains on the previous chunk;
// named barriers (bar.sync / bar.arrive) hand the buffers back and forth.
// ======================================================================================
struct MlpPlan {
  uint32_t Fs, Fd, CW, CWs, nck, H2;
  size_t xs, w, wd, un, as, w2, z, e, d1, lr, rs, ri, bars, chunk, total;
};

__host__ __device__ inline MlpPlan make_mlp_plan(uint32_t F, uint32_t H, uint32_t C, uint32_t B, uint32_t G) {
  MlpPlan p{};
  const uint32_t U = (H + G - 1) / G;
  p.Fs = (F % 4) == 0 ? F + 4 : (F | 1u);  // f32 rows: 16-byte multiple for TMA and float4
  p.Fd = F + ((F % 2) == 0 ? 2 : 1);        // f64 W1 rows: shifted banks between units
  p.H2 = (H % 2) == 0 ? H + 2 : H + 1;
  auto al = [](size_t v) { return (v + 127) & ~static_cast<size_t>(127); };
  const size_t as_bytes = al(static_cast<size_t>(H) * B * 8);
  const size_t w2_bytes = al(static_cast<size_t>(C) * p.H2 * 8);
  for (uint32_t cw = 128;; cw -= 16) {
    p.CW = cw;
    p.CWs = cw + 2;
    p.nck = (F + cw - 1) / cw;
    p.chunk = al(static_cast<size_t>(B) * p.CWs * 8);
    const size_t un = 2 * p.chunk > as_bytes + w2_bytes ? 2 * p.chunk : as_bytes + w2_bytes;
    size_t off = 0;
    p.xs = off;  off = al(off + static_cast<size_t>(B) * p.Fs * 4);
    p.w = off;   off = al(off + static_cast<size_t>(U) * F * 4);
    p.wd = off;  off = al(off + static_cast<size_t>(U) * p.Fd * 8);
    p.un = off;  p.as = off;  p.w2 = off + as_bytes;  off = al(off + un);
    p.z = off;   off = al(off + static_cast<size_t>(B) * C * 8);
    p.e = off;   off = al(off + static_cast<size_t>(B) * C * 8);
    p.d1 = off;  off = al(off + static_cast<size_t>(B) * U * 8);
    p.lr = off;  off = al(off + static_cast<size_t>(B) * 8);
    p.rs = off;  off = al(off + static_cast<size_t>(B) * 8 * 2 + static_cast<size_t>(B) * 4 * 2);
    p.ri = off;  off = al(off + static_cast<size_t>(B) * 4);
    p.bars = off; off = al(off + 8 * (p.nck + 2));
    p.total = off;
    if (p.total <= 216 * 1024 || cw == 16) break;
  }
  return p;
}

__device__ __forceinline__ void named_sync(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void named_arrive(uint32_t id, uint32_t n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

// Producer side of one chunk: rows R of Xs columns [c0, c0+cw) -> dst (f64, row stride
// CWs). Warps [w0, w0+nw) take rows round-robin, lanes take column pairs (LDS.64 in,
// STS.128 out: both at the shared-memory wavefront minimum).
__device__ __forceinline__ void produce_chunk(double* dst, uint32_t CWs, const float* Xs, uint32_t Fs, uint32_t R,
                                              uint32_t c0, uint32_t cw, bool vec, uint32_t w0, uint32_t nw) {
  const uint32_t warp = (threadIdx.x >> 5) - w0, lane = threadIdx.x & 31;
  for (uint32_t r = warp; r < R; r += nw) {
    const float* src = Xs + static_cast<size_t>(r) * Fs + c0;
    double* d = dst + static_cast<size_t>(r) * CWs;
    if (vec) {
      const float2* s2 = reinterpret_cast<const float2*>(src);
      double2* d2 = reinterpret_cast<double2*>(d);
#pragma unroll 2
      for (uint32_t q = lane; q < cw / 2; q += 32) {
        const float2 v = s2[q];
        d2[q] = make_double2(static_cast<double>(v.x), static_cast<double>(v.y));
      }
    } else {
      for (uint32_t j = lane; j < cw; j += 32) d[j] = static_cast<double>(src[j]);
    }
  }
}

// dW1 for NU units [ub, ub+NU) of this CTA: thread tid owns columns j = tid + k*kFT.
// Rows are unrolled by 4 with the loads of the next group issued before the current
// group's chain adds (in-order issue would otherwise expose the LDS latency per row).
template <int NU>
__device__ __forceinline__ void dw1_columns(const FusedArgs& A, const float* Xs, uint32_t Fs, const double* D1,
                                            uint32_t U, uint32_t ub, uint32_t u0, uint32_t R, double inv_b,
                                            float* Ws, double* Wd, uint32_t Fd, float* Pn, uint64_t w1,
                                            uint32_t& bad) {
  const uint32_t F = A.F;
  for (uint32_t j = threadIdx.x; j < F; j += kFT) {
    double acc[NU];
#pragma unroll
    for (int q = 0; q < NU; ++q) acc[q] = 0.0;
    const float* xc = Xs + j;
    uint32_t r = 0;
    for (; r + 4 <= R; r += 4) {
      double x[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) x[t] = static_cast<double>(xc[static_cast<size_t>(r + t) * Fs]);
#pragma unroll
      for (int t = 0; t < 4; ++t)
#pragma unroll
        for (int q = 0; q < NU; ++q) acc[q] = dadd(acc[q], dmul(D1[(r + t) * U + ub + q], x[t]));
    }
    for (; r < R; ++r) {
      const double x = static_cast<double>(xc[static_cast<size_t>(r) * Fs]);
#pragma unroll
      for (int q = 0; q < NU; ++q) acc[q] = dadd(acc[q], dmul(D1[r * U + ub + q], x));
    }
#pragma unroll
    for (int q = 0; q < NU; ++q) {
      const uint32_t uu = ub + q;
      const float o = sgd_apply(acc[q], inv_b, Ws[uu * F + j], A.eta, A.wd, bad);
      Ws[uu * F + j] = o;
      Wd[uu * Fd + j] = static_cast<double>(o);
      Pn[w1 + static_cast<uint64_t>(u0 + uu) * F + j] = o;
    }
  }
}

// Logits z[r][c] = b2[c] + sum_u W2[c][u] * a[r][u] in the reference's order (model.cpp:
// 205-209) for NC classes cb, cb+4, ... of row r: NC interleaved chains per thread, the
// activation loaded once for all of them, products one 4-element block ahead.
constexpr uint32_t kLogitChains = 3;
template <int NC>
__device__ __forceinline__ void logit_chains(double* Z, const double* W2d, uint32_t H2, const double* As, uint32_t B,
                                             uint32_t H, const float* b2, uint32_t r, uint32_t C, uint32_t cb) {
  const double2* w[NC];
  double z[NC];
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    w[i] = reinterpret_cast<const double2*>(W2d + static_cast<size_t>(cb + 4 * i) * H2);
    z[i] = static_cast<double>(ldcg(b2 + cb + 4 * i));
  }
  const double* a = As + r;
  double p[NC][4], q[NC][4];
  auto prod = [&](uint32_t blk, double (&x)[NC][4]) {
    double av[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) av[k] = a[static_cast<size_t>(blk * 4 + k) * B];
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      const double2 w01 = w[i][blk * 2], w23 = w[i][blk * 2 + 1];
      x[i][0] = dmul(w01.x, av[0]);
      x[i][1] = dmul(w01.y, av[1]);
      x[i][2] = dmul(w23.x, av[2]);
      x[i][3] = dmul(w23.y, av[3]);
    }
  };
  const uint32_t nb = H / 4;
  if (nb) {
    prod(0, p);
    for (uint32_t blk = 1; blk < nb; ++blk) {
      prod(blk, q);
#pragma unroll
      for (int k = 0; k < 4; ++k)
#pragma unroll
        for (int i = 0; i < NC; ++i) {
          z[i] = dadd(z[i], p[i][k]);
          p[i][k] = q[i][k];
        }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
#pragma unroll
      for (int i = 0; i < NC; ++i) z[i] = dadd(z[i], p[i][k]);
  }
  for (uint32_t u = nb * 4; u < H; ++u) {
    const double av = a[static_cast<size_t>(u) * B];
#pragma unroll
    for (int i = 0; i < NC; ++i)
      z[i] = dadd(z[i], dmul(W2d[static_cast<size_t>(cb + 4 * i) * H2 + u], av));
  }
#pragma unroll
  for (int i = 0; i < NC; ++i) Z[static_cast<size_t>(r) * C + cb + 4 * i] = z[i];
}

constexpr uint32_t kBarFull = 2, kBarEmpty = 4;  // named barrier ids (+ buffer index)

// Thread-block-cluster helpers: a store into a peer CTA's shared memory (DSMEM) and the
// cluster barrier.
__device__ __forceinline__ void st_cluster_f64(double* local, uint32_t rank, double v) {
  uint32_t ra;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(smem_u32(local)), "r"(rank));
  asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(ra), "d"(v) : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

__global__ void __launch_bounds__(kFT, 1) mlp_kernel(FusedArgs A) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const unsigned int G = gridDim.x;
  const uint32_t F = A.F, H = A.H, C = A.C, B = A.B;
  const MlpPlan sp = make_mlp_plan(F, H, C, B, G);
  const uint32_t CW = sp.CW, CWs = sp.CWs, nck = sp.nck, H2 = sp.H2, Fs = sp.Fs, Fd = sp.Fd;
  const uint32_t U = (H + G - 1) / G;
  const uint32_t u0 = blockIdx.x * U;
  const uint32_t Uo = u0 < H ? (u0 + U <= H ? U : H - u0) : 0;
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t cwarps = (B * U + 31) / 32;  // forward consumer (chain) warps
  const bool vecx = (F % 4) == 0 && (CW % 4) == 0;
  uint32_t crank, csize;  // thread-block cluster: the CTAs of a cluster split the logits by rows
  asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
  asm("mov.u32 %0, %%cluster_nctarank;" : "=r"(csize));

  float* Xs = reinterpret_cast<float*>(smem_raw + sp.xs);    // B x Fs batch rows (f32)
  float* Ws = reinterpret_cast<float*>(smem_raw + sp.w);     // own W1 rows f32 (the parameters)
  double* Wd = reinterpret_cast<double*>(smem_raw + sp.wd);  // same rows as f64, row stride Fd
  double* XD0 = reinterpret_cast<double*>(smem_raw + sp.un); // 2 x [B][CWs] f64 chunk buffers ...
  double* XD1 = reinterpret_cast<double*>(smem_raw + sp.un + sp.chunk);
  double* As = reinterpret_cast<double*>(smem_raw + sp.as);  // ... time-shared with [H][B] activations
  double* W2d = reinterpret_cast<double*>(smem_raw + sp.w2); // ... and [C][H2] W2 in f64
  double* Z = reinterpret_cast<double*>(smem_raw + sp.z);
  double* E = reinterpret_cast<double*>(smem_raw + sp.e);
  double* D1 = reinterpret_cast<double*>(smem_raw + sp.d1);
  double* Lr = reinterpret_cast<double*>(smem_raw + sp.lr);
  double* Zmax = reinterpret_cast<double*>(smem_raw + sp.rs);
  double* Lse = Zmax + B;
  uint32_t* Lab = reinterpret_cast<uint32_t*>(Lse + B);
  uint32_t* Ri = reinterpret_cast<uint32_t*>(smem_raw + sp.ri);      // next batch's shard rows
  uint64_t* abar = reinterpret_cast<uint64_t*>(smem_raw + sp.bars);  // activations
  uint64_t* xbar = abar + 1;  // [nck]: column chunk k of the batch rows landed
  __shared__ double s_loss;
  __shared__ uint32_t s_bad, s_stop, s_flags;
  __shared__ unsigned int s_nbar;
  __shared__ PolicyLocal s_pol;
  __shared__ unsigned long long s_ticket;
  __shared__ uint32_t s_rrows[2];  // stream mode: rows of steps s (s & 1)

  const uint64_t w1 = 0, b1 = static_cast<uint64_t>(H) * F;
  const uint64_t w2 = b1 + H, b2 = w2 + static_cast<uint64_t>(C) * H;
  Slice sl;
  sl.n = 0;
  slice_add(sl, w1 + static_cast<uint64_t>(u0) * F, 1, Uo * F, 0);  // own W1 rows
  slice_add(sl, b1 + u0, 1, Uo, 0);                                  // own b1
  slice_add(sl, w2 + u0, C, Uo, H);                                  // own W2 columns
  if (blockIdx.x == 0) slice_add(sl, b2, 1, C, 0);                   // b2

  DevState* st = A.st;
  if (tid == 0) {
    s_nbar = 0;
    s_pol.cum = st->cum;
    s_pol.cut = st->cut;
    s_pol.tau = st->tau;
    s_pol.adaptive = st->adaptive;
    s_pol.since = st->since;
    s_pol.fire = 0;
    s_pol.period = 0;
    s_stop = st->err ? 1u : 0u;
    for (uint32_t k = 0; k < nck; ++k) mbar_init(xbar + k, kFT);
    mbar_init(abar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (s_stop) return;
  int cur = A.cur;
  uint64_t xcount = 0;
  uint32_t xph = 0, aph = 0;
  const unsigned long long it0 = st->iter;

  auto load_own_rows = [&](const float* P0) {  // Ws / Wd <- own W1 rows
    const float* src = P0 + w1 + static_cast<uint64_t>(u0) * F;
    for (uint32_t uu = warp; uu < Uo; uu += kFT / 32)
      for (uint32_t i = lane; i < F; i += 32) {
        const float v = ldcg(src + static_cast<size_t>(uu) * F + i);
        Ws[uu * F + i] = v;
        Wd[uu * Fd + i] = static_cast<double>(v);
      }
  };
  // Batch rows -> Xs, column-chunk-major so the forward starts on chunk 0 while the rest
  // lands: every thread issues 16-byte LDGSTS pieces, then arrives on chunk k's barrier.
  // (One bulk copy per row-chunk would put ~R*nck serialized TMA issues on one warp.)
  // The caller has synced the block since the last generic access of Xs.
  // Ri holds the batch's shard rows (staged earlier, so no global load sits in this loop).
  // Stream mode (host-fed ring, ds_engine_stream_*): step s's rows sit in ring slot
  // s % ring_slots once the host's H2D copies have landed — the copy engine writes the
  // slot's sequence word after the rows (same copy stream, in order). Thread 0 waits for
  // it (bounded: a stalled host raises DS_FLAG_STREAM_TIMEOUT instead of hanging the GPU).
  auto ring_wait = [&](uint64_t s) {
    if (tid == 0) {
      const uint32_t slot = static_cast<uint32_t>(s % A.ring_slots);
      const uint32_t want = static_cast<uint32_t>(s + 1) & 0xFFFFFu;  // sequence word: rows << 20 | step+1
      unsigned long long t0;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
      uint32_t rows = 1;
      while (true) {
        uint32_t v;
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(A.ring_ready + slot) : "memory");
        if ((v & 0xFFFFFu) == want) {
          rows = v >> 20;
          break;
        }
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > 20000000000ull) {
          atomicOr(&st->flags, DS_FLAG_STREAM_TIMEOUT);
          break;
        }
        __nanosleep(64);
      }
      s_rrows[s & 1] = rows;
    }
    __syncthreads();
  };
  auto step_rows = [&](uint64_t s) -> uint32_t { return A.ring ? s_rrows[s & 1] : A.plan_rows[s]; };
  auto step_x = [&](uint64_t s) -> const float* {
    return A.ring ? A.ring_X + (s % A.ring_slots) * static_cast<uint64_t>(B) * F : A.X;
  };
  auto issue_x = [&](uint64_t s) {
    if (A.ring) ring_wait(s);
    const uint32_t R = step_rows(s);
    const float* Xb = step_x(s);
    for (uint32_t k = 0; k < nck; ++k) {
      const uint32_t c = k * CW + 4 * lane;
      if (4 * lane < (F - k * CW < CW ? F - k * CW : CW))
        for (uint32_t r = warp; r < R; r += kFT / 32)
          cp_async16(Xs + static_cast<size_t>(r) * Fs + c, Xb + static_cast<uint64_t>(Ri[r]) * F + c);
      cp_async_arrive(xbar + k);
    }
  };
  load_own_rows(A.params[cur]);
  if (A.ring) {
    for (uint32_t r = tid; r < B; r += kFT) Ri[r] = r;
  } else if (A.steps > 0) {
    for (uint32_t r = tid; r < A.plan_rows[0]; r += kFT) Ri[r] = A.plan[r];
  }
  __syncthreads();
  if (vecx && A.steps > 0) issue_x(0);

  for (uint64_t step = 0; step < A.steps; ++step) {
    const uint32_t R = step_rows(step);
    const uint32_t* idx = A.plan + step * B;
    const float* P = A.params[cur];
    float* Pn = A.params[cur ^ 1];
    const double inv_b = 1.0 / static_cast<double>(R);
    stamp(A.prof, step, 0);
    if (tid == 0) s_bad = 0;
    if (tid < R) Lab[tid] = A.ring ? A.ring_y[(step % A.ring_slots) * B + tid] : A.y[idx[tid]];

    // ---- A: batch rows (TMA issued at the end of the previous step; generic path here) --
    if (!vecx) {
      __syncthreads();
      for (uint32_t r = warp; r < R; r += kFT / 32)
        for (uint32_t i = lane; i < F; i += 32) Xs[static_cast<size_t>(r) * Fs + i] = __ldg(A.X + static_cast<uint64_t>(idx[r]) * F + i);
      __syncthreads();
    }
    stamp(A.prof, step, 1);

    // ---- forward: consumers (chain warps) || producers (f64 chunk conversion) -----------
    double* act = A.act + static_cast<size_t>(step & 1) * H * B;
    if (warp < cwarps) {
      const bool chain = tid < R * Uo;
      const uint32_t cr = chain ? tid / Uo : 0, cuu = chain ? tid - cr * Uo : 0;
      double zc = chain ? static_cast<double>(ldcg(P + b1 + u0 + cuu)) : 0.0;
      for (uint32_t k = 0; k < nck; ++k) {
        const uint32_t b = k & 1, cw = F - k * CW < CW ? F - k * CW : CW;
        named_sync(kBarFull + b, kFT);
        const double* xd = (b ? XD1 : XD0) + static_cast<size_t>(cr) * CWs;
        if (chain) zc = dot_f64_exact(zc, Wd + cuu * Fd + k * CW, xd, cw, (cw % 2) == 0);
        if (k + 2 < nck) named_arrive(kBarEmpty + b, kFT);
      }
      if (chain) act[static_cast<size_t>(u0 + cuu) * B + cr] = tanh(zc);
    } else {
      for (uint32_t k = 0; k < nck; ++k) {
        const uint32_t b = k & 1, c0 = k * CW, cw = F - c0 < CW ? F - c0 : CW;
        if (k >= 2) named_sync(kBarEmpty + b, kFT);
        if (vecx) mbar_wait(xbar + k, xph);
        produce_chunk(b ? XD1 : XD0, CWs, Xs, Fs, R, c0, cw, vecx, cwarps, kFT / 32 - cwarps);
        named_arrive(kBarFull + b, kFT);
      }
    }
    xph ^= 1;
    stamp(A.prof, step, 2);
    // grid barrier; thread 0 samples the failure flags and starts the activation copy
    __syncthreads();
    stamp_cta(A.prof_cta, step, 0);
    if (tid == 0) {
      grid_arrive_wait(A.bar, s_nbar, G);
      s_flags = *reinterpret_cast<volatile uint32_t*>(&st->flags);
      if (A.ring && blockIdx.x == 0)  // every CTA's loads of this step's ring slot have landed
        asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(A.ring_consumed), "l"(step + 1) : "memory");
      fence_proxy_async();
      if (!s_flags) {
        const uint32_t total = H * B * 8;
        mbar_arrive_expect_tx(abar, total);
        for (uint32_t off = 0; off < total; off += 32768)
          bulk_g2s(reinterpret_cast<unsigned char*>(As) + off, reinterpret_cast<const unsigned char*>(act) + off,
                   total - off < 32768 ? total - off : 32768, abar);
      }
    }
    __syncthreads();
    stamp(A.prof, step, 3);
    stamp_cta(A.prof_cta, step, 1);
    if (s_flags) {
      if (blockIdx.x == 0 && tid == 0) {
        st->err = s_flags;
        st->bad_iter = it0 + step;
      }
      return;
    }
    // ---- B: W2 in f64, logits, softmax-CE ---------------------------------------------
    for (uint32_t c = warp; c < C; c += kFT / 32) {
      const float* src = P + w2 + static_cast<size_t>(c) * H;
      double* dst = W2d + static_cast<size_t>(c) * H2;
      for (uint32_t ub = 0; ub < H; ub += 8 * 32) {
        float v[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t u = ub + k * 32 + lane;
          v[k] = u < H ? ldcg(src + u) : 0.0f;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint32_t u = ub + k * 32 + lane;
          if (u < H) dst[u] = static_cast<double>(v[k]);
        }
      }
    }
    mbar_wait(abar, aph);
    aph ^= 1;
    __syncthreads();
    stamp(A.prof, step, 4);
    // Logits and softmax-CE. Every CTA needs all rows' output deltas, but computing them
    // is FP64-pipe bound (320 chains x 256 terms per CTA). The CTAs of a cluster split
    // the rows: each computes logits, softmax and deltas for R/csize rows, then reads the
    // others' rows from their shared memory (DSMEM) after one cluster barrier.
    const uint32_t rpr = (R + csize - 1) / csize;
    const uint32_t rlo = crank * rpr < R ? crank * rpr : R, rhi = rlo + rpr < R ? rlo + rpr : R;
    if (csize > 1) {
      for (uint32_t t = tid; t < (rhi - rlo) * C; t += kFT)
        logit_chains<1>(Z, W2d, H2, As, B, H, P + b2, rlo + t / C, C, t % C);
    } else {  // lane == row; a warp runs the chains of classes w, w+4, w+8, ... for its
              // rows (4 class sets, one per SM sub-partition: the As reads stay 4x, not Cx)
      const uint32_t ngroups = (R + 31) / 32;
      for (uint32_t item = warp; item < ngroups * 4; item += kFT / 32) {
        const uint32_t r = (item >> 2) * 32 + lane, cs = item & 3;
        if (r >= R) continue;
        for (uint32_t cb = cs; cb < C; cb += 4 * kLogitChains) {
          const uint32_t nc = (C - cb + 3) / 4 < kLogitChains ? (C - cb + 3) / 4 : kLogitChains;
          switch (nc) {
            case 1: logit_chains<1>(Z, W2d, H2, As, B, H, P + b2, r, C, cb); break;
            case 2: logit_chains<2>(Z, W2d, H2, As, B, H, P + b2, r, C, cb); break;
            default: logit_chains<3>(Z, W2d, H2, As, B, H, P + b2, r, C, cb); break;
          }
        }
      }
    }
    __syncthreads();
    stamp(A.prof, step, 5);
    for (uint32_t r = rlo + tid; r < rhi; r += kFT) {
      const double* z = Z + static_cast<size_t>(r) * C;
      double zmax = z[0];
      for (uint32_t c = 1; c < C; ++c) zmax = z[c] > zmax ? z[c] : zmax;
      Zmax[r] = zmax;
    }
    __syncthreads();
    for (uint32_t t = rlo * C + tid; t < rhi * C; t += kFT) E[t] = exp(dsub(Z[t], Zmax[t / C]));
    __syncthreads();
    for (uint32_t r = rlo + tid; r < rhi; r += kFT) {
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
    for (uint32_t t = rlo * C + tid; t < rhi * C; t += kFT) {
      const uint32_t r = t / C, c = t - r * C;
      const double d = dsub(exp(dsub(Z[t], Lse[r])), c == Lab[r] ? 1.0 : 0.0);
      Z[t] = d;
      for (uint32_t q = 1; q < csize; ++q) st_cluster_f64(Z + t, (crank + q) % csize, d);  // push to peers
    }
    if (csize > 1) {  // this rank's per-row losses to the peers, then one cluster barrier
      for (uint32_t t = tid; t < (rhi - rlo) * (csize - 1); t += kFT) {
        const uint32_t r = rlo + t % (rhi - rlo), q = 1 + t / (rhi - rlo);
        st_cluster_f64(Lr + r, (crank + q) % csize, Lr[r]);
      }
      cluster_sync_all();
    }
    __syncthreads();
    if (tid == kFT - 1) {
      double s = 0.0;
      for (uint32_t r = 0; r < R; ++r) s = dadd(s, Lr[r]);
      s_loss = dmul(s, inv_b);
      if (!isfinite(s_loss)) atomicOr(&s_bad, DS_FLAG_LOSS_NONFINITE);
      if (A.ring_loss && blockIdx.x == 0) A.ring_loss[step] = s_loss;  // zero-copy D2H of the result
    }
    if (!A.ring && step + 1 < A.steps)  // next batch's rows for issue_x (latency hidden by the backward)
      for (uint32_t r = tid; r < A.plan_rows[step + 1]; r += kFT) Ri[r] = A.plan[(step + 1) * B + r];
    // ---- C: backward. delta1 || W2 columns + b2 (different warps) ---------------------------
    stamp(A.prof, step, 6);
    uint32_t bad = 0;
    const uint32_t nct = cwarps * 32;
    if (tid < R * Uo) {  // delta1 (model.cpp:225-233)
      const uint32_t r = tid / Uo, uu = tid - r * Uo, u = u0 + uu;
      const double* d = Z + static_cast<size_t>(r) * C;
      double p = 0.0;
      for (uint32_t c = 0; c < C; ++c) p = dadd(p, dmul(d[c], W2d[static_cast<size_t>(c) * H2 + u]));
      const double a = As[static_cast<size_t>(u) * B + r];
      D1[r * U + uu] = dmul(p, dsub(1.0, dmul(a, a)));
    } else if (tid >= nct && tid < nct + C * Uo) {  // own W2 columns (model.cpp:219-221)
      const uint32_t e = tid - nct, c = e / Uo, uu = e - c * Uo, u = u0 + uu;
      double acc = 0.0;
      for (uint32_t r = 0; r < R; ++r)
        acc = dadd(acc, dmul(Z[static_cast<size_t>(r) * C + c], As[static_cast<size_t>(u) * B + r]));
      const uint64_t g = w2 + static_cast<uint64_t>(c) * H + u;
      Pn[g] = sgd_apply(acc, inv_b, static_cast<float>(W2d[static_cast<size_t>(c) * H2 + u]), A.eta, A.wd, bad);
    } else if (blockIdx.x == 0 && tid >= nct + C * Uo && tid < nct + C * Uo + C) {  // b2
      const uint32_t c = tid - nct - C * Uo;
      double acc = 0.0;
      for (uint32_t r = 0; r < R; ++r) acc = dadd(acc, Z[static_cast<size_t>(r) * C + c]);
      const uint64_t g = b2 + c;
      Pn[g] = sgd_apply(acc, inv_b, ldcg(P + g), A.eta, A.wd, bad);
    }
    __syncthreads();
    stamp(A.prof, step, 9);
    // ---- dW1 (+ b1): every thread owns whole columns j (all rows, its CTA's units) -----
    // Each X element is converted to f64 once, by the one thread that uses it for all
    // units; the row order of the sums is the reference's (model.cpp:219-221).
    if (tid >= kFT - Uo) {  // own b1: row-order sums of delta1
      const uint32_t uu = tid - (kFT - Uo);
      double acc = 0.0;
      for (uint32_t r = 0; r < R; ++r) acc = dadd(acc, D1[r * U + uu]);
      const uint64_t g = b1 + u0 + uu;
      Pn[g] = sgd_apply(acc, inv_b, ldcg(P + g), A.eta, A.wd, bad);
    }
    for (uint32_t ub = 0; ub < Uo; ub += 4) {
      const uint32_t nu = Uo - ub < 4 ? Uo - ub : 4;
      switch (nu) {
        case 1: dw1_columns<1>(A, Xs, Fs, D1, U, ub, u0, R, inv_b, Ws, Wd, Fd, Pn, w1, bad); break;
        case 2: dw1_columns<2>(A, Xs, Fs, D1, U, ub, u0, R, inv_b, Ws, Wd, Fd, Pn, w1, bad); break;
        case 3: dw1_columns<3>(A, Xs, Fs, D1, U, ub, u0, R, inv_b, Ws, Wd, Fd, Pn, w1, bad); break;
        default: dw1_columns<4>(A, Xs, Fs, D1, U, ub, u0, R, inv_b, Ws, Wd, Fd, Pn, w1, bad); break;
      }
    }
    bad = __reduce_or_sync(0xffffffffu, bad);
    if (bad && lane == 0) atomicOr(&s_bad, bad);
    __syncthreads();
    stamp(A.prof, step, 7);
    if (vecx && step + 1 < A.steps) issue_x(step + 1);  // Xs is free: overlap the exchange
    // ---- D: policy + exchange ------------------------------------------------------------
    if (s_bad && tid == 0) atomicOr(&st->flags, s_bad);  // all CTAs stop after the next barrier
    if (tid == 0) {
      policy_update(s_pol, s_loss);
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
    if (s_pol.fire && A.has_master) {
      uint64_t tk = kNoTicket;
      if (A.tickets) {
        tk = A.tickets[xcount];
      } else if (A.ticket_src) {
        unsigned long long* slot = reinterpret_cast<unsigned long long*>(A.bar + 4);
        if (blockIdx.x == 0 && tid == 0) *slot = atomicAdd_system(A.ticket_src, 1ull);
        grid_barrier(A.bar, s_nbar, G);
        if (tid == 0) s_ticket = __ldcg(slot);
        __syncthreads();
        tk = s_ticket;
      }
      do_exchange_mlp(A, Pn, sl, tk, G, Ws, Wd, F, Fd);  // also refreshes the resident own rows
      ++xcount;
    }
    cur ^= 1;
    __syncthreads();
    stamp(A.prof, step, 8);
  }
  grid_barrier(A.bar, s_nbar, G);
  const uint32_t fl = *reinterpret_cast<volatile uint32_t*>(&st->flags);
  if (fl) {
    if (blockIdx.x == 0 && tid == 0) {
      st->err = fl;
      st->bad_iter = it0 + A.steps;
    }
    return;
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
  uint32_t U = (H + cap - 1) / cap;
  // Units per CTA: more units per CTA = fewer CTAs pulling the same batch chunks
  // through L2 (the broadcast traffic is what bounds the X passes), at the cost of
  // more chains per SM. DS_FUSED_UNITS overrides the default.
  if (const char* env = std::getenv("DS_FUSED_UNITS")) {
    const int v = std::atoi(env);
    if (v > 0) U = static_cast<uint32_t>(v) > U ? static_cast<uint32_t>(v) : U;
  }
  return static_cast<int>((H + U - 1) / U);
}

size_t smem_for(uint32_t F, uint32_t H, uint32_t C, uint32_t B, uint32_t G) {
  return H > 0 ? make_mlp_plan(F, H, C, B, G).total : make_plan(F, H, C, B, G).total;
}

}  // namespace

int fused_grid(const ModelInfo& m, int device) { return grid_for(m, device); }

size_t fused_xb_doubles(const ModelInfo&, uint32_t, int) { return 0; }  // X stays f32 in shared memory

size_t fused_smem_bytes(const ModelInfo& m, uint32_t batch) {
  const uint32_t H = m.hidden.empty() ? 0 : m.hidden[0];
  return smem_for(m.n_features, H, m.n_classes, batch, static_cast<uint32_t>(grid_for(m, 0)));
}

int fused_supported(const ModelInfo& m, uint32_t batch, int device, const char** why) {
  if (m.kind == DS_MODEL_CIFAR10_QUICK || m.kind == DS_MODEL_ALEXNET) {
    if (why) *why = "convnet models run on the layered path";
    return DS_E_CONTRACT;
  }
  if (m.hidden.size() > 1) {
    if (why) *why = "more than one hidden layer";
    return DS_E_CONTRACT;
  }
  if (batch > 1024) {
    if (why) *why = "batch_size above 1024";
    return DS_E_CONTRACT;
  }
  if (!m.hidden.empty()) {
    const uint32_t G = static_cast<uint32_t>(grid_for(m, device));
    const uint32_t U = (m.hidden[0] + G - 1) / G;
    if (batch * U > static_cast<uint32_t>(kFT) - 128) {  // one forward chain per thread + producer warps
      if (why) *why = "batch x hidden units per CTA exceeds the block";
      return DS_E_CONTRACT;
    }
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
  DS_CUDA_TRY(cudaMemsetAsync(a.bar + kBarCounter, 0, sizeof(unsigned int), s));  // grid_barrier counter
  void* args[] = {const_cast<FusedArgs*>(&a)};
  if (a.H > 0) {
    DS_CUDA_TRY(cudaFuncSetAttribute(mlp_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    // Optional cooperative launch in thread-block clusters (DS_FUSED_CLUSTER=2|4|8): the
    // CTAs of a cluster split the logits/softmax rows and exchange the deltas through
    // DSMEM (see mlp_kernel). Measured neutral on B200 for 784-256-10 (the FP64 pipe work
    // it saves is paid back in the cluster barrier and the exp/log latency), so the
    // default is no clusters.
    unsigned cap = 1;
    if (const char* env = std::getenv("DS_FUSED_CLUSTER")) cap = static_cast<unsigned>(std::max(1, std::atoi(env)));
    // The cluster choice depends on (device, grid, smem, cap); engines on several threads
    // or devices share this cache, so it is keyed and locked.
    int dev = 0;
    cudaGetDevice(&dev);
    static std::mutex cache_mu;
    static std::map<std::tuple<int, int, size_t, unsigned>, unsigned> cache;
    const auto key = std::make_tuple(dev, grid, smem, cap);
    unsigned cached_cl = 1;
    bool have = false;
    {
      std::lock_guard<std::mutex> lk(cache_mu);
      auto it = cache.find(key);
      if (it != cache.end()) cached_cl = it->second, have = true;
    }
    if (!have) {
      unsigned pick = 1;
      for (unsigned cl = 8; cl >= 2; cl /= 2) {
        if (cl > cap || grid % cl) continue;
        cudaLaunchConfig_t q = {};
        q.gridDim = dim3(grid);
        q.blockDim = dim3(kFT);
        q.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cl;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        q.attrs = at;
        q.numAttrs = 1;
        int nclusters = 0;
        if (cudaOccupancyMaxActiveClusters(&nclusters, mlp_kernel, &q) == cudaSuccess &&
            nclusters * static_cast<int>(cl) >= grid) {
          pick = cl;
          break;
        }
        cudaGetLastError();
      }
      cached_cl = pick;
      std::lock_guard<std::mutex> lk(cache_mu);
      cache[key] = pick;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kFT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = cached_cl;
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    DS_CUDA_TRY(cudaLaunchKernelEx(&cfg, mlp_kernel, a));
  } else {
    DS_CUDA_TRY(cudaFuncSetAttribute(fused_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    DS_CUDA_TRY(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(fused_kernel<false>), dim3(1), dim3(kFT), args, smem, s));
  }
  return DS_OK;
}

}  // namespace dsb

void dsb::warm_fused_kernels() { dsb::load_kernels(dsb::fused_kernel<false>, dsb::fused_kernel<true>, dsb::mlp_kernel); }
