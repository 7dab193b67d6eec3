// conv_tc.cu — 5x5 pad-2 convolutions of the convnet as implicit GEMMs on the tcgen05
// tensor cores (kind::tf32: f32 operands rounded to tf32 by the tensor core, f32
// accumulation in TMEM).
//
// Forward / backward-data (conv5_tc_kernel): D[pixels x Cout] = A[pixels x K] * W[Cout x K]^T
// with K = Cin*25 (k = ci*25 + kh*5 + kw) and A the im2col of the zero-padded input. One
// CTA owns a 128-pixel tile (M = 128) of the flattened (sample, h, w) space; its input rows
// are staged once in shared memory as f32, and 4 producer warps (one thread per tile row)
// build 32-deep K chunks of A (im2col gather through a per-CTA offset table) in the
// canonical K-major layout into an NS-stage ring, while each chunk of W — pre-packed in
// that layout by pack_w_kernel — lands by one TMA bulk copy; a 5th warp (one elected
// lane) issues four 128xCOUTx8 MMAs per chunk
// into a TMEM accumulator and commits each stage back to the producers through an
// mbarrier (the issuer must not share a warp with producers that it waits on). The
// epilogue reads the 128xCOUT accumulator with tcgen05.ld, adds the bias, applies relu and
// stores NCHW rows (coalesced over pixels).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "conv_tc.cuh"
#include "ds_common.cuh"

namespace dsb {
namespace {

constexpr int kTile = 128, kKC = 32, kNS = 4;  // pixels per CTA, K per chunk, ring stages

// K order: with CIN % 32 == 0 the channels are innermost (k = (kh*5 + kw)*CIN + ci) and the
// staged input is HWC with a padded channel stride CS, so a 32-deep chunk of one im2col row
// is 8 aligned 16-byte runs (LDS.128 -> STS.128); otherwise (conv1, CIN = 3) the reference
// order k = ci*25 + kh*5 + kw through an offset table. pack_w_kernel packs W to match.
template <int CIN, int COUT, int H>
struct ConvTcShape {
  static constexpr int HW = H * H, HP = H + 4, K = CIN * 25, NKC = (K + kKC - 1) / kKC;
  static constexpr bool kHWC = CIN % kKC == 0;  // a K chunk never straddles two (kh, kw)
  static constexpr int CS = CIN + 4;                          // HWC channel stride (banks)
  static constexpr bool kMulti = HW < kTile;                 // a tile spans several samples
  static constexpr int SPT = kMulti ? kTile / HW : 1;         // samples per tile
  static constexpr int ROWS = kMulti ? HP : kTile / H + 4;    // staged input rows per sample
  static constexpr int XS = kHWC ? SPT * ROWS * HP * CS : SPT * CIN * ROWS * HP;  // staged input floats
  static constexpr int A_BYTES = kTile * kKC * 4, B_BYTES = COUT * kKC * 4;
  static constexpr size_t SMEM = static_cast<size_t>(XS) * 4 + kNS * B_BYTES + NKC * kKC * 4 + 1024;
  // TMEM: accumulator (COUT columns) + the A ring (kNS x 32 columns)
  static constexpr uint32_t TMEM_COLS = COUT + kNS * kKC <= 128 ? 128 : (COUT + kNS * kKC <= 256 ? 256 : 512);
};

template <int CIN, int COUT, int H>
__global__ void __launch_bounds__(kTile + 32, 1) conv5_tc_kernel(const float* __restrict__ in, const float* __restrict__ Wpk,
                                                            const float* __restrict__ bias, float* __restrict__ out,
                                                            uint32_t R, bool relu, const uint32_t* gate) {
  using S = ConvTcShape<CIN, COUT, H>;
  if (gate && *gate) return;
  extern __shared__ __align__(128) unsigned char smem[];
  float* xs = reinterpret_cast<float*>(smem);
  unsigned char* ring = smem + ((static_cast<size_t>(S::XS) * 4 + 127) & ~static_cast<size_t>(127));
  int* koff = reinterpret_cast<int*>(ring + kNS * S::B_BYTES);  // [NKC*32] im2col offsets
  __shared__ __align__(8) uint64_t full[kNS], empty[kNS], done;
  __shared__ uint32_t tmem_base;
  const uint32_t tid = threadIdx.x, warp = tid >> 5;
  const uint64_t total = static_cast<uint64_t>(R) * S::HW;
  const uint64_t g0 = static_cast<uint64_t>(blockIdx.x) * kTile;
  const uint32_t n0 = static_cast<uint32_t>(g0 / S::HW);
  const uint32_t h0 = S::kMulti ? 0 : static_cast<uint32_t>((g0 % S::HW) / H);  // first output row

  constexpr uint32_t kThreads = kTile + 32;
  if (warp == 4) tc::tmem_alloc<S::TMEM_COLS>(&tmem_base);
  if (tid == 0) {
    for (int s = 0; s < kNS; ++s) {
      tc::mbar_init(&full[s], kTile);  // producer arrivals; thread 0 also adds W's tx bytes
      tc::mbar_init(&empty[s], 1);
    }
    tc::mbar_init(&done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  // stage the tile's zero-padded input rows: xs[s][ci][row][col], row r <-> image row
  // h0 - 2 + r (or the whole padded image for multi-sample tiles)
  // one (sample, channel, row) per thread and iteration: a coalesced, vectorised row read
  // all of a thread's line loads are issued before its first shared store (one memory
  // round trip instead of one per line)
  constexpr int kLines = (S::SPT * CIN * S::ROWS + kThreads - 1) / kThreads;
  float4 v[kLines][H / 4];
  auto line = [&](uint32_t i, uint32_t& row, uint32_t& ci, uint32_t& sl) {
    if constexpr (S::kHWC) {  // channel fastest across threads: conflict-free HWC stores
      ci = i % CIN;
      row = (i / CIN) % S::ROWS;
      sl = i / (CIN * S::ROWS);
    } else {
      row = i % S::ROWS;
      ci = (i / S::ROWS) % CIN;
      sl = i / (S::ROWS * CIN);
    }
  };
#pragma unroll
  for (int li = 0; li < kLines; ++li) {
    const uint32_t i = tid + li * kThreads;
    uint32_t row, ci, sl;
    line(i, row, ci, sl);
    const int y = static_cast<int>(h0 + row) - 2;
    const uint32_t n = n0 + sl;
    const bool live = i < static_cast<uint32_t>(S::SPT * CIN * S::ROWS) && n < R && y >= 0 && y < H;
    const float4* src =
        reinterpret_cast<const float4*>(in + ((static_cast<uint64_t>(live ? n : 0) * CIN + ci) * H + (live ? y : 0)) * H);
#pragma unroll
    for (int q = 0; q < H / 4; ++q) v[li][q] = live ? __ldg(src + q) : make_float4(0.f, 0.f, 0.f, 0.f);
  }
#pragma unroll
  for (int li = 0; li < kLines; ++li) {
    const uint32_t i = tid + li * kThreads;
    if (i >= static_cast<uint32_t>(S::SPT * CIN * S::ROWS)) break;
    uint32_t row, ci, sl;
    line(i, row, ci, sl);
    // element col of this (sl, row, ci) line lives at dst[col * step]
    float* dst = S::kHWC ? xs + (static_cast<size_t>(sl) * S::ROWS + row) * S::HP * S::CS + ci
                         : xs + ((static_cast<size_t>(sl) * CIN + ci) * S::ROWS + row) * S::HP;
    constexpr uint32_t step = S::kHWC ? S::CS : 1;
    dst[0] = dst[step] = dst[(H + 2) * step] = dst[(H + 3) * step] = 0.0f;
#pragma unroll
    for (int q = 0; q < H / 4; ++q) {
      dst[(2 + 4 * q) * step] = v[li][q].x;
      dst[(3 + 4 * q) * step] = v[li][q].y;
      dst[(4 + 4 * q) * step] = v[li][q].z;
      dst[(5 + 4 * q) * step] = v[li][q].w;
    }
  }
  for (uint32_t k = tid; k < static_cast<uint32_t>(S::NKC * kKC); k += kThreads) {
    const uint32_t ci = k / 25, r = k - ci * 25, kh = r / 5, kw = r - kh * 5;
    koff[k] = k < static_cast<uint32_t>(S::K) ? static_cast<int>((ci * S::ROWS + kh) * S::HP + kw) : -1;
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base;
  constexpr uint32_t a_lbo = kTile / 8 * 128, b_lbo = COUT / 8 * 128;
  constexpr uint32_t idesc = tc::idesc_tf32(kTile, COUT);
  if (warp == 4) {  // ---- MMA issuer (one lane) ----
    if ((tid & 31) == 0) {
      for (int i = 0; i < S::NKC; ++i) {
        const int s = i % kNS;
        unsigned char* Bs = ring + s * S::B_BYTES;
        const uint32_t ta = tmem + COUT + s * kKC;  // A stage s: TMEM columns
        tc::mbar_wait(&full[s], (i / kNS) & 1);
        tc::fence_after();
#pragma unroll
        for (int t = 0; t < kKC / 8; ++t)
          tc::mma_tf32_ta(tmem, ta + t * 8, tc::saddr(Bs) + t * 2 * b_lbo, b_lbo, idesc, i > 0 || t > 0);
        tc::commit(&empty[s]);
      }
      tc::commit(&done);
    }
    __syncwarp();
  } else {  // ---- producers: this thread's tile row ----
    const uint64_t g = g0 + tid;
    const bool valid = g < total;
    const uint32_t sl = static_cast<uint32_t>((g / S::HW) - n0), p = static_cast<uint32_t>(g % S::HW);
    const uint32_t ph = p / H - h0, pw = p % H;
    const float* xrow = xs + static_cast<size_t>(sl) * CIN * S::ROWS * S::HP + ph * S::HP + pw;
    for (int i = 0; i < S::NKC; ++i) {
      const int s = i % kNS;
      if (i >= kNS) tc::mbar_wait(&empty[s], ((i / kNS) - 1) & 1);
      unsigned char* Bs = ring + s * S::B_BYTES;
      const int k0 = i * kKC;
      if (tid == 0) {  // W chunk i: one bulk copy of the pre-packed block
        asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(tc::saddr(&full[s])), "r"(S::B_BYTES)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                tc::saddr(Bs)),
            "l"(Wpk + static_cast<size_t>(i) * COUT * kKC), "r"(S::B_BYTES), "r"(tc::saddr(&full[s]))
            : "memory");
      }
      // A: this row's 32 K values (im2col) -> TMEM lane tid, the stage's 32 columns
      float av[kKC];
      if constexpr (S::kHWC) {
        const int khw = k0 / CIN, ci0 = k0 - khw * CIN, kh = khw / 5, kw = khw - kh * 5;
        const float4* src = reinterpret_cast<const float4*>(
            xs + ((static_cast<size_t>(sl) * S::ROWS + ph + kh) * S::HP + pw + kw) * S::CS + ci0);
#pragma unroll
        for (int c = 0; c < kKC / 4; ++c) {
          const float4 v = valid ? src[c] : make_float4(0.f, 0.f, 0.f, 0.f);
          av[4 * c] = v.x;
          av[4 * c + 1] = v.y;
          av[4 * c + 2] = v.z;
          av[4 * c + 3] = v.w;
        }
      } else {
#pragma unroll
        for (int j = 0; j < kKC; ++j) {
          const int o = koff[k0 + j];
          av[j] = (valid && o >= 0) ? xrow[o] : 0.0f;
        }
      }
      tc::tmem_st32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + COUT + s * kKC, av);
      tc::fence_before();
      tc::mbar_arrive(&full[s]);
    }
    tc::mbar_wait(&done, 0);
    tc::fence_after();
    // epilogue: row tid of the accumulator -> out[n][co][p]
    float* dst = out + (static_cast<uint64_t>(n0 + sl) * COUT) * S::HW + p;
#pragma unroll
    for (int cb = 0; cb < COUT; cb += 32) {
      float v[32];
      tc::tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + cb, v);
      if (valid) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          float o = v[j] + (bias ? __ldg(bias + cb + j) : 0.0f);
          if (relu) o = o > 0.0f ? o : 0.0f;
          dst[static_cast<uint64_t>(cb + j) * S::HW] = o;
        }
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 4) tc::tmem_free<S::TMEM_COLS>(tmem);
}

// ---- weight (and bias) gradients: D[k' x COUT] = A'[k' x pixels] * dY[COUT x pixels]^T --
// k' in the HWC order (k' = (kh*5 + kw)*CIN + ci), one extra row k' = K of ones so row K of
// D is the bias gradient. A' is the transpose of the forward's im2col, built K-major (one
// thread per k' row gathers 4 pixels per 16-byte unit; MN-major tf32 operands are not
// accepted by the MMA — tools/tc_gemm_test.cu); dY
// rows land by LDGSTS straight into the K-major B layout; a producer arrives on a stage's
// mbarrier one chunk later, after its copies for it completed and a proxy fence (LDGSTS
// writes are generic-proxy data for the tensor core). CTA = (128-row k' tile, a split of
// the batch); the per-split partials
// part[split][K+1][COUT] are summed in split order by wgrad_reduce_kernel.
template <int CIN, int COUT, int H, int SPS>
struct WgradShape {
  static constexpr int HW = H * H, HP = H + 4, CS = CIN + 4, K = CIN * 25, MT = (K + 1 + kTile - 1) / kTile;
  static constexpr bool kHWC = CIN % kKC == 0;  // else CHW staging and the reference k order (conv1)
  static constexpr int XS = kHWC ? HP * HP * CS : CIN * HP * HP, CPS = HW / kKC;  // staged floats, chunks/sample
  static constexpr int B_BYTES = COUT * kKC * 4;
  static constexpr size_t SMEM = static_cast<size_t>(XS) * 4 + kNS * B_BYTES + 1024;
  static constexpr uint32_t TMEM_COLS = COUT + kNS * kKC <= 128 ? 128 : (COUT + kNS * kKC <= 256 ? 256 : 512);
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(tc::saddr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int CIN, int COUT, int H, int SPS>
__global__ void __launch_bounds__(kTile + 32, 1) conv5_wgrad_tc_kernel(const float* __restrict__ in,
                                                                       const float* __restrict__ dout,
                                                                       float* __restrict__ part, uint32_t R,
                                                                       uint32_t sps, const uint32_t* gate) {
  using S = WgradShape<CIN, COUT, H, SPS>;
  static_assert(S::HW % kKC == 0 && COUT % 32 == 0, "wgrad tiling");
  if (gate && *gate) return;
  extern __shared__ __align__(128) unsigned char smem[];
  float* xs = reinterpret_cast<float*>(smem);
  unsigned char* ring = smem + ((static_cast<size_t>(S::XS) * 4 + 127) & ~static_cast<size_t>(127));
  __shared__ __align__(8) uint64_t full[kNS], empty[kNS], done;
  __shared__ uint32_t tmem_base;
  constexpr uint32_t kThreads = kTile + 32;
  const uint32_t tid = threadIdx.x, warp = tid >> 5;
  const uint32_t mt = blockIdx.x, split = blockIdx.y;
  constexpr int kLag = 1;  // chunks of LDGSTS in flight per producer before it hands a stage over
  const uint32_t n_lo = split * sps, n_hi = min(n_lo + sps, R);
  const int nchunks = static_cast<int>(n_hi > n_lo ? (n_hi - n_lo) * S::CPS : 0);
  if (warp == 4) tc::tmem_alloc<S::TMEM_COLS>(&tmem_base);
  if (tid == 0) {
    for (int s = 0; s < kNS; ++s) {
      tc::mbar_init(&full[s], kTile);  // one arrival per producer thread
      tc::mbar_init(&empty[s], 1);
    }
    tc::mbar_init(&done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = tmem_base;
  constexpr uint32_t b_lbo = COUT / 8 * 128;   // between 4-pixel halves (K-major B)
  constexpr uint32_t idesc = tc::idesc_tf32(kTile, COUT);
  if (warp == 4) {  // ---- MMA issuer ----
    if ((tid & 31) == 0) {
      for (int i = 0; i < nchunks; ++i) {
        const int s = i % kNS;
        unsigned char* Bs = ring + s * S::B_BYTES;
        const uint32_t ta = tmem + COUT + s * kKC;  // A' stage s: TMEM columns
        tc::mbar_wait(&full[s], (i / kNS) & 1);
        tc::fence_after();
#pragma unroll
        for (int t = 0; t < kKC / 8; ++t)
          tc::mma_tf32_ta(tmem, ta + t * 8, tc::saddr(Bs) + t * 2 * b_lbo, b_lbo, idesc, i > 0 || t > 0);
        tc::commit(&empty[s]);
      }
      tc::commit(&done);
    }
    __syncwarp();
  } else {  // ---- producers ----
    // this thread's row k' of the tile: (kh, kw, ci), the ones row (bias) or padding
    const uint32_t krow = mt * kTile + tid;
    const bool real = krow < static_cast<uint32_t>(S::K), ones = krow == static_cast<uint32_t>(S::K);
    uint32_t rci = 0, rkh = 0, rkw = 0;
    if (real) {
      if constexpr (S::kHWC) {
        const uint32_t khw = krow / CIN;
        rci = krow - khw * CIN;
        rkh = khw / 5;
        rkw = khw - rkh * 5;
      } else {
        rci = krow / 25;
        const uint32_t r = krow - rci * 25;
        rkh = r / 5;
        rkw = r - rkh * 5;
      }
    }
    for (int i = 0; i < nchunks; ++i) {
      const uint32_t n = n_lo + i / S::CPS, p0 = (i % S::CPS) * kKC;
      if (i % S::CPS == 0) {  // stage sample n as HWC (all producers; the ring holds copies)
        // every global load of the sample is issued before the first shared store (one
        // memory round trip per sample instead of one per (channel, row) line a thread owns)
        constexpr int kLines = (CIN * S::HP + kTile - 1) / kTile;  // lines per thread
        float4 v[kLines][H / 4];
#pragma unroll
        for (int li = 0; li < kLines; ++li) {
          const uint32_t j = tid + li * kTile, ci = j % CIN, row = j / CIN;
          const int y = static_cast<int>(row) - 2;
          const bool live = j < static_cast<uint32_t>(CIN * S::HP) && y >= 0 && y < H;
          const float4* src = reinterpret_cast<const float4*>(in + ((static_cast<uint64_t>(n) * CIN + ci) * H + (live ? y : 0)) * H);
#pragma unroll
          for (int q = 0; q < H / 4; ++q) v[li][q] = live ? __ldg(src + q) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kTile) : "memory");
#pragma unroll
        for (int li = 0; li < kLines; ++li) {
          const uint32_t j = tid + li * kTile;
          if (j >= static_cast<uint32_t>(CIN * S::HP)) break;
          const uint32_t ci = j % CIN, row = j / CIN;
          constexpr uint32_t step = S::kHWC ? S::CS : 1;
          float* dst = S::kHWC ? xs + static_cast<size_t>(row) * S::HP * S::CS + ci
                               : xs + (static_cast<size_t>(ci) * S::HP + row) * S::HP;
          dst[0] = dst[step] = dst[(H + 2) * step] = dst[(H + 3) * step] = 0.0f;
#pragma unroll
          for (int q = 0; q < H / 4; ++q) {
            dst[(2 + 4 * q) * step] = v[li][q].x;
            dst[(3 + 4 * q) * step] = v[li][q].y;
            dst[(4 + 4 * q) * step] = v[li][q].z;
            dst[(5 + 4 * q) * step] = v[li][q].w;
          }
        }
        asm volatile("bar.sync 1, %0;" ::"n"(kTile) : "memory");
      }
      const int s = i % kNS;
      if (i >= kNS) tc::mbar_wait(&empty[s], ((i / kNS) - 1) & 1);
      unsigned char* Bs = ring + s * S::B_BYTES;
      // B: dY[n][co][p0 .. p0+32) -> K-major rows co (LDGSTS, 16 bytes each)
      for (uint32_t t = tid; t < static_cast<uint32_t>(COUT * (kKC / 4)); t += kTile) {
        const uint32_t co = t / (kKC / 4), c = t % (kKC / 4);
        cp_async16(Bs + tc::kmajor_off(co, c * 4, COUT),
                   dout + (static_cast<uint64_t>(n) * COUT + co) * S::HW + p0 + c * 4);
      }
      // A': row k' x 32 pixels (4 per image row segment) -> TMEM lane tid, 32 columns
      float av[kKC];
#pragma unroll
      for (int j = 0; j < kKC / 4; ++j) {
        const uint32_t pj = p0 + 4 * j, h = pj / H, w = pj % H;
        if (real) {
          if constexpr (S::kHWC) {
            const float* b = xs + ((h + rkh) * S::HP + w + rkw) * S::CS + rci;
            av[4 * j] = b[0];
            av[4 * j + 1] = b[S::CS];
            av[4 * j + 2] = b[2 * S::CS];
            av[4 * j + 3] = b[3 * S::CS];
          } else {
            const float* b = xs + (rci * S::HP + h + rkh) * S::HP + w + rkw;
            av[4 * j] = b[0];
            av[4 * j + 1] = b[1];
            av[4 * j + 2] = b[2];
            av[4 * j + 3] = b[3];
          }
        } else {
          const float o = ones ? 1.0f : 0.0f;
          av[4 * j] = av[4 * j + 1] = av[4 * j + 2] = av[4 * j + 3] = o;
        }
      }
      tc::tmem_st32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + COUT + s * kKC, av);
      tc::fence_before();
      cp_async_commit();
      if (i >= kLag) {  // chunk i-kLag: its LDGSTS landed, A' stores done -> hand the stage over
        cp_async_wait<kLag>();
        tc::fence_async_smem();
        tc::mbar_arrive(&full[(i - kLag) % kNS]);
      }
    }
    if (nchunks > 0) {
      cp_async_wait<0>();
      tc::fence_async_smem();
      for (int i = nchunks > kLag ? nchunks - kLag : 0; i < nchunks; ++i) tc::mbar_arrive(&full[i % kNS]);
      tc::mbar_wait(&done, 0);
      tc::fence_after();
    }
    // epilogue: TMEM row tid = k' (tile mt) -> part[split][k'][co]
    const uint32_t kp = mt * kTile + tid;
#pragma unroll
    for (int cb = 0; cb < COUT; cb += 32) {
      float v[32];
      tc::tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + cb, v);
      if (kp <= static_cast<uint32_t>(S::K)) {
        float* dst = part + (static_cast<uint64_t>(split) * (S::K + 1) + kp) * COUT + cb;
#pragma unroll
        for (int j = 0; j < 32; ++j) dst[j] = nchunks > 0 ? v[j] : 0.0f;
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 4) tc::tmem_free<S::TMEM_COLS>(tmem);
}

// grad W[co][ci*25 + kh*5 + kw] and b[co] from part[split][k'][co], splits summed in order
__global__ void wgrad_reduce_kernel(const float* __restrict__ part, uint32_t nsplit, uint32_t cin, uint32_t cout,
                                    bool hwc, float* __restrict__ gW, float* __restrict__ gb, float inv_b,
                                    uint32_t* flags, const uint32_t* gate) {
  if (gate && *gate) return;
  const uint32_t K = cin * 25, t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (K + 1) * cout) return;
  const uint32_t kp = t / cout, co = t % cout;
  float s = 0.0f;
  const uint64_t stride = static_cast<uint64_t>(K + 1) * cout;
  const float* src = part + static_cast<uint64_t>(kp) * cout + co;
  uint32_t sp = 0;
  for (; sp + 8 <= nsplit; sp += 8) {  // loads batched, adds in split order
    float v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = src[(sp + j) * stride];
#pragma unroll
    for (int j = 0; j < 8; ++j) s += v[j];
  }
  for (; sp < nsplit; ++sp) s += src[sp * stride];
  const float g = s * inv_b;
  if (!isfinite(g)) atomicOr(flags, DS_FLAG_GRAD_NONFINITE);
  if (kp == K) {
    gb[co] = g;
  } else if (hwc) {
    const uint32_t khw = kp / cin, ci = kp - khw * cin;
    gW[static_cast<uint64_t>(co) * K + ci * 25 + khw] = g;
  } else {
    gW[static_cast<uint64_t>(co) * K + kp] = g;
  }
}

// Wpk[chunk][canonical K-major COUT x 32] = W[co][chunk*32 + kk] (0 beyond K): each K
// chunk of the weights becomes one contiguous block for a single TMA bulk copy.
// flip: W is the forward weight of the layer whose backward-data this is ([cin][cout][5][5]
// here); the packed operand is its transposed, 180-degree-rotated kernel
// W'[co][ci][kh][kw] = W[ci][co][4-kh][4-kw] (no separate flip pass).
__global__ void pack_w_kernel(const float* __restrict__ W, float* __restrict__ Wpk, uint32_t cout, uint32_t cin,
                              uint32_t nkc, bool hwc, bool flip, const uint32_t* gate) {
  if (gate && *gate) return;
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nkc * cout * kKC) return;
  const uint32_t K = cin * 25;
  const uint32_t chunk = t / (cout * kKC), rem = t % (cout * kKC), co = rem / kKC, kk = rem % kKC;
  const uint32_t k = chunk * kKC + kk;  // GEMM k; the weight's own index below
  float v = 0.0f;
  if (k < K) {
    uint32_t ci, khw;
    if (hwc) {  // k = (kh*5 + kw)*cin + ci
      khw = k / cin;
      ci = k - khw * cin;
    } else {  // k = ci*25 + kh*5 + kw
      ci = k / 25;
      khw = k - ci * 25;
    }
    v = flip ? W[(static_cast<size_t>(ci) * cout + co) * 25 + (24 - khw)] : W[static_cast<size_t>(co) * K + ci * 25 + khw];
  }
  Wpk[static_cast<size_t>(chunk) * cout * kKC + tc::kmajor_off(co, kk, cout) / 4] = v;
}

}  // namespace

template <int CIN, int COUT, int H>
int launch_conv5_tc(const float* in, const float* W, bool flip, float* Wpk, const float* b, float* out, uint32_t R,
                    bool relu, const uint32_t* gate, cudaStream_t s) {
  using S = ConvTcShape<CIN, COUT, H>;
  static_assert(COUT % 32 == 0 && COUT <= 256, "COUT: multiple of 32 (tcgen05 N, TMEM columns)");
  static_assert(H % 4 == 0, "rows are staged as float4");
  auto k = conv5_tc_kernel<CIN, COUT, H>;
  static bool attr = false;
  if (!attr) {
    DS_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(S::SMEM)));
    attr = true;
  }
  const uint64_t tiles = (static_cast<uint64_t>(R) * S::HW + kTile - 1) / kTile;
  const uint32_t n = S::NKC * COUT * kKC;
  pack_w_kernel<<<(n + 255) / 256, 256, 0, s>>>(W, Wpk, COUT, CIN, S::NKC, S::kHWC, flip, gate);
  k<<<static_cast<unsigned>(tiles), kTile + 32, S::SMEM, s>>>(in, Wpk, b, out, R, relu, gate);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

// the convnet's layers: forward (conv1..3) and backward-data (conv3 -> dp2, conv2 -> dr1)
template int launch_conv5_tc<3, 32, 32>(const float*, const float*, bool, float*, const float*, float*,
                                        uint32_t, bool, const uint32_t*, cudaStream_t);
template int launch_conv5_tc<32, 32, 16>(const float*, const float*, bool, float*, const float*, float*,
                                        uint32_t, bool, const uint32_t*, cudaStream_t);
template int launch_conv5_tc<32, 64, 8>(const float*, const float*, bool, float*, const float*, float*,
                                        uint32_t, bool, const uint32_t*, cudaStream_t);
template int launch_conv5_tc<64, 32, 8>(const float*, const float*, bool, float*, const float*, float*,
                                        uint32_t, bool, const uint32_t*, cudaStream_t);


// many splits (conv1: one per sample): a warp per output, lanes over the splits, fixed tree
__global__ void wgrad_reduce_warp_kernel(const float* __restrict__ part, uint32_t nsplit, uint32_t cin, uint32_t cout,
                                         bool hwc, float* __restrict__ gW, float* __restrict__ gb, float inv_b,
                                         uint32_t* flags, const uint32_t* gate) {
  if (gate && *gate) return;
  const uint32_t K = cin * 25, w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= (K + 1) * cout) return;
  const uint32_t kp = w / cout, co = w % cout;
  const uint64_t stride = static_cast<uint64_t>(K + 1) * cout;
  float s = 0.0f;
  for (uint32_t sp = lane; sp < nsplit; sp += 32) s += part[sp * stride + static_cast<uint64_t>(kp) * cout + co];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane != 0) return;
  const float g = s * inv_b;
  if (!isfinite(g)) atomicOr(flags, DS_FLAG_GRAD_NONFINITE);
  if (kp == K) {
    gb[co] = g;
  } else if (hwc) {
    const uint32_t khw = kp / cin, ci = kp - khw * cin;
    gW[static_cast<uint64_t>(co) * K + ci * 25 + khw] = g;
  } else {
    gW[static_cast<uint64_t>(co) * K + kp] = g;
  }
}

template <int CIN, int COUT, int H, int SPS>
int launch_conv5_wgrad_tc(const float* in, const float* dout, float* part, float* gW, float* gb, uint32_t R,
                          float inv_b, uint32_t* flags, const uint32_t* gate, cudaStream_t s) {
  using S = WgradShape<CIN, COUT, H, SPS>;
  auto k = conv5_wgrad_tc_kernel<CIN, COUT, H, SPS>;
  static bool attr = false;
  if (!attr) {
    DS_CUDA_TRY(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(S::SMEM)));
    attr = true;
  }
  // samples per split: as few as fill ONE wave of CTAs (S::MT x nsplit <= 148; conv2's 7 x 25
  // = 175 CTAs ran a second wave for 27 of them), never fewer than SPS (the partials buffer
  // holds ceil(R / SPS) splits)
  int nsm = 148, dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const uint32_t per_wave = std::max<uint32_t>(1, static_cast<uint32_t>(nsm) / S::MT);
  const uint32_t sps = std::max<uint32_t>(SPS, (R + per_wave - 1) / per_wave);
  const uint32_t nsplit = (R + sps - 1) / sps;
  k<<<dim3(S::MT, nsplit), kTile + 32, S::SMEM, s>>>(in, dout, part, R, sps, gate);
  const uint32_t n = (S::K + 1) * COUT;
  if (nsplit >= 32)
    wgrad_reduce_warp_kernel<<<(n * 32 + 255) / 256, 256, 0, s>>>(part, nsplit, CIN, COUT, S::kHWC, gW, gb, inv_b, flags,
                                                                   gate);
  else
    wgrad_reduce_kernel<<<(n + 255) / 256, 256, 0, s>>>(part, nsplit, CIN, COUT, S::kHWC, gW, gb, inv_b, flags, gate);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

template int launch_conv5_wgrad_tc<3, 32, 32, 1>(const float*, const float*, float*, float*, float*, uint32_t, float,
                                                  uint32_t*, const uint32_t*, cudaStream_t);
template int launch_conv5_wgrad_tc<32, 32, 16, 4>(const float*, const float*, float*, float*, float*, uint32_t, float,
                                                   uint32_t*, const uint32_t*, cudaStream_t);
template int launch_conv5_wgrad_tc<32, 64, 8, 4>(const float*, const float*, float*, float*, float*, uint32_t, float,
                                                  uint32_t*, const uint32_t*, cudaStream_t);

}  // namespace dsb
