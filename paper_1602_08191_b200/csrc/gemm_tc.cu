// gemm_tc.cu — the dense contraction of the AlexNet-shaped convnet (BASELINE config 4):
// D[M x N] = epilogue( A[M x K] . B[N x K]^T ), f32 operands in HBM, tf32 tcgen05 MMA,
// f32 accumulation in TMEM.
//
// Pipeline (one output tile per CTA, 256 threads, warp-specialised):
//   warp 0: TMA producer. Two 2-D tensor maps (SWIZZLE_128B, 32 f32 = 128 B inner box)
//           stream [128 x 32] A and [BN x 32] B k-slices into a kStages-deep smem ring
//           (full/empty mbarriers). Tails beyond M, N, K are zero-filled by TMA.
//   warp 1: one elected lane issues 4 tcgen05.mma kind::tf32 (K = 8 each) per stage and
//           frees the stage with tcgen05.commit; after the last stage commits the
//           accumulator-full barrier.
//   warps 4-7: epilogue. Each warp reads its TMEM lane quadrant (32 rows) 32 columns at a
//           time (tcgen05.ld 32x32b.x32) and applies scale, bias and ReLU, then stores
//           row-major D with leading dimension ldd. With split-K (gridDim.z > 1) each
//           split stores raw partials to its own slab, and gemm_reduce_kernel sums the
//           slabs in split order (deterministic) before the epilogue.
// Grid: (ceil(N/BN), ceil(M/128), splits). N is the fastest index, so CTAs that are
// adjacent in launch order reuse the same A tile from L2.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>

#include "conv_tc.cuh"
#include "ds_common.cuh"
#include "gemm_tc.cuh"

namespace dsb {
namespace {

// 8 warps: 0 TMA producer, 1 MMA issuer, 2-3 idle, 4-7 epilogue. A multiple of 4 warps
// keeps CTA-relative warp % 4 equal to the SM sub-partition when two CTAs share an SM, so
// each epilogue warp reads its own TMEM lane quadrant.
constexpr int kBM = 128, kBK = 32, kThreads = 256;

template <int BN>
struct GemmSmem {
  static constexpr uint32_t A_BYTES = kBM * kBK * 4;  // 16 KB
  static constexpr uint32_t B_BYTES = BN * kBK * 4;
  static constexpr uint32_t STAGE = A_BYTES + B_BYTES;
  // ~100 KB so two CTAs share an SM: one's epilogue and prologue overlap the other's
  // mainloop (measured better than one CTA with a deep ring for every tile width; the
  // 256-wide tile then has 2 stages of 48 KB)
#ifndef DS_GEMM_SMEM_SMALL
#define DS_GEMM_SMEM_SMALL (100 * 1024)
#endif
#ifndef DS_GEMM_TWO_CTA_MAX_BN
#define DS_GEMM_TWO_CTA_MAX_BN 256
#endif
  // up to 128 wide: two (three up to 64) persistent CTAs per SM; 192 / 240 / 256 wide: one
  // CTA with a deep ring, two accumulator buffers and eight epilogue warps (two CTAs with one
  // buffer each, or one CTA with four epilogue warps, were slower: the epilogue of these
  // tiles is as long as a short-K mainloop)
  static constexpr bool TWO_CTA = BN <= DS_GEMM_TWO_CTA_MAX_BN && BN <= 128;
  static constexpr int THREADS = BN <= 128 ? 256 : 384;  // warps 4.. are the epilogue
  static constexpr int EPI_WARPS = THREADS / 32 - 4;
#ifndef DS_GEMM_THREE_CTA_MAX_BN
#define DS_GEMM_THREE_CTA_MAX_BN 64
#endif
  // CTAs per SM: three for tiles up to 64 wide (70 KB each: more stages in flight per SM for
  // the operand-heavy narrow tiles; measured +2.5% on the AlexNet step), else two / one
  static constexpr int CTAS = BN <= DS_GEMM_THREE_CTA_MAX_BN ? 3 : (TWO_CTA ? 2 : 1);
  static constexpr uint32_t BUDGET = CTAS == 3 ? 70 * 1024 : (TWO_CTA ? DS_GEMM_SMEM_SMALL : 200 * 1024);
  static constexpr int STAGES = BUDGET / STAGE > 8 ? 8 : BUDGET / STAGE;
  static constexpr uint32_t TOTAL = STAGES * STAGE + 1024 /*align*/ + 256 /*barriers*/;
  static constexpr uint32_t TMEM_COLS = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;  // power of 2
  // accumulator buffers per CTA: two (the epilogue of tile j overlaps the MMAs of tile j + 1)
  // when every co-resident CTA's pair fits in the 512 TMEM columns, else one (192 / 256-wide
  // tiles: two CTAs per SM overlap each other's epilogues instead — measured faster than one
  // CTA per SM with two buffers, whose four epilogue warps could not keep up)
  static constexpr uint32_t NBUF = CTAS * 2 * TMEM_COLS <= 512 ? 2 : 1;
};

// SWIZZLE_128B K-major descriptor: 8-row x 128 B atoms, atoms 1024 B apart (SBO); the
// k-offset inside the atom is added to the start address (LBO unused for this layout).
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t addr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((addr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>(1) << 16;            // LBO (ignored for swizzled K-major)
  d |= static_cast<uint64_t>(1024 >> 4) << 32;    // SBO
  d |= 1ull << 46;                                // version
  d |= 2ull << 61;                                // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          tc::saddr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(tc::saddr(bar))
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
          tc::saddr(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(z), "r"(tc::saddr(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc::saddr(b)), "r"(bytes) : "memory");
}

// Output row of accumulator row `row` under the epilogue's row map; -1 for a border row.
__device__ __forceinline__ int64_t map_row(const GemmEpilogue& ep, uint32_t row) {
  if (ep.map_Hp == 0) return row;
  const uint32_t hp2 = ep.map_Hp * ep.map_Hp;
  const uint32_t img = row / hp2, pix = row - img * hp2;
  const uint32_t yp = pix / ep.map_Hp, xp = pix - yp * ep.map_Hp;
  if (yp < ep.map_pad || xp < ep.map_pad || yp >= ep.map_pad + ep.map_H || xp >= ep.map_pad + ep.map_H) return -1;
  if (ep.map_out_padded) return row;
  return (static_cast<int64_t>(img) * ep.map_H + (yp - ep.map_pad)) * ep.map_H + (xp - ep.map_pad);
}

// One output tile's coordinates and k-loop (blockIdx of the one-tile-per-CTA grid).
struct TileJob {
  uint32_t n0, m0, z, split, t0, ntg, nvalid, stage_tx, nk, nkt, k_begin;
  int tap;
};
template <int BN>
__device__ __forceinline__ TileJob tile_job(uint32_t T, uint32_t gx, uint32_t gy, const GemmTaps& tp, uint32_t N,
                                            uint32_t K, uint32_t k_per_split, uint32_t splits) {
  using S = GemmSmem<BN>;
  TileJob j;
  const uint32_t bx = T % gx, rest = T / gx, by = rest % gy;
  j.z = rest / gy;
  j.n0 = bx * BN;
  j.m0 = by * kBM;
  const bool acc_taps = tp.n > 0 && !tp.per_z;
  j.tap = (tp.n > 0 && tp.per_z) ? static_cast<int>(j.z / splits) : -1;  // tap group
  j.split = j.tap >= 0 ? j.z % splits : j.z;
  // per_z with tpc > 1: taps tap*tpc .. + ntg - 1 share the A tile; their B tiles (n_tap rows
  // each) are stacked along N in one BN-wide stage and one MMA covers them all
  j.t0 = j.tap >= 0 ? static_cast<uint32_t>(j.tap) * tp.tpc : 0;
  j.ntg = j.tap >= 0 ? min(tp.tpc, static_cast<uint32_t>(tp.n) - j.t0) : 1;
  j.nvalid = (j.tap >= 0 && tp.tpc > 1) ? j.ntg * tp.n_tap : N;
  j.stage_tx = (j.tap >= 0 && tp.tpc > 1) ? S::A_BYTES + j.ntg * tp.n_tap * kBK * 4 : S::STAGE;
  j.nkt = 1;
  j.k_begin = 0;
  if (acc_taps) {
    j.nkt = (tp.kt + kBK - 1) / kBK;
    j.nk = tp.n * j.nkt;
  } else {
    j.k_begin = j.split * k_per_split;
    const uint32_t k_end = min(K, j.k_begin + k_per_split);
    j.nk = (k_end > j.k_begin) ? (k_end - j.k_begin + kBK - 1) / kBK : 0;
  }
  return j;
}

// Persistent: gridDim.x CTAs walk the tiles T = blockIdx.x, + gridDim.x, ... of the logical
// (gx, gy, gz) grid (x fastest, so concurrently running CTAs share A tiles in L2). The TMA
// ring runs on across tiles, and the accumulator is double-buffered in TMEM where it fits
// (NBUF): the MMA warp fills buffer j % NBUF for tile j while the epilogue warps drain the
// previous tile from the other.
template <int BN>
__global__ void __launch_bounds__(GemmSmem<BN>::THREADS, GemmSmem<BN>::CTAS)
    gemm_tf32_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ GemmEpilogue ep, const __grid_constant__ GemmTaps tp, uint32_t M,
                     uint32_t N, uint32_t K, uint32_t k_per_split, uint32_t splits, uint32_t gx, uint32_t gy,
                     uint32_t ntiles) {
  using S = GemmSmem<BN>;
  constexpr int kStages = S::STAGES;
  constexpr uint32_t kAcc = S::TMEM_COLS;  // columns per accumulator buffer
  constexpr uint32_t kNB = S::NBUF;
  if (ep.gate && *ep.gate) return;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kStages * S::STAGE);
  uint64_t* empty = full + kStages;
  uint64_t* acc_full = empty + kStages;  // [2]
  uint64_t* acc_empty = acc_full + 2;    // [2], one arrival per epilogue warp
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const bool acc_taps = tp.n > 0 && !tp.per_z;
  const uint32_t gz_total = ntiles / (gx * gy);

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    for (int s = 0; s < kStages; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&acc_full[b], 1);
      tc::mbar_init(&acc_empty[b], S::EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) tc::tmem_alloc<kNB * kAcc>(tmem_slot);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer; the ring index i runs on across tiles
      uint32_t i = 0;
      for (uint32_t T = blockIdx.x; T < ntiles; T += gridDim.x) {
        const TileJob j = tile_job<BN>(T, gx, gy, tp, N, K, k_per_split, splits);
        for (uint32_t kk = 0; kk < j.nk; ++kk, ++i) {
          const int s = i % kStages;
          if (i >= kStages) tc::mbar_wait(&empty[s], ((i / kStages) - 1) & 1);
          uint8_t* sa = smem + s * S::STAGE;
          mbar_expect_tx(&full[s], j.stage_tx);
          int ax, ay, bx, by;
          if (acc_taps) {
            const uint32_t t = kk / j.nkt, kc = kk - t * j.nkt;
            ax = tp.a_col[t] + static_cast<int>(kc * kBK);
            ay = static_cast<int>(j.m0) + tp.a_row[t];
            bx = tp.b_col[t] + static_cast<int>(kc * kBK);
            by = static_cast<int>(j.n0) + tp.b_row[t];
          } else {
            ax = bx = static_cast<int>(j.k_begin + kk * kBK);
            ay = static_cast<int>(j.m0);
            by = static_cast<int>(j.n0);
            if (j.tap >= 0) {
              ax += tp.a_col[j.t0], ay += tp.a_row[j.t0];
              if (tp.tpc > 1) {  // one B sub-tile per tap of the group
                for (uint32_t g = 1; g < j.ntg; ++g)
                  tma_load_2d(sa + S::A_BYTES + g * tp.n_tap * kBK * 4, &tmB, &full[s], bx + tp.b_col[j.t0 + g],
                              by + tp.b_row[j.t0 + g]);
              }
              bx += tp.b_col[j.t0], by += tp.b_row[j.t0];
            }
          }
          tma_load_2d(sa, &tmA, &full[s], ax, ay);
          tma_load_2d(sa + S::A_BYTES, &tmB, &full[s], bx, by);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      constexpr uint32_t idesc = tc::idesc_tf32(kBM, BN);
      uint32_t i = 0, jt = 0;
      for (uint32_t T = blockIdx.x; T < ntiles; T += gridDim.x, ++jt) {
        const TileJob j = tile_job<BN>(T, gx, gy, tp, N, K, k_per_split, splits);
        const uint32_t ab = jt % kNB;
        if (jt >= kNB) tc::mbar_wait(&acc_empty[ab], ((jt / kNB) - 1) & 1);  // tile jt - kNB drained
        tc::fence_after();
        const uint32_t acc_t = tmem + ab * kAcc;
        for (uint32_t kk = 0; kk < j.nk; ++kk, ++i) {
          const int s = i % kStages;
          uint32_t nsub = kBK / 8;
          if (acc_taps) {  // a tap's last chunk may be partial (kt multiple of 8)
            const uint32_t rem = tp.kt - (kk % j.nkt) * kBK;
            nsub = rem >= kBK ? kBK / 8 : rem / 8;
          }
          tc::mbar_wait(&full[s], (i / kStages) & 1);
          tc::fence_after();
          const uint32_t a = tc::saddr(smem + s * S::STAGE), b = a + S::A_BYTES;
          for (uint32_t q = 0; q < nsub; ++q) {
            const uint64_t da = sdesc_sw128(a + q * 32), db = sdesc_sw128(b + q * 32);
            const uint32_t acc = (kk | q) ? 1u : 0u;
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(acc_t),
                "l"(da), "l"(db), "r"(idesc), "r"(acc));
          }
          tc::commit(&empty[s]);
        }
        tc::commit(&acc_full[ab]);  // (a tile without k-steps: arrives once earlier MMAs are done)
      }
    }
  } else if (warp >= 4) {  // epilogue warps: TMEM lane quadrant = warp % 4; with eight, column halves
    const int q = warp & 3;
    constexpr int kHalf = (BN / 2 + 31) / 32 * 32;
    const int c_beg = S::EPI_WARPS == 8 && warp >= 8 ? kHalf : 0;
    const int c_end = S::EPI_WARPS == 8 && warp < 8 ? kHalf : BN;
    uint32_t jt = 0;
    for (uint32_t T = blockIdx.x; T < ntiles; T += gridDim.x, ++jt) {
      const TileJob j = tile_job<BN>(T, gx, gy, tp, N, K, k_per_split, splits);
      const uint32_t ab = jt % kNB;
      tc::mbar_wait(&acc_full[ab], (jt / kNB) & 1);
      tc::fence_after();
      const uint32_t acc_t = tmem + ab * kAcc;
      const uint32_t row = j.m0 + q * 32 + lane;
      const bool raw = ep.raw || (j.tap < 0 && gz_total > 1) || (j.tap >= 0 && splits > 1);
      float* out = raw ? ep.D + static_cast<uint64_t>(j.z) * ep.split_stride
                       : ep.D + (j.tap >= 0 ? static_cast<uint64_t>(j.t0) * tp.d_col_step : 0);
      const int64_t orow = row < M ? (raw ? static_cast<int64_t>(row) : map_row(ep, row)) : -1;
      const uint64_t ldo = raw ? N : ep.ldd;
      const float bm = (!raw && ep.bias_m && orow >= 0) ? ep.bias_m[row] : 0.f;
      const uint32_t n0 = j.n0, nvalid = j.nvalid;
#pragma unroll 1
      for (int c = c_beg; c < c_end; c += 32) {
        float v[32];
        if (j.nk > 0) {
          tc::tmem_ld32(acc_t + (static_cast<uint32_t>(q * 32) << 16) + c, v);
        } else {
#pragma unroll
          for (int x = 0; x < 32; ++x) v[x] = 0.f;
        }
        if (orow < 0 || n0 + c >= nvalid) continue;
        float* dst = out + static_cast<uint64_t>(orow) * ldo + n0 + c;
        // BN = 48: last chunk 16 wide; 240: the second half's last chunk 16 wide
        const uint32_t lim = min(min(32u, static_cast<uint32_t>(c_end - c)), nvalid - (n0 + c));
        if (!raw) {
          const float* mrow = ep.mask ? ep.mask + static_cast<uint64_t>(orow) * ep.ldm + n0 + c : nullptr;
          float mk[32];  // the ReLU mask row (data gradient), 16-byte loads when aligned
          if (mrow) {
            if (lim == 32 && (reinterpret_cast<uintptr_t>(mrow) & 15) == 0) {
#pragma unroll
              for (int x = 0; x < 32; x += 4) {
                const float4 m4 = __ldg(reinterpret_cast<const float4*>(mrow + x));
                mk[x] = m4.x, mk[x + 1] = m4.y, mk[x + 2] = m4.z, mk[x + 3] = m4.w;
              }
            } else {
#pragma unroll
              for (int x = 0; x < 32; ++x) mk[x] = static_cast<uint32_t>(x) < lim ? mrow[x] : 1.f;
            }
          }
#pragma unroll
          for (int x = 0; x < 32; ++x) {
            float y = v[x] * ep.scale + bm;
            if (static_cast<uint32_t>(x) < lim) {
              if (ep.bias_n) y += __ldg(ep.bias_n + n0 + c + x);
              if (mrow && !(mk[x] > 0.f)) y = 0.f;
            }
            v[x] = ep.relu ? fmaxf(y, 0.f) : y;
          }
        }
        if (lim == 32 && (ldo % 4) == 0 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
#pragma unroll
          for (int x = 0; x < 32; x += 4) *reinterpret_cast<float4*>(dst + x) = make_float4(v[x], v[x + 1], v[x + 2], v[x + 3]);
        } else {
#pragma unroll
          for (int x = 0; x < 32; ++x)
            if (static_cast<uint32_t>(x) < lim) dst[x] = v[x];
        }
      }
      tc::fence_before();  // this warp's TMEM reads of the buffer are complete
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&acc_empty[ab]);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_free<kNB * kAcc>(tmem);
}

// Halo variant of the accumulating taps mode (conv forward / data gradient; opt-in, see
// halo_enabled), usable when the taps' A row shifts span <= 128 rows: per 32-channel chunk
// the CTA loads the A rows [m0 + lo, m0 + 128 + hi) ONCE and every tap's MMA reads its
// 128-row window inside that buffer; only the B tiles stream per tap. Layout
// (DS_HALO_SW128): 128-byte swizzled rows (a window starts 128 * shift bytes in), or the
// canonical no-swizzle K-major layout [8 k-chunks][rows][16 B] (3-D TMA box), in which
// consecutive rows are 16 bytes apart.
// A traffic per chunk drops from taps x 16 KB to halo_rows x 128 B.
#ifndef DS_HALO_SW128
#define DS_HALO_SW128 1   // 128-byte swizzled halo rows; the start may sit anywhere in the 8-row atom (base offset 0)
#endif
#ifndef DS_HALO_BASEOFF
#define DS_HALO_BASEOFF 0
#endif
constexpr uint32_t kHaloBytes = 256 * 128;
template <int BN>
struct HaloSmem {
  static constexpr uint32_t B_BYTES = BN * kBK * 4;
  static constexpr int STAGES = (48 * 1024) / B_BYTES > 8 ? 8 : ((48 * 1024) / B_BYTES < 2 ? 2 : (48 * 1024) / B_BYTES);
  static constexpr uint32_t TOTAL = 2 * kHaloBytes + STAGES * B_BYTES + 1024 + 512;
};

template <int BN>
__global__ void __launch_bounds__(kThreads, HaloSmem<BN>::TOTAL <= 113 * 1024 ? 2 : 1)
    gemm_halo_kernel(const __grid_constant__ CUtensorMap tmA3, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ GemmEpilogue ep, const __grid_constant__ GemmTaps tp, uint32_t M,
                     uint32_t N) {
  using S = HaloSmem<BN>;
  using T = GemmSmem<BN>;
  constexpr int kB = S::STAGES;
  if (ep.gate && *ep.gate) return;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* halo = smem;                  // [2][kHaloBytes]
  uint8_t* bst = smem + 2 * kHaloBytes;  // [kB][B_BYTES]
  uint64_t* hfull = reinterpret_cast<uint64_t*>(bst + kB * S::B_BYTES);
  uint64_t* hempty = hfull + 2;
  uint64_t* bfull = hempty + 2;
  uint64_t* bempty = bfull + kB;
  uint64_t* acc_full = bempty + kB;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t n0 = blockIdx.x * BN, m0 = blockIdx.y * kBM;
  const uint32_t nkc = (tp.kt + kBK - 1) / kBK, ntap = static_cast<uint32_t>(tp.n);
  const uint32_t hrows = tp.halo_rows, lbo = hrows * 16;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmA3)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmB)) : "memory");
    for (int i = 0; i < 2; ++i) tc::mbar_init(&hfull[i], 1), tc::mbar_init(&hempty[i], 1);
    for (int i = 0; i < kB; ++i) tc::mbar_init(&bfull[i], 1), tc::mbar_init(&bempty[i], 1);
    tc::mbar_init(acc_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) tc::tmem_alloc<T::TMEM_COLS>(tmem_slot);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // TMA producer: the chunk's halo, then its B tile per tap
      uint32_t bi = 0;
      for (uint32_t kc = 0; kc < nkc; ++kc) {
        const uint32_t h = kc & 1;
        if (kc >= 2) tc::mbar_wait(&hempty[h], ((kc >> 1) - 1) & 1);
        mbar_expect_tx(&hfull[h], hrows * 128);
#if DS_HALO_SW128
        tma_load_2d(halo + h * kHaloBytes, &tmA3, &hfull[h], tp.a_col[0] + static_cast<int>(kc * kBK),
                    static_cast<int>(m0) + tp.halo_lo);
#else
        tma_load_3d(halo + h * kHaloBytes, &tmA3, &hfull[h], 0, static_cast<int>(m0) + tp.halo_lo,
                    tp.a_col[0] / 4 + static_cast<int>(kc * 8));
#endif
        for (uint32_t t = 0; t < ntap; ++t, ++bi) {
          const uint32_t s = bi % kB;
          if (bi >= kB) tc::mbar_wait(&bempty[s], ((bi / kB) - 1) & 1);
          mbar_expect_tx(&bfull[s], S::B_BYTES);
          tma_load_2d(bst + s * S::B_BYTES, &tmB, &bfull[s], tp.b_col[t] + static_cast<int>(kc * kBK),
                      static_cast<int>(n0) + tp.b_row[t]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      constexpr uint32_t idesc = tc::idesc_tf32(kBM, BN);
      uint32_t bi = 0;
      for (uint32_t kc = 0; kc < nkc; ++kc) {
        const uint32_t h = kc & 1;
        const uint32_t rem = tp.kt - kc * kBK, nsub = rem >= kBK ? kBK / 8 : rem / 8;
        tc::mbar_wait(&hfull[h], (kc >> 1) & 1);
        tc::fence_after();
        const uint32_t abase = tc::saddr(halo + h * kHaloBytes);
        for (uint32_t t = 0; t < ntap; ++t, ++bi) {
          const uint32_t s = bi % kB;
          tc::mbar_wait(&bfull[s], (bi / kB) & 1);
          tc::fence_after();
#if DS_HALO_SW128
          // 128-byte swizzled rows: a tap's window starts whole rows into the halo
          const uint32_t a = abase + static_cast<uint32_t>(tp.a_row[t]) * 128, b = tc::saddr(bst + s * S::B_BYTES);
#else
          const uint32_t a = abase + static_cast<uint32_t>(tp.a_row[t]) * 16, b = tc::saddr(bst + s * S::B_BYTES);
#endif
          for (uint32_t kk = 0; kk < nsub; ++kk) {
#if DS_HALO_SW128
            uint64_t da = sdesc_sw128(a + kk * 32);
#if DS_HALO_BASEOFF == 1
            da |= static_cast<uint64_t>(((a + kk * 32) >> 7) & 7) << 49;
#elif DS_HALO_BASEOFF == 2
            da |= static_cast<uint64_t>((8 - (((a + kk * 32) >> 7) & 7)) & 7) << 49;
#endif
            const uint64_t db = sdesc_sw128(b + kk * 32);
#else
            const uint64_t da = tc::sdesc(a + kk * 2 * lbo, lbo, 128), db = sdesc_sw128(b + kk * 32);
#endif
            const uint32_t acc = (kc | t | kk) ? 1u : 0u;
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                "l"(da), "l"(db), "r"(idesc), "r"(acc));
          }
          tc::commit(&bempty[s]);
        }
        tc::commit(&hempty[h]);
      }
      tc::commit(acc_full);
    }
  } else if (warp >= 4) {  // epilogue warps 4..7
    const int q = warp & 3;
    const uint32_t row = m0 + q * 32 + lane;
    tc::mbar_wait(acc_full, 0);
    tc::fence_after();
    const bool raw = ep.raw;
    float* out = raw ? ep.D + static_cast<uint64_t>(blockIdx.z) * ep.split_stride : ep.D;
    const int64_t orow = row < M ? (raw ? static_cast<int64_t>(row) : map_row(ep, row)) : -1;
    const uint64_t ldo = raw ? N : ep.ldd;
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      float v[32];
      tc::tmem_ld32(tmem + (static_cast<uint32_t>(q * 32) << 16) + c, v);
      if (orow < 0 || n0 + c >= N) continue;
      float* dst = out + static_cast<uint64_t>(orow) * ldo + n0 + c;
      const uint32_t lim = min(min(32u, static_cast<uint32_t>(BN - c)), N - (n0 + c));
      if (!raw) {
        const float* mrow = ep.mask ? ep.mask + static_cast<uint64_t>(orow) * ep.ldm + n0 + c : nullptr;
        const float bm = ep.bias_m ? ep.bias_m[row] : 0.f;
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          float x = v[j] * ep.scale + bm;
          if (static_cast<uint32_t>(j) < lim) {
            if (ep.bias_n) x += __ldg(ep.bias_n + n0 + c + j);
            if (mrow && !(mrow[j] > 0.f)) x = 0.f;
          }
          v[j] = ep.relu ? fmaxf(x, 0.f) : x;
        }
      }
      if (lim == 32 && (ldo % 4) == 0 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
#pragma unroll
        for (int j = 0; j < 32; j += 4) *reinterpret_cast<float4*>(dst + j) = make_float4(v[j], v[j + 1], v[j + 2], v[j + 3]);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (static_cast<uint32_t>(j) < lim) dst[j] = v[j];
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_free<T::TMEM_COLS>(tmem);
}

// Sum of raw slabs in a fixed order, then the epilogue (row map, tap columns, scale,
// biases, mask, ReLU). Slab (tap t, part p) starts at t * tap_stride + p * part_stride and
// is dense [M][N].
__global__ void gemm_reduce_kernel(const float* __restrict__ slabs, uint32_t ntaps, uint64_t tap_stride,
                                   uint32_t nparts, uint64_t part_stride, uint32_t d_col_step, GemmEpilogue ep,
                                   uint32_t M, uint32_t N, uint32_t col_limit) {
  if (ep.gate && *ep.gate) return;
  const uint64_t total = static_cast<uint64_t>(ntaps) * M * N;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t mn = static_cast<uint64_t>(M) * N;
    const uint32_t t = static_cast<uint32_t>(i / mn);
    const uint64_t e = i - t * mn;
    const uint32_t r = static_cast<uint32_t>(e / N), c = static_cast<uint32_t>(e % N);
    const int64_t orow = map_row(ep, r);
    if (orow < 0 || static_cast<uint64_t>(t) * d_col_step + c >= col_limit) continue;
    float s = 0.f;
    for (uint32_t p = 0; p < nparts; ++p) s += slabs[t * tap_stride + p * part_stride + e];
    float x = s * ep.scale;
    if (ep.bias_m) x += ep.bias_m[r];
    if (ep.bias_n) x += ep.bias_n[c];
    if (ep.mask && !(ep.mask[static_cast<uint64_t>(orow) * ep.ldm + c] > 0.f)) x = 0.f;
    ep.D[static_cast<uint64_t>(orow) * ep.ldd + static_cast<uint64_t>(t) * d_col_step + c] = ep.relu ? fmaxf(x, 0.f) : x;
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q{};
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// row-major [rows x cols] f32 with leading dimension ld, box [box_rows x 32]
int make_map(CUtensorMap* m, const float* base, uint64_t rows, uint64_t cols, uint64_t ld, uint32_t box_rows) {
  auto fn = encode_fn();
  if (!fn) return set_error(DS_E_CUDA, "gemm: cuTensorMapEncodeTiled unavailable");
  if ((ld * 4) % 16 != 0 || (reinterpret_cast<uintptr_t>(base) & 15) != 0)
    return set_error(DS_E_CONTRACT, "gemm: operands need 16-byte aligned rows (ld %% 4 == 0)");
  const cuuint64_t dims[2] = {cols, rows};
  const cuuint64_t strides[1] = {ld * 4};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(kBK), box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(DS_E_CUDA, "gemm: cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
  return DS_OK;
}

// A as [rows][cols/4 chunks][4] viewed 3-D {4, rows, cols/4}: the no-swizzle K-major halo box
int make_map_halo(CUtensorMap* m, const GemmOperand& A, uint32_t box_rows) {
  auto fn = encode_fn();
  if (!fn) return set_error(DS_E_CUDA, "gemm: cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[3] = {4, A.rows, A.cols / 4};
  const cuuint64_t strides[2] = {A.ld * 4, 16};
  const cuuint32_t box[3] = {4, box_rows, 8};
  const cuuint32_t estr[3] = {1, 1, 1};
  const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(A.p), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(DS_E_CUDA, "gemm: halo tensor map failed (%d)", static_cast<int>(r));
  return DS_OK;
}

template <int BN>
int launch_halo(const GemmOperand& A, const GemmOperand& B, const GemmEpilogue& ep, const GemmTaps& tp, uint32_t M,
                uint32_t N, cudaStream_t s) {
  CUtensorMap ma, mb;
#if DS_HALO_SW128
  DS_TRY(make_map(&ma, A.p, A.rows, A.cols, A.ld, tp.halo_rows));
#else
  DS_TRY(make_map_halo(&ma, A, tp.halo_rows));
#endif
  DS_TRY(make_map(&mb, B.p, B.rows, B.cols, B.ld, BN));
  static uint64_t attr_set = 0;  // per device
  int dev = 0;
  DS_CUDA_TRY(cudaGetDevice(&dev));
  if (!(attr_set >> (dev & 63) & 1)) {
    DS_CUDA_TRY(cudaFuncSetAttribute(gemm_halo_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     HaloSmem<BN>::TOTAL));
    attr_set |= 1ull << (dev & 63);
  }
  dim3 grid((N + BN - 1) / BN, (M + kBM - 1) / kBM, 1);
  gemm_halo_kernel<BN><<<grid, kThreads, HaloSmem<BN>::TOTAL, s>>>(ma, mb, ep, tp, M, N);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

template <int BN>
int launch_bn(const GemmOperand& A, const GemmOperand& B, const GemmEpilogue& ep, const GemmTaps& tp, uint32_t M,
              uint32_t N, uint32_t K, uint32_t splits, cudaStream_t s) {
  CUtensorMap ma, mb;
  DS_TRY(make_map(&ma, A.p, A.rows, A.cols, A.ld, kBM));
  DS_TRY(make_map(&mb, B.p, B.rows, B.cols, B.ld, (tp.per_z && tp.tpc > 1) ? tp.n_tap : BN));
  static uint64_t attr_set = 0;  // per device
  int dev = 0;
  DS_CUDA_TRY(cudaGetDevice(&dev));
  if (!(attr_set >> (dev & 63) & 1)) {
    DS_CUDA_TRY(cudaFuncSetAttribute(gemm_tf32_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     GemmSmem<BN>::TOTAL));
    attr_set |= 1ull << (dev & 63);
  }
  const uint32_t kps = ((K + splits - 1) / splits + kBK - 1) / kBK * kBK;
  const uint32_t ngroups = (tp.n > 0 && tp.per_z) ? (tp.n + tp.tpc - 1) / tp.tpc : 1;
  const uint32_t zdim = (tp.n > 0 && tp.per_z) ? ngroups * splits : (tp.n > 0 ? 1 : splits);
  const uint32_t gx = (N + BN - 1) / BN, gy = (M + kBM - 1) / kBM;
  const uint64_t ntiles = 1ull * gx * gy * zdim;
  if (ntiles == 0) return DS_OK;
  if (ntiles > 0xFFFFFFFFull) return set_error(DS_E_CONTRACT, "gemm: too many tiles");
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const uint64_t slots = static_cast<uint64_t>(nsm) * GemmSmem<BN>::CTAS;  // persistent CTAs
  const uint32_t grid = static_cast<uint32_t>(ntiles < slots ? ntiles : slots);
  gemm_tf32_kernel<BN><<<grid, GemmSmem<BN>::THREADS, GemmSmem<BN>::TOTAL, s>>>(ma, mb, ep, tp, M, N, K, kps, splits, gx, gy,
                                                                   static_cast<uint32_t>(ntiles));
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

int launch_any(const GemmOperand& A, const GemmOperand& B, const GemmEpilogue& ep, const GemmTaps& tp, uint32_t M,
               uint32_t N, uint32_t K, uint32_t splits, cudaStream_t s) {
  if (tp.n > 0 && !tp.per_z && tp.halo_rows > 0) {
    switch (gemm_pick_bn(N)) {
      case 48: return launch_halo<48>(A, B, ep, tp, M, N, s);
      case 64: return launch_halo<64>(A, B, ep, tp, M, N, s);
      case 96: return launch_halo<96>(A, B, ep, tp, M, N, s);
      case 128: return launch_halo<128>(A, B, ep, tp, M, N, s);
      case 192: return launch_halo<192>(A, B, ep, tp, M, N, s);
      default: return launch_halo<256>(A, B, ep, tp, M, N, s);
    }
  }
  if (tp.per_z && tp.tpc > 1) {  // grouped taps: the tile is exactly tpc x n_tap wide
    switch (tp.tpc * tp.n_tap) {
      case 192: return launch_bn<192>(A, B, ep, tp, M, N, K, splits, s);
      case 240: return launch_bn<240>(A, B, ep, tp, M, N, K, splits, s);
      case 256: return launch_bn<256>(A, B, ep, tp, M, N, K, splits, s);
      default: return set_error(DS_E_CONTRACT, "gemm: no tile for %u taps x %u", tp.tpc, tp.n_tap);
    }
  }
  switch (gemm_pick_bn(N)) {
    case 48: return launch_bn<48>(A, B, ep, tp, M, N, K, splits, s);
    case 64: return launch_bn<64>(A, B, ep, tp, M, N, K, splits, s);
    case 96: return launch_bn<96>(A, B, ep, tp, M, N, K, splits, s);
    case 128: return launch_bn<128>(A, B, ep, tp, M, N, K, splits, s);
    case 192: return launch_bn<192>(A, B, ep, tp, M, N, K, splits, s);
    default: return launch_bn<256>(A, B, ep, tp, M, N, K, splits, s);
  }
}

int launch_reduce(const float* slabs, uint32_t ntaps, uint64_t tap_stride, uint32_t nparts, uint64_t part_stride,
                  uint32_t d_col_step, const GemmEpilogue& ep, uint32_t M, uint32_t N, cudaStream_t s,
                  uint32_t col_limit = 0xFFFFFFFFu) {
  const uint64_t total = static_cast<uint64_t>(ntaps) * M * N;
  const unsigned blocks = static_cast<unsigned>(std::min<uint64_t>((total + 255) / 256, 148ull * 16));
  gemm_reduce_kernel<<<blocks, 256, 0, s>>>(slabs, ntaps, tap_stride, nparts, part_stride, d_col_step, ep, M, N,
                                            col_limit);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

// hi = x with the 13 low mantissa bits cleared (exact in tf32), lo = x - hi (exact in f32)
__global__ void split_tf32_kernel(const float* __restrict__ x, uint64_t n, float* __restrict__ hi,
                                  float* __restrict__ lo) {
  for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < n; i += gridDim.x * 256ull) {
    const float v = x[i];
    const float h = __uint_as_float(__float_as_uint(v) & 0xFFFFE000u);
    hi[i] = h;
    lo[i] = v - h;
  }
}

// DS_GEMM_HALO=1 enables the halo conv tiles. Off by default: measured on B200 both halo
// layouts are exact but slower end to end for the AlexNet layers — the canonical no-swizzle
// halo (3-D TMA box, 16-byte inner dimension) 1.2x, the 128-byte swizzled halo (tap windows
// start at any row of the 8-row swizzle atom; the descriptor base offset stays 0 because the
// hardware swizzles on absolute address bits — tools/taps_test.cu ACC_TAPS checks it) 1.15x:
// the per-tap operand traffic it removes was not the limiter. Read per call.
bool halo_enabled() {
  const char* e = getenv("DS_GEMM_HALO");
  return e && e[0] == '1';
}

bool exact_mode() {  // DS_GEMM_3XTF32=1: f32-accurate products (parity diagnostics; read per call)
  const char* e = getenv("DS_GEMM_3XTF32");
  return e && e[0] == '1';
}

// 3xTF32: A.B ~= Ahi.Bhi + Ahi.Blo + Alo.Bhi as three raw slab sets, reduced with the epilogue
int launch_3xtf32(const GemmOperand& A, const GemmOperand& B, uint32_t M, uint32_t N, uint32_t K, const GemmTaps& tp,
                  const GemmEpilogue& ep_in, cudaStream_t s) {
  const uint64_t na = A.rows * A.ld, nb = B.rows * B.ld;
  const uint32_t ntz = (tp.n > 0 && tp.per_z) ? (tp.n + tp.tpc - 1) / tp.tpc : 1;
  const uint64_t set = static_cast<uint64_t>(ntz) * M * N;
  float *ab = nullptr, *bb = nullptr, *slab = nullptr;
  DS_CUDA_TRY(cudaMallocAsync(&ab, 2 * na * 4, s));
  DS_CUDA_TRY(cudaMallocAsync(&bb, 2 * nb * 4, s));
  DS_CUDA_TRY(cudaMallocAsync(&slab, 3 * set * 4, s));
  split_tf32_kernel<<<4096, 256, 0, s>>>(A.p, na, ab, ab + na);
  split_tf32_kernel<<<4096, 256, 0, s>>>(B.p, nb, bb, bb + nb);
  GemmEpilogue raw = ep_in;
  raw.raw = true;
  raw.split_stride = static_cast<uint64_t>(M) * N;
  int rc = DS_OK;
  const int ia[3] = {0, 0, 1}, ib[3] = {0, 1, 0};
  for (int t = 0; t < 3 && rc == DS_OK; ++t) {
    GemmOperand a = A, b = B;
    a.p = ab + ia[t] * na;
    b.p = bb + ib[t] * nb;
    raw.D = slab + t * set;
    rc = launch_any(a, b, raw, tp, M, N, K, 1, s);
  }
  if (rc == DS_OK)
    rc = launch_reduce(slab, ntz, static_cast<uint64_t>(M) * N, 3, set, tp.per_z ? tp.tpc * tp.d_col_step : 0, ep_in, M,
                       N, s, tp.per_z ? tp.n * tp.d_col_step : 0xFFFFFFFFu);
  cudaFreeAsync(ab, s);
  cudaFreeAsync(bb, s);
  cudaFreeAsync(slab, s);
  return rc;
}

}  // namespace

uint32_t gemm_ctas_per_sm(uint32_t bn) {  // co-resident CTAs of one tile width (GemmSmem<BN>::CTAS)
  switch (bn) {
    case 48: return GemmSmem<48>::CTAS;
    case 64: return GemmSmem<64>::CTAS;
    case 96: return GemmSmem<96>::CTAS;
    case 128: return GemmSmem<128>::CTAS;
    case 192: return GemmSmem<192>::CTAS;
    case 240: return GemmSmem<240>::CTAS;
    default: return GemmSmem<256>::CTAS;
  }
}

// the tile width (MMA N) with the least padding past N; ties go to the wider tile, which
// re-reads the A operand fewer times
uint32_t gemm_pick_bn(uint32_t N) {
  static const uint32_t cap = [] {  // DS_GEMM_MAXBN: cap the tile width (experiments)
    const char* e = getenv("DS_GEMM_MAXBN");
    return e ? static_cast<uint32_t>(atoi(e)) : 256u;
  }();
  uint32_t best = 0, waste = ~0u;
  for (uint32_t bn : {256u, 192u, 128u, 96u, 64u, 48u}) {
    if (bn > cap && bn != 48) continue;
    const uint32_t w = (N + bn - 1) / bn * bn - N;
    if (w < waste) best = bn, waste = w;
  }
  return best;
}

int launch_gemm(const GemmOperand& A, const GemmOperand& B, uint32_t M, uint32_t N, uint32_t K, const GemmTaps* taps,
                const GemmEpilogue& ep_in, uint32_t splits, float* part, cudaStream_t s) {
  if (M == 0 || N == 0) return DS_OK;
  GemmTaps tp;
  if (taps) tp = *taps;
  if (tp.n < 0 || tp.n > kMaxTaps) return set_error(DS_E_CONTRACT, "gemm: at most %d taps", kMaxTaps);
  if (tp.n > 0 && !tp.per_z && (tp.kt == 0 || tp.kt % 8)) return set_error(DS_E_CONTRACT, "gemm: tap width %% 8");
  tp.tpc = 1;
  tp.n_tap = N;
  tp.halo_rows = 0;
  if (tp.n > 0 && !tp.per_z && halo_enabled() && A.cols % 4 == 0 && A.ld % 4 == 0) {
    // halo mode: one A column offset, shifts within 128 rows (a_row becomes the row inside the halo)
    int32_t lo = tp.a_row[0], hi = tp.a_row[0];
    bool same_col = (tp.a_col[0] % 4) == 0;
    for (int t = 1; t < tp.n; ++t) {
      lo = std::min(lo, tp.a_row[t]);
      hi = std::max(hi, tp.a_row[t]);
      same_col = same_col && tp.a_col[t] == tp.a_col[0];
    }
    if (same_col && hi - lo <= 128) {
      tp.halo_lo = lo;
      tp.halo_rows = static_cast<uint32_t>(kBM + hi - lo);
      for (int t = 0; t < tp.n; ++t) tp.a_row[t] -= lo;
    }
  }
  if (tp.n > 1 && tp.per_z && tp.d_col_step == N) {  // stack taps along N: one A tile feeds up to 256 columns
    const uint32_t g = std::min<uint32_t>(static_cast<uint32_t>(tp.n), 256 / N);
    if (g > 1 && (g * N == 192 || g * N == 240 || g * N == 256)) {
      tp.tpc = g;
      N = g * N;  // the kernel's N is the group width; columns past the last tap are clipped
    }
  }
  if (exact_mode()) return launch_3xtf32(A, B, M, N, K, tp, ep_in, s);
  if (splits == 0) splits = 1;
  if (tp.n > 0 && !tp.per_z) {
    splits = 1;  // K is given by the taps
  } else {
    const uint32_t max_splits = std::max<uint32_t>(1, (K + kBK - 1) / kBK);
    if (splits > max_splits) splits = max_splits;
  }
  if (splits > 1 && !part) return set_error(DS_E_CONTRACT, "gemm: split-K needs a partial buffer");
  GemmEpilogue ep = ep_in;
  const uint32_t ntz = (tp.n > 0 && tp.per_z) ? (tp.n + tp.tpc - 1) / tp.tpc : 1;
  if (splits > 1) {  // raw partial slabs [tap][split][M][N], reduced below with the epilogue
    ep.D = part;
    ep.raw = true;
    ep.split_stride = static_cast<uint64_t>(M) * N;
  }
  DS_TRY(launch_any(A, B, ep, tp, M, N, K, splits, s));
  if (splits > 1)
    DS_TRY(launch_reduce(part, ntz, static_cast<uint64_t>(splits) * M * N, splits, static_cast<uint64_t>(M) * N,
                         tp.per_z ? tp.tpc * tp.d_col_step : 0, ep_in, M, N, s,
                         tp.per_z ? tp.n * tp.d_col_step : 0xFFFFFFFFu));
  return DS_OK;
}

int launch_gemm_tf32(const float* A, uint64_t lda, const float* B, uint64_t ldb, uint32_t M, uint32_t N, uint32_t K,
                     const GemmEpilogue& ep, uint32_t splits, float* part, cudaStream_t s) {
  GemmOperand a, b;
  a.p = A, a.rows = M, a.cols = K, a.ld = lda;
  b.p = B, b.rows = N, b.cols = K, b.ld = ldb;
  return launch_gemm(a, b, M, N, K, nullptr, ep, splits, part, s);
}

}  // namespace dsb

extern "C" int ds_gemm_tf32(const float* A, uint64_t lda, const float* B, uint64_t ldb, float* D, uint64_t ldd,
                            uint32_t M, uint32_t N, uint32_t K, float scale, const float* bias_n, const float* bias_m,
                            int relu, uint32_t splits, float* part, void* stream) {
  if (!A || !B || !D) return dsb::set_error(DS_E_CONTRACT, "gemm: null operand");
  dsb::GemmEpilogue ep{};
  ep.D = D;
  ep.ldd = ldd;
  ep.scale = scale;
  ep.bias_n = bias_n;
  ep.bias_m = bias_m;
  ep.relu = relu != 0;
  return dsb::launch_gemm_tf32(A, lda, B, ldb, M, N, K, ep, splits, part, static_cast<cudaStream_t>(stream));
}
