// mlp_tc.cu — the fast (tensor-core) mode of the worker's local SGD step for the
// one-hidden-layer MLP: sample_loss_grad / loss_and_grad (model.cpp:185-263), the SGD
// update (param_vector.cpp:21-39 + engine.cpp:75-78), ExchangePolicy (engine.cpp:35-48)
// and the elastic exchange (exchanger.cpp:76-92 / simulator.cpp:114-121), as ONE
// persistent launch of one thread-block cluster per worker.
//
// Numerics (DS_ENGINE_TC): the two dense contractions run on the 5th-generation tensor
// cores with bf16 operands and f32 accumulation in TMEM —
//   forward  Z1[b x 16] = X[b x F] . W1s[16 x F]^T      (tcgen05.mma kind::f16)
//   dW1      D[128 f x 16] = X^T[128 f x b] . d1[b x 16] (A = the same X tile read MN-major)
// everything else (tanh, logits, softmax-CE, the small W2/bias gradients, SGD, policy,
// exchange) in f32 on the CUDA cores; the parameters stay f32 (the master copy of the
// CTA's W1 rows lives in shared memory, a bf16 copy feeds the MMA). This is a tolerance
// mode (bf16 <= 1e-3 relative); the bit-exact f64 reference order is the
// DS_ENGINE_FUSED / LAYERED path.
//
// Work split (measured, profiles/r02_umma_timing.md): a tcgen05.mma of these small shapes
// costs ~55 cycles however small N is, one SM ingests a 32 x 784 batch at ~50 B/cycle, and
// a cross-SM exchange costs ~500 cycles per phase. So the hidden units are split over the
// CTAs of ONE cluster (16 units per CTA: H = 256 -> 16 CTAs), each CTA streams the whole
// batch, and the only cross-CTA traffic per step is two tiny DSMEM phases (st.async +
// mbarrier complete_tx): a reduce-scatter of the partial logits by batch rows and an
// all-gather of the output deltas and per-row losses.
//
// Batches: the engine keeps a bf16 copy of the shard (and of host-fed rows); warp 4 stages
// step s+2's rows while step s+1 computes with TMA tile::gather4 loads (4 gathered rows x
// 64 features per instruction, written straight into the SWIZZLE_128B layout), each CTA
// issuing 1/NC of them MULTICAST to every CTA of the cluster: one L2 read per row chunk
// per cluster, no register or LSU traffic. A buffer is refilled once every CTA finished
// the dW1 MMAs that read it (known from the next step's R messages).
// Warp roles (warp specialisation): warps 0-7 compute, warp 8 issues the TMA gathers,
// warp 9 every tcgen05.mma. The MMA warp feeds the next step's forward tile by tile as the
// compute warps release each tile's updated W1 (mbarriers), so no compute warp ever waits
// behind an MMA issue.
// The compute warps never use a CTA-wide or cluster-wide barrier inside the step loop;
// cross-CTA signals are st.async messages that complete a receiver's mbarrier.
//
// Shared memory (operand tiles 1 KB aligned):
//   X[2]  bf16 batch rows, K-major SWIZZLE_128B: [atom a = 64 features][row group g]
//         [row%8][128 B] (16-byte chunk index XOR row%8), plus one atom of slack: the
//         forward MMA runs with M = 64, so rows 32..63 alias the next atom (ignored);
//   Wbf   bf16 copy of the CTA's 16 W1 rows, MN-major SWIZZLE_32B: per feature one 32-byte
//         row of the 16 units (chunk XOR (f>>2)&1), 8-feature atoms of 256 B — so a thread
//         owning feature f writes its 16 updated weights as two 16-byte stores;
//   D1b   bf16 delta1^T [16 units x 32 rows], K-major SWIZZLE_128B (B operand of dW1);
//   small f32 state (activations, deltas, W2 columns, biases, DSMEM inboxes).
// TMEM (256 columns): forward accumulator at column 0 (M = 64 layout: rows 0-15 in lanes
// 0-15, rows 16-31 in lanes 32-47); dW1 tile t at column 32 + 16 t and the f32 MASTER copy
// of the CTA's W1 rows at column 144 + 16 t (lane = feature within the 128-feature tile,
// column = unit). Keeping the master in TMEM keeps the SGD's f32 traffic off shared memory,
// whose bandwidth the overlapped forward MMAs need for their operands.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>

#include <algorithm>
#include <mutex>
#include <cstdlib>

#include "conv_tc.cuh"
#include "ds_common.cuh"
#include "engine.cuh"

namespace dsb {
namespace {

constexpr uint32_t kCW = 8;              // compute warps 0-7
constexpr uint32_t kCT = kCW * 32;       // compute threads
constexpr int kTT = (kCW + 2) * 32;      // + the TMA warp (kCW) and the MMA warp (kCW + 1)
constexpr int kHC = 16;        // hidden units per CTA (MMA N of the forward)
constexpr int kBM = 32;        // max batch rows (MMA rows 0..31 of M = 64)
constexpr int kMaxC = 16;      // classes: the logits MMA's N
constexpr int kMaxNC = 16;     // CTAs per cluster (non-portable size above 8)
constexpr uint32_t kTmemCols = 256;
constexpr uint32_t kBarCompute = 1;  // named barrier of the compute warps
constexpr uint32_t kBarAct = 2;      // named barrier of compute warps 0, 1, 4, 5 (activations, W2 / b SGD)
constexpr uint32_t kNumBars = 28;

// ---------------------------------------------------------------------------------
// PTX helpers
// ---------------------------------------------------------------------------------
using tc::saddr;

__device__ __forceinline__ uint64_t sdesc_sw(uint32_t addr, uint32_t lbo, uint32_t sbo, uint64_t layout) {
  return static_cast<uint64_t>((addr >> 4) & 0x3FFF) | (static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16) |
         (static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46) | (layout << 61);
}
constexpr uint64_t kSw128 = 2, kSw32 = 6;
// kind::f16 with bf16 A/B, f32 D; a_mn / b_mn: operand is MN-major
__host__ __device__ constexpr uint32_t idesc_bf16(int m, int n, int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(a_mn) << 15) |
         (static_cast<uint32_t>(b_mn) << 16) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(m >> 4) << 24);
}
// Issued by a whole warp with warp-uniform operands; one elected lane issues.
__device__ __forceinline__ void mma_bf16(uint32_t tmem, uint64_t da, uint64_t db, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
      "l"(da), "l"(db), "r"(id), "r"(acc));
}
// one thread issues (the caller picks it): no per-MMA elect in a long chain
__device__ __forceinline__ void mma_bf16_1(uint32_t tmem, uint64_t da, uint64_t db, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(
                   tmem),
               "l"(da), "l"(db), "r"(id), "r"(acc));
}
__device__ __forceinline__ void mma_tf32(uint32_t tmem, uint64_t da, uint64_t db, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred e, p;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
      "l"(da), "l"(db), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit_1(uint64_t* mbar) {  // one thread (the caller picks it)
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(saddr(mbar))
               : "memory");
}
__device__ __forceinline__ void mma_tf32_1(uint32_t tmem, uint64_t da, uint64_t db, uint32_t id, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(
                   tmem),
               "l"(da), "l"(db), "r"(id), "r"(acc));
}
__device__ __forceinline__ void commit_elect(uint64_t* mbar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(saddr(mbar))
      : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync() {  // every thread of every CTA
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(rank));
  return r;
}
// 16 bytes into peer `rank`'s shared memory; completes tx bytes on the peer's mbarrier
__device__ __forceinline__ void st_async16(const void* local_dst, const void* local_bar, uint32_t rank, float4 v) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.f32 [%0], {%1,%2,%3,%4}, [%5];" ::"r"(
                   mapa(saddr(local_dst), rank)),
               "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w), "r"(mapa(saddr(local_bar), rank))
               : "memory");
}
// A receiver arms its mbarrier with the bytes it expects; a sender's complete_tx may land
// before the arming (the transaction count goes transiently negative, the phase cannot
// complete before the local arrival).
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void named_sync(uint32_t id, uint32_t n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void csync() { named_sync(kBarCompute, kCT); }  // compute warps only
// Center accesses: weak loads that never allocate in L1 (so no stale line exists for another
// worker's writes) and plain stores (L1 is write-through); measured several times faster
// here than the strong .cg forms.
__device__ __forceinline__ float ld_center(const float* p) {
  float v;
  asm volatile("ld.global.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p) : "memory");
  return v;
}
// TMA bulk copies of the CTA's center rows (one-shard exchange): global -> shared with an
// mbarrier transaction count, and back shared -> global as a bulk group
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src), "r"(bytes), "r"(static_cast<uint32_t>(__cvta_generic_to_shared(bar)))
               : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(static_cast<uint32_t>(__cvta_generic_to_shared(src))), "r"(bytes)
               : "memory");
}
// dst[i] += src[i] (f32, round to nearest) for a whole row, as one bulk reduction
__device__ __forceinline__ void bulk_add_s2g(float* dst, const float* src, uint32_t bytes) {
  asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(dst),
               "r"(static_cast<uint32_t>(__cvta_generic_to_shared(src))), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t*>(&h);
}

// byte offset of (row, 8-element chunk q) in a K-major SW128 tile with `rpa` rows per atom
__device__ __forceinline__ uint32_t sw128_chunk(uint32_t row, uint32_t q, uint32_t rpa) {
  return (q >> 3) * (rpa * 128) + (row >> 3) * 1024 + (row & 7) * 128 + (((q & 7) ^ (row & 7)) << 4);
}
__device__ __forceinline__ uint32_t sw128_elem(uint32_t row, uint32_t k, uint32_t rpa) {
  return sw128_chunk(row, k >> 3, rpa) + (k & 7) * 2;
}
// MN-major SW32 W1 copy: feature f's 16 units, 16-byte half h (units 8h..8h+7)
__device__ __forceinline__ uint32_t wbf_chunk(uint32_t f, uint32_t h) {
  return (f >> 3) * 256 + (f & 7) * 32 + ((h ^ ((f >> 2) & 1)) << 4);
}
constexpr uint32_t kColLg = 16, kColDw = 32, kColW1 = 144;  // TMEM columns: logits, dW1 tiles, f32 W1 master
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const float (&v)[16]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15]))
      : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const float (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr),
               "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])),
               "r"(__float_as_uint(v[3])), "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])),
               "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7]))
               : "memory");
}
__device__ __forceinline__ void tmem_ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
// tcgen05.ld without the wait, and a wait that names the destination registers (so no use
// of them can be scheduled above it): two loads in flight behind one wait
__device__ __forceinline__ void tmem_ld8_raw(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
}
__device__ __forceinline__ void tmem_wait_ld2(uint32_t (&a)[8], uint32_t (&b)[8]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(a[0]), "+r"(a[1]), "+r"(a[2]), "+r"(a[3]), "+r"(a[4]), "+r"(a[5]), "+r"(a[6]), "+r"(a[7]),
                 "+r"(b[0]), "+r"(b[1]), "+r"(b[2]), "+r"(b[3]), "+r"(b[4]), "+r"(b[5]), "+r"(b[6]), "+r"(b[7])
               :
               : "memory");
}
// 8 units (half h) of feature f's bf16 row in the MN-major SW32 W1 copy
__device__ __forceinline__ void store_wbf_half(unsigned char* Wbf, uint32_t f, uint32_t h, const float (&o)[8]) {
  *reinterpret_cast<uint4*>(Wbf + wbf_chunk(f, h)) =
      make_uint4(pack_bf16(o[0], o[1]), pack_bf16(o[2], o[3]), pack_bf16(o[4], o[5]), pack_bf16(o[6], o[7]));
}

// rows owned per CTA in the logits reduce-scatter, and the R / G message sizes (floats)
struct TcMsg {
  uint32_t RP, Cp, MR, MG;
};
__host__ __device__ inline TcMsg tc_msg(uint32_t B, uint32_t C, uint32_t NC) {
  TcMsg m{};
  m.RP = (B + NC - 1) / NC;
  m.Cp = (C + 3) & ~3u;                                // a row's classes, padded to 16 bytes
  m.MR = m.RP * m.Cp + 4;                              // [RP][Cp] partial logits, flags piece
  m.MG = m.RP * (m.Cp + 4);                           // per row: [Cp] deltas, loss, flags, 2 pad
  return m;
}

struct TcSmem {
  uint32_t NA, NT, NK;      // 64-feature atoms, 128-feature dW1 tiles, 16-feature K steps
  uint32_t xbytes;          // one X buffer (+1 atom slack)
  uint32_t x0, wbf, d1b, a1c, w2c, small, total;
};
// small f32 state, in order: D1 [32][17]; b1c [16]; b2s [kMaxC]; inR [NC][MR];
// inG [NC][MG]; b2in [kMaxC]; then u32 lab [2][32], 32 spare words; then the mbarriers.
__host__ __device__ inline uint32_t tc_small_floats(uint32_t NC, const TcMsg& m) {
  return kBM * 17 + kHC + kMaxC + NC * m.MR + NC * m.MG + kMaxC;
}
// tf32 canonical K-major (no swizzle) offsets, in floats: A1 [64 rows][16 units] and the
// W2 columns as the logits MMA's B operand [16 classes][16 units]
__device__ __forceinline__ uint32_t a1c_idx(uint32_t r, uint32_t j) {
  return (j >> 2) * 256 + (r >> 3) * 32 + (r & 7) * 4 + (j & 3);
}
__device__ __forceinline__ uint32_t w2c_idx(uint32_t k, uint32_t j) {
  return (j >> 2) * 64 + (k >> 3) * 32 + (k & 7) * 4 + (j & 3);
}
__host__ __device__ inline uint32_t tc_bars_off(uint32_t small, uint32_t NC, const TcMsg& m) {
  return (small + tc_small_floats(NC, m) * 4 + 4 * kBM * 4 + 7) & ~7u;
}
__host__ __device__ inline TcSmem tc_smem(uint32_t F, uint32_t B, uint32_t C, uint32_t NC) {
  TcSmem p{};
  p.NA = (F + 63) / 64;
  p.NT = (F + 127) / 128;
  p.NK = (F + 15) / 16;
  p.xbytes = (p.NA + 1) * 4096;
  p.x0 = 0;                                        // X[0], X[1]
  p.wbf = 2 * p.xbytes;                            // NK * 2 atoms x 256 B
  p.d1b = p.wbf + ((p.NK * 512 + 1023) & ~1023u);  // 16 rows x 128 B
  p.a1c = p.d1b + 2048;                            // A1 tf32 canonical: 64 rows x 16 units
  p.w2c = p.a1c + 4096;                            // W2 columns tf32 canonical: 16 classes x 16 units
  p.small = p.w2c + 1024;
  p.total = tc_bars_off(p.small, NC, tc_msg(B, C, NC)) + kNumBars * 8;
  return p;
}

// DS_FUSED_PROFILE: per-phase globaltimer stamps of CTA 0 (run_fused prints the medians)
__device__ __forceinline__ void tstamp(unsigned long long* prof, uint64_t step, int slot, uint32_t rank) {
  if (prof && rank == 0 && threadIdx.x == 0) prof[step * kProfSlots + slot] = globaltimer_ns();
}
// variant builds (tools/ experiments): DS_TC_PROF_X stamps inside the exchange, DS_TC_PROF_M
// stamps the MMA warp's timeline, instead of the compute warps' step phases
__device__ __forceinline__ void tstamp_m(unsigned long long* prof, uint64_t step, int slot, uint32_t rank) {
  if (prof && rank == 0 && threadIdx.x == (kCW + 1) * 32) prof[step * kProfSlots + slot] = globaltimer_ns();
}
__device__ __forceinline__ void tstamp_t(unsigned long long* prof, uint64_t step, int slot, uint32_t rank) {
  if (prof && rank == 0 && threadIdx.x == kCW * 32) prof[step * kProfSlots + slot] = globaltimer_ns();
}
#if defined(DS_TC_PROF_T)
#define TSTAMP_MAIN(...)
#define TSTAMP_X(...)
#define TSTAMP_M(...)
#define TSTAMP_T(...) tstamp_t(__VA_ARGS__)
#define TSTAMP_TM(...) tstamp_m(__VA_ARGS__)
#elif defined(DS_TC_PROF_X)
#define TSTAMP_MAIN(...)
#define TSTAMP_X(...) tstamp(__VA_ARGS__)
#define TSTAMP_M(...)
#elif defined(DS_TC_PROF_M)
#define TSTAMP_MAIN(...)
#define TSTAMP_X(...)
#define TSTAMP_M(...) tstamp_m(__VA_ARGS__)
#else
#define TSTAMP_MAIN(...) tstamp(__VA_ARGS__)
#define TSTAMP_X(...)
#define TSTAMP_M(...)
#endif
#ifndef TSTAMP_T
#define TSTAMP_T(...)
#define TSTAMP_TM(...)
#endif


constexpr int kMaxGroup = 8;  // workers per launch
struct TcLaunch {
  CUtensorMap maps[kMaxGroup];  // batch-row maps (64-byte aligned, first)
  FusedArgs args[kMaxGroup];
  uint32_t n;
};

struct PolicyTc {
  double cum, cut;
  uint32_t tau, since, fire, period;
  int32_t adaptive;
};

// Polling mbarrier wait that gives up when the compute warps quit (early stop).
__device__ __forceinline__ bool mbar_wait_or_quit(uint64_t* b, uint32_t parity, const volatile uint32_t* quit) {
  while (true) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(saddr(b)), "r"(parity)
        : "memory");
    if (ok) return true;
    if (*quit) return false;
  }
}

// One launch trains `n` workers (engines), one cluster each: worker w = cluster w. All
// clusters are co-resident (cooperative launch when n > 1), so workers may wait on each
// other's exchange tickets inside the kernel (the deterministic multi-worker schedule).
__global__ void __launch_bounds__(kTT, 1) mlp_tc_kernel(const __grid_constant__ TcLaunch P) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // dynamic smem base must be 1 KB aligned for SWIZZLE_128B tiles
  unsigned char* sm = smem_raw + ((1024 - (saddr(smem_raw) & 1023)) & 1023);
  uint32_t NC;  // CTAs per worker = cluster size
  asm("mov.u32 %0, %%cluster_nctarank;" : "=r"(NC));
  const uint32_t wid = blockIdx.x / NC;
  const FusedArgs& A = P.args[wid];
  const CUtensorMap& tmx = P.maps[wid];
  const uint32_t F = A.F, H = A.H, C = A.C, B = A.B;
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const TcSmem L = tc_smem(F, B, C, NC);
  const TcMsg M = tc_msg(B, C, NC);
  const uint32_t rank = cluster_rank();
  const uint32_t u0 = rank * kHC;
  const uint32_t HU = u0 < H ? min(static_cast<uint32_t>(kHC), H - u0) : 0u;  // valid units of this CTA
  const uint32_t RP = M.RP, Cp = M.Cp, MR = M.MR, MG = M.MG;  // rows owned per CTA, message floats
  // rows of this CTA's R messages that exist (rows < 32): what every peer sends us
  const uint32_t own_rows = rank * RP < kBM ? min(RP, kBM - rank * RP) : 0u;

  auto Xbuf = [&](uint32_t b) -> unsigned char* { return sm + L.x0 + b * L.xbytes; };  // X[b]
  unsigned char* Wbf = sm + L.wbf;
  unsigned char* D1b = sm + L.d1b;
  float* A1c = reinterpret_cast<float*>(sm + L.a1c);   // tanh activations (tf32 A operand)
  float* W2cc = reinterpret_cast<float*>(sm + L.w2c);  // own W2 columns (tf32 B operand, f32 master)
  float* fs = reinterpret_cast<float*>(sm + L.small);
  float* D1 = fs;                       // [32][17] delta1 (f32)
  float* b1c = D1 + kBM * 17;           // [16]
  float* b2s = b1c + kHC;               // [kMaxC] replicated b2
  float* inR = b2s + kMaxC;             // [NC][MR]: slot p = CTA p's contribution
  float* inG = inR + NC * MR;           // [NC][MG]
  float* b2in = inG + NC * MG;          // [kMaxC] ticket / b2 broadcast from CTA 0
  uint32_t* lab = reinterpret_cast<uint32_t*>(b2in + kMaxC);  // [2][32] labels per X buffer
  // row r's delta2 / loss in the gathered G messages: fs[d2off[r] + k], fs[d2off[r] + RP*Cp - ..]
  // (slot r / RP); rows without a slot point at 16 zero words (zblk)
  uint32_t* d2off = lab + 2 * kBM;                            // [32]
  float* zblk = reinterpret_cast<float*>(d2off + kBM);        // [32] zeros (setup)
  uint64_t* bars = reinterpret_cast<uint64_t*>(sm + tc_bars_off(L.small, NC, M));
  uint64_t* xbar = bars;        // [2] batch staged in X[b] (armed with the batch bytes by the TMA warp)
  uint64_t* fbar = bars + 2;    // forward MMAs done
  uint64_t* rbar = bars + 3;    // R messages landed
  uint64_t* gbar = bars + 4;    // G messages landed
  uint64_t* ebar = bars + 5;    // (CTA != 0) ticket / exchanged b2 from CTA 0 landed
  uint64_t* cbar = bars + 6;    // (CTA 0) every peer finished its exchange slice
  uint64_t* d1rdy = bars + 7;   // delta1 of the step written (compute -> MMA warp)
  uint64_t* exdone = bars + 8;  // the step's exchange done (compute -> MMA warp)
  uint64_t* a1rdy = bars + 9;   // A1 of the step written (warps 0, 1, 4, 5 -> MMA warp)
  uint64_t* lgbar = bars + 10;  // partial logits in TMEM (MMA warp -> warps 0, 1)
  uint64_t* dtile = bars + 11;  // [8] dW1 MMAs of 128-feature tile t done (MMA warp -> compute)
  uint64_t* sgdd = bars + 19;   // [8] W1 SGD of tile t done by all compute warps (-> MMA warp)
  uint64_t* cxbar = bars + 27;  // the CTA's center rows staged for a one-shard exchange
  __shared__ uint32_t s_tmem, s_bad, s_stop, s_quit, s_rows[2];
  __shared__ unsigned long long s_can_stage;  // the TMA warp may stage steps <= s_can_stage
  __shared__ double s_loss;
  __shared__ PolicyTc s_pol;
  __shared__ unsigned long long s_ticket;

  DevState* st = A.st;
  const unsigned long long it0 = st->iter;
  const uint64_t w1o = 0, b1o = static_cast<uint64_t>(H) * F, w2o = b1o + H, b2o = w2o + static_cast<uint64_t>(C) * H;
  const float* Pin = A.params[A.cur];
  float* Pout = A.params[A.cur ^ static_cast<int>(A.steps & 1)];
  const float eta = A.eta, wd = A.wd;

  // ---- setup ---------------------------------------------------------------------
  if (warp == 0) tc::tmem_alloc<kTmemCols>(&s_tmem);
  if (tid == 0) {
    for (uint32_t i = 0; i < kNumBars; ++i) tc::mbar_init(bars + i, (i >= 19 && i < 27) ? kCW : (i == 9 ? 4u : 1u));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    s_pol.cum = st->cum;
    s_pol.cut = st->cut;
    s_pol.tau = st->tau;
    s_pol.since = st->since;
    s_pol.adaptive = st->adaptive;
    s_pol.fire = 0;
    s_pol.period = 0;
    s_stop = st->err ? 1u : 0u;
    s_bad = 0;
    s_quit = 0;
    s_can_stage = 1;  // both buffers start free
    s_loss = 0.0;
  }
  // zero the operand tiles once: padding chunks / rows must be finite
  for (uint32_t i = tid; i < L.small / 16; i += kTT) reinterpret_cast<float4*>(sm)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (uint32_t i = tid; i < tc_small_floats(NC, M); i += kTT) fs[i] = 0.f;  // inboxes: pad words stay 0
  if (tid < kBM) {
    const uint32_t p = tid / RP;
    d2off[tid] = p < NC ? static_cast<uint32_t>(inG - fs) + p * MG + (tid - p * RP) * (Cp + 4)
                        : static_cast<uint32_t>(zblk - fs);
    zblk[tid] = 0.f;
  }
  __syncthreads();
  for (uint32_t i = tid; i < kMaxC * kHC; i += kTT) {  // own W2 columns, b1 slice, b2
    const uint32_t k = i / kHC, j = i - k * kHC;
    W2cc[w2c_idx(k, j)] = (k < C && j < HU) ? Pin[w2o + static_cast<uint64_t>(k) * H + u0 + j] : 0.f;
  }
  if (tid < kHC) b1c[tid] = tid < HU ? Pin[b1o + u0 + tid] : 0.f;
  if (tid < kMaxC) b2s[tid] = tid < C ? Pin[b2o + tid] : 0.f;
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = s_tmem;
  // TMEM lane quarter and column half of a compute warp (tcgen05.ld/st reach lanes
  // 32*(warp%4)..+31 only): warps 0-3 take units 0-7, warps 4-7 units 8-15
  const uint32_t quarter = warp & 3, chalf = (warp >> 2) & 1;
  const uint32_t lane_base = (quarter * 32u) << 16;
  if (warp < kCW) {  // own W1 rows -> f32 master in TMEM (lane = feature) + bf16 MMA copy
    for (uint32_t t = 0; t < L.NT; ++t) {
      const uint32_t f = t * 128 + quarter * 32 + lane;
      float w[8];
#pragma unroll
      for (uint32_t i = 0; i < 8; ++i) {
        const uint32_t j = chalf * 8 + i;
        w[i] = (f < F && j < HU) ? Pin[w1o + static_cast<uint64_t>(u0 + j) * F + f] : 0.f;
      }
      tmem_st8(tmem + lane_base + kColW1 + t * kHC + chalf * 8, w);
      if (f < F) store_wbf_half(Wbf, f, chalf, w);
    }
    tmem_wait_st();
  }
  tc::fence_async_smem();
  tc::fence_before();
  __syncthreads();
  cluster_sync();  // every peer's barriers exist before any DSMEM traffic
  tc::fence_after();
  const long long clk0 = clock64();
  const unsigned long long gt0 = globaltimer_ns();
  uint64_t done = 0, xcount = 0;
  uint32_t bad_iter_step = 0;
  bool failed = false;
  const volatile uint32_t* quitp = &s_quit;

  if (warp == kCW) {
    // ================= TMA warp: stage every step's batch ===============================
    // Lane r holds batch row r's source row; gather g = (atom a, 4-row group g4) lands in
    // X[buf] + a*4096 + g4*512: 4 rows x 128 B, hardware-swizzled like the MMA reads it.
    // This CTA issues gathers g = rank, rank+NC, ... and multicasts them to the cluster.
    const uint32_t ngath = 8 * L.NA;
    const uint32_t xbytes_step = kBM * L.NA * 128;
    for (uint64_t s = 0; s < A.steps && !s_stop; ++s) {
      const uint32_t buf = static_cast<uint32_t>(s & 1);
      uint32_t R, row, y = 0;
      TSTAMP_T(A.prof, s, 0, rank);
      // the batch description first (host ring: a PCIe round trip for the word and one for
      // the labels), while the X buffer is still being read by step s-2's dW1 MMAs
      if (A.ring) {
        const uint32_t slot = static_cast<uint32_t>(s % A.ring_slots);
        uint32_t nrows = 1;
        if (lane == 0) {
          const uint32_t want = static_cast<uint32_t>(s + 1) & 0xFFFFFu;
          const unsigned long long t0 = globaltimer_ns();
          while (true) {
            uint32_t v;
            asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(A.ring_ready + slot) : "memory");
            if ((v & 0xFFFFFu) == want) {
              nrows = v >> 20;
              break;
            }
            if (globaltimer_ns() - t0 > 20000000000ull || *quitp) {
              atomicOr(&s_bad, DS_FLAG_STREAM_TIMEOUT);
              break;
            }
            __nanosleep(64);
          }
        }
        TSTAMP_T(A.prof, s, 1, rank);
        R = __shfl_sync(0xffffffffu, nrows, 0);
        row = slot * A.ring_slot_rows + (lane < R ? lane : 0u);
        // the slot was written by the copy engine before its word: labels after the acquire,
        // and the async proxy (the TMA gathers below) ordered after it
        if (lane < R) y = __ldcg(A.ring_y + static_cast<uint64_t>(slot) * A.ring_y_stride + lane);
        asm volatile("fence.proxy.async.global;" ::: "memory");
        if (y == 0xFFFFFFFFu) TSTAMP_T(A.prof, s, 9, rank);  // (keeps the label load before the stamp)
        TSTAMP_T(A.prof, s, 2, rank);
      } else {
        R = A.plan_rows[s];
        const uint32_t r0 = A.plan[s * B];
        row = lane < R ? A.plan[s * B + lane] : r0;  // padding rows repeat a valid row
        if (lane < R) y = __ldg(A.y + row);
      }
      if (lane == 0)  // every CTA finished the dW1 MMAs that last read X[buf]
        while (*reinterpret_cast<volatile unsigned long long*>(&s_can_stage) < s && !*quitp) __nanosleep(32);
      __syncwarp();
      if (*quitp) break;
      TSTAMP_T(A.prof, s, 3, rank);
      lab[buf * kBM + lane] = y;
      if (lane == 0) {
        s_rows[buf] = R;
        mbar_expect_tx(xbar + buf, xbytes_step);  // the multicasts of every CTA land here
      }
      const uint32_t mcast = (1u << NC) - 1u;
      const uint32_t cnt = ngath > rank ? (ngath - rank + NC - 1) / NC : 0u;  // this CTA's gathers
      for (uint32_t i0 = 0; i0 < cnt; i0 += 32) {  // warp-uniform trip count (shuffles below)
        const uint32_t i = i0 + lane;
        const uint32_t g = rank + i * NC;
        const uint32_t g4 = g & 7;
        const uint32_t r0 = __shfl_sync(0xffffffffu, row, (4 * g4) & 31);
        const uint32_t r1 = __shfl_sync(0xffffffffu, row, (4 * g4 + 1) & 31);
        const uint32_t r2 = __shfl_sync(0xffffffffu, row, (4 * g4 + 2) & 31);
        const uint32_t r3 = __shfl_sync(0xffffffffu, row, (4 * g4 + 3) & 31);
        if (i < cnt) {
          const uint32_t a = g >> 3;
          const uint32_t dst = saddr(Xbuf(buf) + a * 4096 + g4 * 512);
          if (NC > 1)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                ".multicast::cluster [%0], [%1, {%3, %4, %5, %6, %7}], [%2], %8;" ::"r"(dst),
                "l"(&tmx), "r"(saddr(xbar + buf)), "r"(a * 64), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
                "h"(static_cast<uint16_t>(mcast))
                : "memory");
          else
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes"
                " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(dst),
                "l"(&tmx), "r"(saddr(xbar + buf)), "r"(a * 64), "r"(r0), "r"(r1), "r"(r2), "r"(r3)
                : "memory");
        }
      }
      TSTAMP_T(A.prof, s, 4, rank);
    }
  } else if (warp == kCW + 1) {
    // ================= MMA warp: every tcgen05.mma of the step ============================
    // forward(s): Z1[64 x 16] = X[64 x F] . W1s[16 x F]^T, K = 16 per MMA, issued per
    // 128-feature tile as soon as the compute warps finished that tile's SGD of step s-1
    // (or after the exchange, or at once for the first step); dW1(s) per tile, one commit
    // each, once delta1(s) is written.
    const uint32_t idesc_fwd = idesc_bf16(64, kHC, 0, 1);
    const uint32_t idesc_dw = idesc_bf16(128, kHC, 1, 0);
    const uint32_t idesc_lg = tc::idesc_tf32(64, kMaxC);
    const uint64_t dw_b = sdesc_sw(saddr(D1b), 16, 1024, kSw128);
    const uint64_t fwd_b = sdesc_sw(saddr(Wbf), 0, 256, kSw32);
    uint32_t xph = 0;  // exdone parity
    for (uint64_t s = 0; s < A.steps && !s_stop; ++s) {
      const uint32_t buf = static_cast<uint32_t>(s & 1);
      const uint32_t pp = static_cast<uint32_t>((s - 1) & 1);  // phase parity of step s-1's barriers
      if (!mbar_wait_or_quit(xbar + buf, static_cast<uint32_t>((s >> 1) & 1), quitp)) break;
      TSTAMP_TM(A.prof, s, 5, rank);
      // the whole W1 update of step s-1 first: forward MMAs issued while the compute warps
      // still run the SGD (TMEM / smem traffic) were measured at half the tensor-pipe rate
      bool quit = false;
      if (s > 0)
        for (uint32_t t = 0; t < L.NT && !quit; ++t) quit = !mbar_wait_or_quit(sgdd + t, pp, quitp);
      if (quit) break;
      // step s-1's policy decision is final (computed before the compute warps' SGD arrivals)
      const bool prev_fired = s > 0 && s_pol.fire && A.has_master;
      if (prev_fired) {
        if (!mbar_wait_or_quit(exdone, xph, quitp)) break;
        xph ^= 1;
      }
      tc::fence_after();
      const uint64_t da0 = sdesc_sw(saddr(Xbuf(buf)), 16, 1024, kSw128);
      tc::fence_after();
      TSTAMP_M(A.prof, s, 2, rank);
      if (lane == 0) {  // +4096 B per 4 K steps (next atom), +32 B inside; B +512 B per K step
        uint64_t a = da0, b = fwd_b;
#pragma unroll 4
        for (uint32_t k = 0; k < L.NK; ++k, b += 32) {
          mma_bf16_1(tmem, a + (k & 3) * 2, b, idesc_fwd, k > 0);
          if ((k & 3) == 3) a += 256;
        }
      }
      if (lane == 0) commit_1(fbar);
      __syncwarp();
      TSTAMP_M(A.prof, s, 4, rank);
      TSTAMP_M(A.prof, s, 5, rank);
      // the CTA's partial logits: P[64 x 16] = A1[64 x 16] . W2c[16 x 16]^T, tf32, K = 8 x 2
      if (!mbar_wait_or_quit(a1rdy, buf, quitp)) break;
      tc::fence_after();
      if (lane == 0) {
#pragma unroll
        for (uint32_t kk = 0; kk < 2; ++kk)
          mma_tf32_1(tmem + kColLg, sdesc_sw(saddr(A1c) + kk * 2048, 1024, 128, 0),
                     sdesc_sw(saddr(W2cc) + kk * 512, 256, 128, 0), idesc_lg, kk > 0);
        commit_1(lgbar);
      }
      __syncwarp();
      TSTAMP_M(A.prof, s, 6, rank);
      if (!mbar_wait_or_quit(d1rdy, buf, quitp)) break;  // delta1(s) in D1b; the policy decided
      TSTAMP_M(A.prof, s, 0, rank);
      tc::fence_after();
      const uint64_t dx0 = sdesc_sw(saddr(Xbuf(buf)), 4096, 1024, kSw128);
      if (lane == 0) {
        for (uint32_t t = 0; t < L.NT; ++t) {
#pragma unroll
          for (uint32_t kk = 0; kk < 2; ++kk)  // K = 16 batch rows per MMA (2 row groups)
            mma_bf16_1(tmem + kColDw + t * kHC, dx0 + t * 512 + kk * 128, dw_b + kk * 2, idesc_dw, kk > 0);
          commit_1(dtile + t);
        }
      }
      __syncwarp();
      TSTAMP_M(A.prof, s, 1, rank);
    }
  } else {
    // ================= compute warps ======================================================
    uint32_t ph = 0;   // fbar / dtile / rbar / gbar / d1rdy parity: one completion per step
    uint32_t eph = 0;  // ebar / cbar parity: completions per exchange
    uint32_t cxph = 0;  // cxbar parity: one completion per bulk exchange
    for (uint64_t step = 0; step < A.steps && !s_stop; ++step) {
      const uint32_t buf = static_cast<uint32_t>(step & 1);
      TSTAMP_MAIN(A.prof, step, 0, rank);
      tc::mbar_wait(fbar, ph);
      tc::fence_after();
      TSTAMP_MAIN(A.prof, step, 1, rank);
      const uint32_t R = s_rows[buf];
      if (tid == 0 && NC > 1) mbar_expect_tx(rbar, (NC - 1) * (own_rows * Cp + 4) * 4);
      // ---- hidden activations (warps 0, 1; lane = row) -> A1c; logits on the tensor core -
      // tanh(x) = 1 - 2 / (exp(2x) + 1) (saturates correctly at +-inf); the MMA warp then
      // computes the CTA's partial logits P[64 x 16] = A1[64 x 16] . W2c[16 x 16]^T (tf32)
      if (warp < 2 || warp == 4 || warp == 5) {
        // warps 0/4 rows 0-15, 1/5 rows 16-31 (TMEM lanes 0-15 / 32-47); warps 0, 1 the
        // units 0-7, warps 4, 5 the units 8-15
        const uint32_t rw = warp & 1u, uh = warp >> 2;
        float z[8];
        tmem_ld8(tmem + ((rw * 32u) << 16) + uh * 8, z);
        const uint32_t r = rw * 16 + lane;
        if (lane < 16) {
          float a[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const float x = z[j] + b1c[uh * 8 + j];
            a[j] = r < R ? 1.f - __fdividef(2.f, __expf(2.f * x) + 1.f) : 0.f;
          }
#pragma unroll
          for (int c = 0; c < 2; ++c)
            *reinterpret_cast<float4*>(A1c + a1c_idx(r, uh * 8 + 4 * c)) =
                make_float4(a[4 * c], a[4 * c + 1], a[4 * c + 2], a[4 * c + 3]);
        }
        tc::fence_async_smem();
        tc::fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(a1rdy);
      }
      if (warp < 2) {
        const uint32_t r = warp * 16 + lane;
        tc::mbar_wait(lgbar, ph);
        tc::fence_after();
        float lg[16];
        tmem_ld16(tmem + ((warp * 32u) << 16) + kColLg, lg);
        // R phase: row r's partial logits go to its owner q = r / RP (slot `rank`)
        const uint32_t q = r / RP, rr = r - q * RP;
        if (lane < 16 && q < NC) {
          float* dst = inR + rank * MR + rr * Cp;
#pragma unroll
          for (uint32_t c4 = 0; c4 < 4; ++c4) {
            if (4 * c4 >= Cp) break;
            const float4 v = make_float4(4 * c4 < C ? lg[4 * c4] : 0.f, 4 * c4 + 1 < C ? lg[4 * c4 + 1] : 0.f,
                                         4 * c4 + 2 < C ? lg[4 * c4 + 2] : 0.f, 4 * c4 + 3 < C ? lg[4 * c4 + 3] : 0.f);
            if (q == rank)
              *reinterpret_cast<float4*>(dst + 4 * c4) = v;
            else
              st_async16(dst + 4 * c4, rbar, q, v);
          }
        }
      } else if (warp == 2 && lane < NC) {  // the flags word of every R message
        const float4 v = make_float4(__uint_as_float(s_bad), 0.f, 0.f, 0.f);
        float* dst = inR + rank * MR + RP * Cp;
        if (lane == rank)
          *reinterpret_cast<float4*>(dst) = v;
        else
          st_async16(dst, rbar, lane, v);
      }
      TSTAMP_MAIN(A.prof, step, 2, rank);
      if (NC > 1) tc::mbar_wait(rbar, ph);
      // every CTA sent its R message after finishing step-1: the X buffer of step-1 is free
      // cluster-wide, so the TMA warp may stage step+1 into it
      if (tid == 0) *reinterpret_cast<volatile unsigned long long*>(&s_can_stage) = step + 1;
      if (tid == 0 && NC > 1) mbar_expect_tx(gbar, (NC - 1) * MG * 4);
      csync();
      TSTAMP_MAIN(A.prof, step, 3, rank);
      // any CTA's failure of the previous step (its SGD) stops everyone here, together
      uint32_t prev_bad = 0;
#pragma unroll
      for (uint32_t p = 0; p < kMaxNC; ++p)
        if (p < NC) prev_bad |= __float_as_uint(inR[p * MR + RP * Cp]);
      if (prev_bad) {
        failed = true;
        bad_iter_step = static_cast<uint32_t>(step ? step : 1);  // step-1 failed (1-based: step)
        if (tid == 0) atomicOr(&st->flags, prev_bad);
        break;
      }
      // ---- softmax-CE for the CTA's own rows (one warp per row, lane = class) -----------
      // Each row's warp sends the row's record — [Cp] deltas, loss, flags — straight from
      // registers to every peer (G phase: every CTA gets every row), and writes its own copy.
      const uint32_t nch = Cp / 4 + 1;  // float4 chunks per row record
      for (uint32_t rr = warp; rr < RP; rr += kCW) {
        const uint32_t r = rank * RP + rr;
        const bool valid = r < R;  // rows past the batch (or past kBM) send zero records
        float z = -INFINITY;
        if (lane < C) {
          float acc[4] = {b2s[lane], 0.f, 0.f, 0.f};
#pragma unroll
          for (uint32_t p = 0; p < kMaxNC; ++p)
            if (p < NC) acc[p & 3] += inR[p * MR + rr * Cp + lane];
          z = (acc[0] + acc[1]) + (acc[2] + acc[3]);
        }
        float mx = z;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        const float ez = lane < C ? __expf(z - mx) : 0.f;
        float se = ez;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) se += __shfl_xor_sync(0xffffffffu, se, o);
        const uint32_t y = valid ? lab[buf * kBM + (r < kBM ? r : 0u)] : 0u;
        uint32_t bad = 0;
        if (valid && y >= C) bad |= DS_FLAG_LABEL_RANGE;
        const float lse = mx + __logf(se);
        const float zy = __shfl_sync(0xffffffffu, z, y < C ? y : 0);
        const float loss = valid ? lse - zy : 0.f;
        if (valid && !isfinite(loss)) bad |= DS_FLAG_LOSS_NONFINITE;
        const float d = valid && lane < C ? (ez / se - (lane == y ? 1.f : 0.f)) / static_cast<float>(R) : 0.f;
        const float fl = __uint_as_float(__reduce_or_sync(0xffffffffu, bad));
        float* own = inG + rank * MG + rr * (Cp + 4);
        if (lane < Cp) own[lane] = d;
        if (lane == 0) own[Cp] = loss, own[Cp + 1] = fl;
        for (uint32_t i0 = 0; i0 < (NC - 1) * nch; i0 += 32) {  // warp-uniform trips (shuffles)
          const uint32_t i = i0 + lane;
          const uint32_t c = i % nch, qi = i / nch;
          const uint32_t src = c * 4 < Cp ? c * 4 : 0u;
          const float v0 = __shfl_sync(0xffffffffu, d, src), v1 = __shfl_sync(0xffffffffu, d, (src + 1) & 31),
                      v2 = __shfl_sync(0xffffffffu, d, (src + 2) & 31), v3 = __shfl_sync(0xffffffffu, d, (src + 3) & 31);
          const float lz = __shfl_sync(0xffffffffu, loss, 0);
          if (i < (NC - 1) * nch) {
            const uint32_t q = qi + (qi >= rank ? 1u : 0u);  // every peer but us
            const float4 v = c * 4 < Cp ? make_float4(v0, v1, v2, v3) : make_float4(lz, fl, 0.f, 0.f);
            st_async16(own + c * 4, gbar, q, v);
          }
        }
      }
      if (NC > 1) tc::mbar_wait(gbar, ph);
      csync();
      TSTAMP_MAIN(A.prof, step, 4, rank);
      uint32_t gbad = __float_as_uint(fs[d2off[lane] + Cp + 1]);  // lane = row (zero records past R)
      gbad = __reduce_or_sync(0xffffffffu, gbad);
      if (gbad) {  // label / loss failure in loss_and_grad: stop before the update (model.cpp:176-181, 256)
        failed = true;
        bad_iter_step = static_cast<uint32_t>(step + 1);
        if (tid == 0) atomicOr(&st->flags, gbad);
        break;
      }
      // delta2 / per-row loss of row r straight from the gathered messages (slot r / RP)
      auto D2 = [&](uint32_t r, uint32_t k) -> float { return fs[d2off[r] + k]; };
      // ---- delta1 = (delta2 . W2[:, own]) * (1 - a^2): thread = (row r, 2 units) --------
      {
        const uint32_t r = tid >> 3, j0 = (tid & 7) * 2;
        float acc0 = 0.f, acc1 = 0.f;
        for (uint32_t k = 0; k < C; ++k) {
          const float d = D2(r, k);
          const float2 w = *reinterpret_cast<const float2*>(W2cc + w2c_idx(k, j0));
          acc0 = fmaf(d, w.x, acc0);
          acc1 = fmaf(d, w.y, acc1);
        }
        const float2 a = *reinterpret_cast<const float2*>(A1c + a1c_idx(r, j0));
        const float d0 = r < R ? acc0 * (1.f - a.x * a.x) : 0.f, d1 = r < R ? acc1 * (1.f - a.y * a.y) : 0.f;
        D1[r * 17 + j0] = d0;
        D1[r * 17 + j0 + 1] = d1;
        *reinterpret_cast<__nv_bfloat16*>(D1b + sw128_elem(j0, r, kHC)) = __float2bfloat16_rn(d0);
        *reinterpret_cast<__nv_bfloat16*>(D1b + sw128_elem(j0 + 1, r, kHC)) = __float2bfloat16_rn(d1);
      }
      tc::fence_async_smem();
      tc::fence_before();
      csync();
      if (tid == 0) tc::mbar_arrive(d1rdy);  // the MMA warp issues dW1(s)
      TSTAMP_MAIN(A.prof, step, 5, rank);
      // the batch loss and the policy, off the path to the dW1 MMAs: the MMA warp reads the
      // decision only at the next step, after every compute warp's SGD arrivals
      if (warp == kCW - 1) {  // batch loss (mean over rows) and the policy (engine.cpp:35-48)
        const uint32_t p = lane / RP;
        double l = (lane < R && p < NC) ? static_cast<double>(fs[d2off[lane] + Cp]) : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
        if (lane == 0) {
          s_loss = l / static_cast<double>(R);
          PolicyTc& pl = s_pol;
          pl.cum += s_loss;
          pl.since += 1;
          const bool fire = pl.adaptive ? (pl.cum > pl.cut) : (pl.since == pl.tau);
          pl.period = fire ? pl.since : 0u;
          pl.fire = fire ? 1u : 0u;
          if (fire) pl.cum = 0.0, pl.since = 0;
        }
      }

      uint32_t ubad = 0;
      // ---- W1 SGD per tile from the TMEM dW1 tile and master; release the tile to the
      // MMA warp (forward of step s+1 reads the bf16 copy) ------------------------------
      uint32_t wn[8];  // the next tile's master, loaded while this tile is processed
      tmem_ld8_raw(tmem + lane_base + kColW1 + chalf * 8, wn);
      for (uint32_t t = 0; t < L.NT; ++t) {
        uint32_t gr[8], wr[8];
        tc::mbar_wait(dtile + t, ph);
        tc::fence_after();
        tmem_ld8_raw(tmem + lane_base + kColDw + t * kHC + chalf * 8, gr);
        tmem_wait_ld2(wn, gr);  // also completes the master load issued last iteration
#pragma unroll
        for (int i = 0; i < 8; ++i) wr[i] = wn[i];
        if (t + 1 < L.NT) tmem_ld8_raw(tmem + lane_base + kColW1 + (t + 1) * kHC + chalf * 8, wn);
        const uint32_t f = t * 128 + quarter * 32 + lane;
        float o[8];
#pragma unroll
        for (uint32_t i = 0; i < 8; ++i) {
          const float w = __uint_as_float(wr[i]), g = __uint_as_float(gr[i]);
          o[i] = chalf * 8 + i < HU ? fmaf(-eta, fmaf(wd, w, g), w) : 0.f;  // padding units stay zero
          if (f < F && !isfinite(o[i])) ubad |= DS_FLAG_OUT_NONFINITE;
        }
        tmem_st8(tmem + lane_base + kColW1 + t * kHC + chalf * 8, o);
        if (f < F) store_wbf_half(Wbf, f, chalf, o);
        tc::fence_async_smem();
        tc::fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(sgdd + t);
      }
      tmem_wait_st();  // the master's stores (read by this thread again: next step or exchange)
      // ---- W2 / b1 / b2 SGD, off the path to the next forward: warps 0, 1, 4, 5 — the
      // ones that write the next step's activations and arrive on a1rdy, so their W2c /
      // b1 updates are ordered before the next logits MMA and tanh -------------------------
      if (warp < 2 || warp == 4 || warp == 5) {
        const uint32_t gi = ((warp & 1u) | ((warp >> 2) << 1)) * 32 + lane;  // 0..127
        for (uint32_t o = gi; o < kHC * C + kHC + C; o += 128) {
          float g0 = 0.f, g1 = 0.f;
          float* dst;
          if (o < kHC * C) {  // own W2 column entry (k, j) (model.cpp:219-221)
            const uint32_t k = o >> 4, j = o & 15;
            if (j >= HU) continue;
#pragma unroll
            for (int r = 0; r < kBM; r += 2) {
              g0 = fmaf(D2(r, k), A1c[a1c_idx(r, j)], g0);
              g1 = fmaf(D2(r + 1, k), A1c[a1c_idx(r + 1, j)], g1);
            }
            dst = W2cc + w2c_idx(k, j);
          } else if (o < kHC * C + kHC) {  // own b1
            const uint32_t j = o - kHC * C;
            if (j >= HU) continue;
#pragma unroll
            for (int r = 0; r < kBM; r += 2) g0 += D1[r * 17 + j], g1 += D1[(r + 1) * 17 + j];
            dst = b1c + j;
          } else {  // b2, replicated in every CTA (same arithmetic)
            const uint32_t k = o - kHC * C - kHC;
#pragma unroll
            for (int r = 0; r < kBM; r += 2) g0 += D2(r, k), g1 += D2(r + 1, k);
            dst = b2s + k;
          }
          const float w = *dst;
          const float out = fmaf(-eta, fmaf(wd, w, g0 + g1), w);
          if (!isfinite(out)) ubad |= DS_FLAG_OUT_NONFINITE;
          *dst = out;
        }
        tc::fence_async_smem();  // W2c is the next step's logits operand
        named_sync(kBarAct, 128);  // b1 / W2c complete before any of the four warps' next tanh
      }
      ubad = __reduce_or_sync(0xffffffffu, ubad);
      if (ubad && lane == 0) atomicOr(&s_bad, ubad);
      TSTAMP_MAIN(A.prof, step, 6, rank);
      // ---- TrainLog row, exchange --------------------------------------------------------
      if (tid == 0 && rank == 0) {
        const PolicyTc& pl = s_pol;
        const unsigned long long row = it0 + step;
        if (row < A.log.cap) {
          A.log.loss[row] = s_loss;
          A.log.cum[row] = pl.cum;
          A.log.exchanged[row] = static_cast<uint8_t>(pl.fire);
          A.log.period[row] = pl.period;
        }
        if (A.ring_loss) A.ring_loss[step] = s_loss;
        if (A.ring && A.ring_consumed)  // every CTA's gathers of this step's slot have landed
          // relaxed: nothing written before needs to be visible to the host with it (a system
          // fence here would stall this warp for a PCIe round trip every step)
          asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(A.ring_consumed), "l"(step + 1) : "memory");
      }
      done = step + 1;
      if (s_pol.fire && A.has_master) {
        csync();  // every warp's SGD done before the exchange reads the master
        TSTAMP_X(A.prof, step, 0, rank);
        const ShardTable& T = A.table;
        uint64_t tk = kNoTicket;
        if (A.tickets) {
          tk = A.tickets[xcount];
        } else if (A.ticket_src) {  // Locked: CTA 0 takes the next ticket and sends it to the peers
          if (rank == 0) {
            if (tid == 0) s_ticket = atomicAdd_system(A.ticket_src, 1ull);
            csync();
            if (tid > 0 && tid < NC)
              st_async16(b2in, ebar, tid, make_float4(__uint_as_float(static_cast<uint32_t>(s_ticket)),
                                                       __uint_as_float(static_cast<uint32_t>(s_ticket >> 32)), 0.f, 0.f));
          } else {
            if (tid == 0) mbar_expect_tx(ebar, 16);
            tc::mbar_wait(ebar, eph);
            if (tid == 0)
              s_ticket = static_cast<unsigned long long>(__float_as_uint(b2in[0])) |
                         (static_cast<unsigned long long>(__float_as_uint(b2in[1])) << 32);
          }
          if (rank != 0) eph ^= 1;
          csync();
          tk = s_ticket;
        }
        const bool ordered = tk != kNoTicket;
        if (ordered && tid == 0) {
          bool ok = true;
          for (int s = 0; s < T.n && ok; ++s) {
            ok = wait_seq_eq(reinterpret_cast<const uint64_t*>(&T.flags[s]->seq), tk, 64);
            if (!ok) atomicAdd_system(&T.flags[s]->timeouts, 1ull);
          }
          if (!ok) atomicOr(&s_bad, DS_FLAG_TICKET_TIMEOUT), atomicOr(&st->flags, DS_FLAG_TICKET_TIMEOUT);
        }
        // ordered exchanges release the next ticket only after every CTA's slice is written
        // ("slice done" messages to CTA 0 + system fences); LockFree needs neither
        if (rank == 0 && tid == 0 && NC > 1 && ordered) mbar_expect_tx(cbar, (NC - 1) * 16);
        if (rank != 0 && tid == 0 && NC > 1) mbar_expect_tx(ebar, ((C + 3) / 4) * 16);
        csync();
        TSTAMP_X(A.prof, step, 1, rank);
        const float a = A.alpha;
        const bool one_shard = T.n == 1;
        float* const c0p = T.ptr[0];
        auto center = [&](uint64_t g) -> float* {
          if (one_shard) return c0p + g;  // the whole center on this GPU
          int s = 0;
          while (s + 1 < T.n && g >= T.begin[s + 1]) ++s;
          return T.ptr[s] + (g - T.begin[s]);
        };
        // the small slices (own W2 columns, own b1, b2 on CTA 0): thread tid < nsmall owns one
        const uint32_t nsmall = C * HU + HU + (rank == 0 ? C : 0u);
        auto small_slice = [&](float*& mp, float*& wp) {
          if (tid < C * HU) {
            const uint32_t k = tid / HU, j = tid - k * HU;
            mp = center(w2o + static_cast<uint64_t>(k) * H + u0 + j);
            wp = W2cc + w2c_idx(k, j);
          } else if (tid < C * HU + HU) {
            mp = center(b1o + u0 + (tid - C * HU));
            wp = b1c + (tid - C * HU);
          } else {
            mp = center(b2o + (tid - C * HU - HU));
            wp = b2s + (tid - C * HU - HU);
          }
        };
        if (!(s_bad & DS_FLAG_TICKET_TIMEOUT) && (F & 3u) == 0 && HU > 0) {
          // own W1 rows: the HU center rows (contiguous, F floats each; split where a shard
          // boundary — 32-float aligned — crosses a row, the remote pieces over NVLink) come
          // in by TMA bulk copies into this step's X buffer (free: dW1(step) is done and
          // step+2 is staged only after the next R phase), are updated in place next to the
          // TMEM master, and go back by bulk stores / bulk f32 reductions — one latency each
          // way instead of a dependent load round per tile pair
          const uint64_t g0 = w1o + static_cast<uint64_t>(u0) * F;
          float* cst = reinterpret_cast<float*>(Xbuf(static_cast<uint32_t>(step & 1)));
          // row j's pieces: [lo, hi) of the global vector inside shard k (one piece, the
          // whole row, for a one-GPU center). mode 0: load, 1: store, 2: reduce-add
          auto pieces = [&](int mode) {
#pragma unroll 1
            for (uint32_t j = 0; j < HU; ++j) {
              const uint64_t r0 = g0 + static_cast<uint64_t>(j) * F;
#pragma unroll
              for (int k = 0; k < kMaxShards; ++k) {  // static indices: the table stays in the parameter bank
                if (k >= T.n) break;
                const uint64_t b0 = one_shard ? 0 : T.begin[k], b1 = one_shard ? ~0ull : T.begin[k + 1];
                const uint64_t lo = r0 > b0 ? r0 : b0, hi = r0 + F < b1 ? r0 + F : b1;
                if (lo >= hi) continue;
                float* g = (one_shard ? c0p : T.ptr[k]) + (lo - b0);
                float* sp = cst + j * F + (lo - r0);
                const uint32_t bytes = static_cast<uint32_t>(hi - lo) * 4u;
                if (mode == 0)
                  bulk_g2s(sp, g, bytes, cxbar);
                else if (mode == 1)
                  bulk_s2g(g, sp, bytes);
                else
                  bulk_add_s2g(g, sp, bytes);
              }
            }
          };
          if (tid == 0) {
            mbar_expect_tx(cxbar, HU * F * 4);
            if (one_shard) {
              for (uint32_t j = 0; j < HU; ++j) bulk_g2s(cst + j * F, c0p + g0 + static_cast<uint64_t>(j) * F, F * 4, cxbar);
            } else {
              pieces(0);
            }
          }
          float* smp = nullptr;
          float* swp = nullptr;
          float smv = 0.f;
          if (tid < nsmall) {  // the small slice's center load overlaps the bulk copies
            small_slice(smp, swp);
            smv = ld_center(smp);
          }
          tc::mbar_wait(cxbar, cxph);
          cxph ^= 1;
          TSTAMP_X(A.prof, step, 6, rank);
          for (uint32_t t = 0; t < L.NT; ++t) {
            const uint32_t f = t * 128 + quarter * 32 + lane;
            float o[8];
            tmem_ld8(tmem + lane_base + kColW1 + t * kHC + chalf * 8, o);
            if (f < F) {
#pragma unroll
              for (uint32_t i = 0; i < 8; ++i) {
                const uint32_t j = chalf * 8 + i;
                if (j < HU) {  // elastic_elem: e = a (w - m); w' = w - e; m' = m + e
                  const float e = fmul(a, fsub(o[i], cst[j * F + f]));
                  o[i] = fsub(o[i], e);
                  cst[j * F + f] = ordered ? fadd(cst[j * F + f], e) : e;
                }
              }
            }
            tmem_st8(tmem + lane_base + kColW1 + t * kHC + chalf * 8, o);
            if (f < F) store_wbf_half(Wbf, f, chalf, o);
          }
          tmem_wait_st();
          TSTAMP_X(A.prof, step, 7, rank);
          if (tid < nsmall) {
            const float e = fmul(a, fsub(*swp, smv));
            *swp = fsub(*swp, e);
            if (ordered)
              *smp = fadd(smv, e);
            else
              atomicAdd_system(smp, e);  // LockFree: the increment is never lost (m' = m + e when alone)
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the updates, to the bulk stores
          csync();
          if (tid == 0) {
            // ordered: the new rows (this worker holds the center exclusively); LockFree: the
            // increments e as bulk f32 reductions — concurrent workers' exchanges add up
            // instead of overwriting each other (a lone writer gets m + e, as elastic_elem)
            if (one_shard) {
              for (uint32_t j = 0; j < HU; ++j) {
                float* dst = c0p + g0 + static_cast<uint64_t>(j) * F;
                if (ordered)
                  bulk_s2g(dst, cst + j * F, F * 4);
                else
                  bulk_add_s2g(dst, cst + j * F, F * 4);
              }
            } else {
              pieces(ordered ? 1 : 2);
            }
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            if (ordered)  // written before the next ticket is released
              asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
            else  // the X buffer read out (it is restaged after the next R phase)
              asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          }
          TSTAMP_X(A.prof, step, 8, rank);
        } else if (!(s_bad & DS_FLAG_TICKET_TIMEOUT)) {
          // own W1 rows: thread = feature of a tile (its TMEM lane), 8 units (its column
          // half); per unit the center row is contiguous in f (coalesced). Two tiles per
          // round: all 16 center loads of a thread are issued before any update.
          const uint64_t g0 = w1o + static_cast<uint64_t>(u0) * F;
          for (uint32_t t0 = 0; t0 < L.NT; t0 += 2) {
            float mv[2][8];
#pragma unroll
            for (uint32_t h = 0; h < 2; ++h) {  // unconditional loads (out-of-range lanes read
              const uint32_t f = (t0 + h) * 128 + quarter * 32 + lane;  // element 0): all in flight
              const bool fin = t0 + h < L.NT && f < F;
#pragma unroll
              for (uint32_t i = 0; i < 8; ++i) {
                const uint32_t j = chalf * 8 + i;
                const uint64_t g = (fin && j < HU) ? g0 + static_cast<uint64_t>(j) * F + f : g0;
                mv[h][i] = ld_center(center(g));
              }
            }
#pragma unroll
            for (uint32_t h = 0; h < 2; ++h) {
              if (t0 + h >= L.NT) break;
              const uint32_t t = t0 + h, f = t * 128 + quarter * 32 + lane;
              float o[8];
              tmem_ld8(tmem + lane_base + kColW1 + t * kHC + chalf * 8, o);
#pragma unroll
              for (uint32_t i = 0; i < 8; ++i) {
                const uint32_t j = chalf * 8 + i;
                if (f < F && j < HU) {
                  const float e = fmul(a, fsub(o[i], mv[h][i]));
                  o[i] = fsub(o[i], e);
                  float* cp = center(g0 + static_cast<uint64_t>(j) * F + f);
                  if (ordered)
                    *cp = fadd(mv[h][i], e);
                  else
                    atomicAdd_system(cp, e);  // LockFree: increments add up across workers / GPUs
                }
              }
              tmem_st8(tmem + lane_base + kColW1 + t * kHC + chalf * 8, o);
              if (f < F) store_wbf_half(Wbf, f, chalf, o);
              if (h == 0 && t0 == 0) TSTAMP_X(A.prof, step, 6, rank);
            }
            if (t0 == 0) TSTAMP_X(A.prof, step, 7, rank);
            if (t0 == 2) TSTAMP_X(A.prof, step, 8, rank);
          }
          tmem_wait_st();
          // the small slices: own W2 columns, own b1, b2 (CTA 0): loads first, then updates
          TSTAMP_X(A.prof, step, 2, rank);
          if (tid < nsmall) {
            float* mp;
            float* wp;
            small_slice(mp, wp);
            const float mv0 = ld_center(mp);
            const float e = fmul(a, fsub(*wp, mv0));
            *wp = fsub(*wp, e);
            if (ordered)
              *mp = fadd(mv0, e);
            else
              atomicAdd_system(mp, e);
          }
        }
        tc::fence_async_smem();
        tc::fence_before();
        csync();
        // this CTA's center writes (cumulative over the barrier); a center that only this GPU
        // touches needs gpu scope — the system-scope fences cost ~4 us per ordered exchange
        if (tid == 0 && ordered) A.center_local ? __threadfence() : __threadfence_system();
        TSTAMP_X(A.prof, step, 3, rank);
        if (NC > 1) {
          if (rank != 0) {
            if (tid == 0 && ordered) st_async16(b2in + kMaxC - 4, cbar, 0, make_float4(0.f, 0.f, 0.f, 0.f));  // "slice done"
            tc::mbar_wait(ebar, eph);  // CTA 0's exchanged b2
            if (tid < C) b2s[tid] = b2in[tid];
            eph ^= 1;
          } else {
            if (ordered) {
              tc::mbar_wait(cbar, eph);  // every peer's slice done
              eph ^= 1;
            }
            TSTAMP_X(A.prof, step, 4, rank);
            if (tid < (C + 3) / 4 * (NC - 1)) {  // b2 lives in every CTA
              const uint32_t q = 1 + tid / ((C + 3) / 4), pc = tid % ((C + 3) / 4);
              float v[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) v[e] = pc * 4 + e < C ? b2s[pc * 4 + e] : 0.f;
              st_async16(b2in + pc * 4, ebar, q, make_float4(v[0], v[1], v[2], v[3]));
            }
          }
        }
        if (rank == 0 && tid == 0 && !(s_bad & DS_FLAG_TICKET_TIMEOUT)) {
          if (ordered) {
            if (A.center_local) {
              __threadfence();
              T.flags[0]->exchanges += 1;
              asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(&T.flags[0]->seq), "l"(tk + 1) : "memory");
            } else {
              __threadfence_system();
              T.flags[0]->exchanges += 1;
              __threadfence_system();
              for (int s = 0; s < T.n; ++s) st_release_sys(reinterpret_cast<uint64_t*>(&T.flags[s]->seq), tk + 1);
            }
          } else {
            atomicAdd_system(&T.flags[0]->exchanges, 1ull);
          }
        }
        ++xcount;
        csync();
        TSTAMP_X(A.prof, step, 5, rank);
        if (tid == 0) tc::mbar_arrive(exdone);  // the MMA warp issues forward(s+1) now
      }
      TSTAMP_MAIN(A.prof, step, 7, rank);
      ph ^= 1;
    }
    if (tid == 0) *reinterpret_cast<volatile uint32_t*>(&s_quit) = 1;  // the other warps stop waiting
  }

  // ---- write back the parameters, the policy state, errors --------------------------
  if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // LockFree center stores landed
  __syncthreads();
  tc::fence_after();
  if (warp < kCW) {  // own W1 rows from the TMEM master
    for (uint32_t t = 0; t < L.NT; ++t) {
      const uint32_t f = t * 128 + quarter * 32 + lane;
      float w[8];
      tmem_ld8(tmem + lane_base + kColW1 + t * kHC + chalf * 8, w);
      if (f < F) {
#pragma unroll
        for (uint32_t i = 0; i < 8; ++i) {
          const uint32_t j = chalf * 8 + i;
          if (j < HU) Pout[w1o + static_cast<uint64_t>(u0 + j) * F + f] = w[i];
        }
      }
    }
  }
  if (tid < HU) Pout[b1o + u0 + tid] = b1c[tid];
  for (uint32_t i = tid; i < C * HU; i += kTT) {
    const uint32_t k = i / HU, j = i - k * HU;
    Pout[w2o + static_cast<uint64_t>(k) * H + u0 + j] = W2cc[w2c_idx(k, j)];
  }
  if (rank == 0 && tid < C) Pout[b2o + tid] = b2s[tid];
  tc::fence_before();
  __syncthreads();
  cluster_sync();  // every CTA's flags and parameters are out; no DSMEM traffic after this
  if (rank == 0 && tid == 0) {
    const uint32_t fl = *reinterpret_cast<volatile uint32_t*>(&st->flags);
    if (fl || failed) {
      st->err = fl ? fl : DS_FLAG_OUT_NONFINITE;
      st->bad_iter = it0 + (bad_iter_step ? bad_iter_step : done);
    }
    st->cum = s_pol.cum;
    st->since = s_pol.since;
    st->fire = s_pol.fire;
    st->period = s_pol.period;
    st->loss = s_loss;
    st->iter = it0 + done;
    st->exchanges += xcount;
  }
  if (A.prof && rank == 0 && tid == 0) {  // SM clock over the launch: cycles / ns
    A.prof[A.steps * kProfSlots + 0] = globaltimer_ns() - gt0;
    A.prof[A.steps * kProfSlots + 1] = static_cast<unsigned long long>(clock64() - clk0);
  }
  if (warp == 0) tc::tmem_free<kTmemCols>(tmem);
}

}  // namespace

int tc_cluster(const ModelInfo& m) { return static_cast<int>((m.hidden[0] + kHC - 1) / kHC); }

size_t tc_smem_bytes(const ModelInfo& m, uint32_t batch) {
  return tc_smem(m.n_features, batch, m.n_classes, static_cast<uint32_t>(tc_cluster(m))).total + 1024;
}

int tc_supported(const ModelInfo& m, uint32_t batch, int device, const char** why) {
  auto no = [&](const char* w) {
    if (why) *why = w;
    return DS_E_CONTRACT;
  };
  if (m.kind != 1 || m.hidden.size() != 1) return no("the tensor-core step covers one-hidden-layer MLPs");
  if (m.hidden[0] > static_cast<uint32_t>(kHC * kMaxNC)) return no("more than 256 hidden units");
  if (m.n_classes > static_cast<uint32_t>(kMaxC)) return no("more than 16 classes");
  if (batch > static_cast<uint32_t>(kBM)) return no("batch_size above 32");
  if (m.n_features > 896) return no("more than 896 features");  // 7 dW1 tiles + 7 master tiles in TMEM
  int optin = 0;
  if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device) != cudaSuccess) optin = 227 * 1024;
  if (tc_smem_bytes(m, batch) > static_cast<size_t>(optin)) return no("batch rows x features do not fit in shared memory");
  int major = 0;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, device);
  if (major != 10) return no("tcgen05 needs an sm_100 device");
  return DS_OK;
}

namespace {
// f32 rows [rows x F] -> bf16 rows [rows x pitch] (zero padded), 8 elements per thread
__global__ void rows_to_bf16_kernel(const float* __restrict__ src, uint64_t rows, uint32_t F,
                                    __nv_bfloat16* __restrict__ dst, uint32_t pitch) {
  const uint32_t q8 = pitch / 8;
  const uint64_t n = rows * q8;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint64_t r = i / q8;
    const uint32_t c0 = static_cast<uint32_t>(i - r * q8) * 8;
    const float* sp = src + r * F;
    float v[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] = c0 + e < F ? sp[c0 + e] : 0.f;
    *reinterpret_cast<uint4*>(dst + r * pitch + c0) =
        make_uint4(pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]), pack_bf16(v[4], v[5]), pack_bf16(v[6], v[7]));
  }
}

PFN_cuTensorMapEncodeTiled_v12000 tc_encode_fn() {
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

}  // namespace

uint32_t tc_pitch(uint32_t F) { return (F + 7) & ~7u; }

int tc_rows_to_bf16(const float* src, uint64_t rows, uint32_t F, void* dst, cudaStream_t s) {
  if (rows == 0) return DS_OK;
  const uint32_t pitch = tc_pitch(F);
  const uint64_t n = rows * (pitch / 8);
  const unsigned grid = static_cast<unsigned>(std::min<uint64_t>((n + 255) / 256, 148 * 8));
  rows_to_bf16_kernel<<<grid, 256, 0, s>>>(src, rows, F, static_cast<__nv_bfloat16*>(dst), pitch);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

// bf16 [rows x pitch] row-major; box = 64 features x 1 row (the gather4 box), SWIZZLE_128B
int tc_make_map(CUtensorMap* m, const void* base, uint64_t rows, uint32_t F) {
  auto fn = tc_encode_fn();
  if (!fn) return set_error(DS_E_CUDA, "tc: cuTensorMapEncodeTiled unavailable");
  const uint32_t pitch = tc_pitch(F);
  const cuuint64_t dims[2] = {pitch, rows};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(pitch) * 2};
  const cuuint32_t box[2] = {64, 1};
  const cuuint32_t es[2] = {1, 1};
  const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_error(DS_E_CUDA, "tc: cuTensorMapEncodeTiled failed (%d)", static_cast<int>(r));
  return DS_OK;
}

int launch_tc_group(const FusedArgs* a, const CUtensorMap* tm, uint32_t n, int nc, cudaStream_t s) {
  if (nc < 1 || nc > kMaxNC) return set_error(DS_E_CONTRACT, "tc: cluster size %d", nc);
  if (n < 1 || n > static_cast<uint32_t>(kMaxGroup)) return set_error(DS_E_CONTRACT, "tc: %u workers per launch (1..%d)", n, kMaxGroup);
  const size_t smem = tc_smem(a[0].F, a[0].B, a[0].C, static_cast<uint32_t>(nc)).total + 1024;
  DS_CUDA_TRY(cudaFuncSetAttribute(mlp_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  if (nc > 8) DS_CUDA_TRY(cudaFuncSetAttribute(mlp_tc_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  static TcLaunch P;  // ~5 KB: kernel parameter, copied at launch
  static std::mutex mu;
  std::lock_guard<std::mutex> lk(mu);
  for (uint32_t i = 0; i < n; ++i) P.maps[i] = tm[i], P.args[i] = a[i];
  P.n = n;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(n * nc);
  cfg.blockDim = dim3(kTT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = nc;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  // co-residency is needed only when workers wait on each other (ordered exchanges:
  // Locked arrival tickets or deterministic tickets); LockFree and master-less groups
  // launch as plain cluster grids (which profilers can also replay)
  bool waits = false;
  for (uint32_t i = 0; i < n; ++i) waits = waits || (a[i].has_master && !a[i].lockfree);
  at[1].id = cudaLaunchAttributeCooperative;
  at[1].val.cooperative = 1;
  cfg.attrs = at;
  cfg.numAttrs = (n > 1 && waits) ? 2 : 1;
  if (n > 1 && waits) {
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, mlp_tc_kernel, &cfg) == cudaSuccess && nclusters < static_cast<int>(n))
      return set_error(DS_E_CONTRACT, "tc: %u workers of %d CTAs do not fit on the GPU at once (max %d)", n, nc, nclusters);
    cudaGetLastError();
  }
  DS_CUDA_TRY(cudaLaunchKernelEx(&cfg, mlp_tc_kernel, P));
  return DS_OK;
}

int launch_tc(const FusedArgs& a, int nc, const CUtensorMap& tm, cudaStream_t s) {
  return launch_tc_group(&a, &tm, 1, nc, s);
}

}  // namespace dsb

void dsb::warm_tc_kernels() { dsb::load_kernels(dsb::mlp_tc_kernel, dsb::rows_to_bf16_kernel); }
