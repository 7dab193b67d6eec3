// sync.cu — synchronous data-parallel training over GPUs, one process per GPU:
//   * synchronous SGD with gradient averaging (simulate_sync, simulator.cpp:156-223);
//   * synchronous EASGD (NOT IN THE REFERENCE; the EASGD paper's synchronous variant).
// The "allreduce" is fused into the update as a worker-ordered reduce-scatter + all-gather
// over NVLink, with no NCCL on the data path:
//
//   reduce-scatter: rank r owns the contiguous, 128-byte aligned slice r of the vector. Its
//     kernel reads every rank's contribution for that slice only (CUDA IPC mappings), sums
//     in f64 in WORKER ORDER k = 0..G-1 (the reference's gsum loop, simulator.cpp:192-200 —
//     a ring/tree allreduce would reorder the additions), applies the update and writes
//     the new slice into its replica and into its published buffer `pub`;
//   all-gather: after every peer published the round, each rank copies the other slices
//     from the peers' `pub` buffers into its replica.
// NVLink traffic per rank and round: 2 (G-1)/G x 4P bytes (one read of the peers' slot
// slices, one read of the peers' published slices), against (G-1) x 4P when every rank
// summed the whole vector. All replicas receive the owner's values, so they stay
// bit-identical.
//
// Round protocol (round r = 1, 2, ..., slots and pubs double-buffered by r % 2):
//   ds_sync_begin: returns this round's slot; no wait (the previous round's all-gather
//     waited for every peer's `sliced`, i.e. every peer finished reading slot r-2 and the
//     pub of r-2 is read by peers before they publish `ready` of r-1);
//   the caller writes its contribution into the slot on the same stream;
//   ds_sync_reduce_update / ds_sync_easgd_update: publish ready = r, wait for every peer's
//     ready, reduce own slice -> replica + pub, publish sliced = r, wait for every peer's
//     sliced, all-gather. Waits are bounded (30 s, then DS_FLAG_TICKET_TIMEOUT).
//
// Single process, several ranks on ONE GPU (ds_sync_*_group): every rank's contribution is
// written before the launch (stream order), so one kernel reduces all slices and writes
// every replica — the same per-element arithmetic with no cross-kernel waiting.
#include <cuda_runtime.h>
#include <stdint.h>
#include <unistd.h>

#include <cstring>
#include <vector>

#include "ds_common.cuh"
#include "ds_cuda.h"

namespace dsb {
namespace {

constexpr int kMaxRanks = 8;
constexpr int kT = 256;

struct alignas(128) SyncFlags {
  unsigned long long ready;   // last round whose slot contribution is complete
  unsigned long long sliced;  // last round whose owned slice is published in pub
  unsigned long long pad[14];
};

struct SyncTable {
  int world;
  uint64_t begin[kMaxRanks + 1];  // slice bounds
  const float* slot[kMaxRanks];   // each rank's [2][dim] contribution slots
  const float* pub[kMaxRanks];    // each rank's [2][dim] published slices
  SyncFlags* flags[kMaxRanks];
};

__device__ __forceinline__ void st_release_sys_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
// bounded wait for every peer's word >= r; false after 30 s
__device__ bool wait_all(const SyncTable& t, int self, unsigned long long r, bool sliced) {
  const unsigned long long t0 = globaltimer_ns();
  for (int k = 0; k < t.world; ++k) {
    if (k == self) continue;
    const unsigned long long* w = sliced ? &t.flags[k]->sliced : &t.flags[k]->ready;
    while (ld_acquire_sys_u64(w) < r) {
      if (globaltimer_ns() - t0 > kSeqTimeoutNs) return false;
      __nanosleep(32);
    }
  }
  return true;
}

// SGD mode: contribution = gradient; x' = sgd_step(x, f32(gsum / n) (+ wd x), eta)
__device__ __forceinline__ float sgd_elem(double gsum, int n, float x, float eta, float wd, uint32_t& bad) {
  float g = static_cast<float>(__ddiv_rn(gsum, static_cast<double>(n)));
  if (wd > 0.0f) g = fadd(g, fmul(wd, x));       // simulator.cpp:205-207
  if (!isfinite(x)) bad |= DS_FLAG_X_NONFINITE;  // sgd_step's checks (param_vector.cpp:21-39)
  if (!isfinite(g)) bad |= DS_FLAG_G_NONFINITE;
  const float o = fsub(x, fmul(eta, g));
  if (!isfinite(o)) bad |= DS_FLAG_OUT_NONFINITE;
  return o;
}

// Reduce-scatter for ranks [r0, r1) (their slices) + (EASGD) the workers' elastic steps.
// mode 0: SGD (replica = params); mode 1: EASGD (replica = center; the slot holds x_k and,
// at +dpad, the OLD center; worker = x_k's home, updated x_k' = x_k - e_k). group != 0:
// single-process group (all replicas local, written directly, no flags).
struct RoundArgs {
  SyncTable t;
  int self, r0, r1, mode, group, vec;
  unsigned long long round;
  uint64_t dim, dpad;
  uint64_t off;                 // slot offset of this round's parity ((r % 2) * 2 dpad)
  uint64_t poff;                // pub offset of this round's parity ((r % 2) * dpad)
  float* replica[kMaxRanks];    // group: every rank's replica; else [0] = own
  float* worker[kMaxRanks];     // EASGD: every rank's worker parameters (group) or [0] = own
  float eta, wd, alpha;
  uint32_t* flags;
};

template <int V>
__device__ __forceinline__ void ldv(const float* p, float (&v)[V]) {
  if constexpr (V == 4) {
    const float4 t = __ldcg(reinterpret_cast<const float4*>(p));
    v[0] = t.x, v[1] = t.y, v[2] = t.z, v[3] = t.w;
  } else {
    v[0] = __ldcg(p);
  }
}
template <int V>
__device__ __forceinline__ void stv(float* p, const float (&v)[V]) {
  if constexpr (V == 4)
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  else
    *p = v[0];
}

// V consecutive elements from i of the owned slices
template <int V>
__device__ __forceinline__ void reduce_elems(const RoundArgs& a, uint64_t i, uint32_t& bad) {
  const SyncTable& t = a.t;
  float s[kMaxRanks][V];
#pragma unroll
  for (int k = 0; k < kMaxRanks; ++k)  // every rank's contribution first: all loads in flight
    if (k < t.world) ldv<V>(t.slot[k] + a.off + i, s[k]);
  float c[V], o[V];
  ldv<V>(a.replica[0] + i, c);  // replicas are identical before the round
#pragma unroll
  for (int j = 0; j < V; ++j) {
    double acc = 0.0;  // simulator.cpp:192: std::vector<double> gsum(P, 0.0), worker order
    if (a.mode == 0) {
#pragma unroll
      for (int k = 0; k < kMaxRanks; ++k)
        if (k < t.world) acc = dadd(acc, static_cast<double>(s[k][j]));
      o[j] = sgd_elem(acc, t.world, c[j], a.eta, a.wd, bad);
    } else {  // e_k = f32(alpha * f32(x_k - c)); c' = c + f32(sum_k e_k)
#pragma unroll
      for (int k = 0; k < kMaxRanks; ++k)
        if (k < t.world) acc = dadd(acc, static_cast<double>(fmul(a.alpha, fsub(s[k][j], c[j]))));
      o[j] = fadd(c[j], static_cast<float>(acc));
      if (!isfinite(o[j])) bad |= DS_FLAG_OUT_NONFINITE;
    }
  }
  if (a.group) {
#pragma unroll
    for (int k = 0; k < kMaxRanks; ++k)
      if (k < t.world) stv<V>(a.replica[k] + i, o);
  } else {
    stv<V>(a.replica[0] + i, o);
    stv<V>(const_cast<float*>(t.pub[a.self]) + a.poff + i, o);
  }
}
// EASGD worker step x_k' = x_k - f32(alpha * f32(x_k - c_old)) for V elements from i
template <int V>
__device__ __forceinline__ void worker_elems(const RoundArgs& a, int k, uint64_t i) {
  const float* xs = a.t.slot[a.group ? k : a.self] + a.off;
  float x[V], c[V], o[V];
  ldv<V>(xs + i, x);
  ldv<V>(xs + a.dpad + i, c);
#pragma unroll
  for (int j = 0; j < V; ++j) o[j] = fsub(x[j], fmul(a.alpha, fsub(x[j], c[j])));
  stv<V>(a.worker[k] + i, o);
}

__global__ void __launch_bounds__(kT) round_kernel(RoundArgs a) {
  const SyncTable& t = a.t;
  __shared__ int s_ok;
  if (!a.group && t.world > 1) {
    if (threadIdx.x == 0) {
      if (blockIdx.x == 0) {
        __threadfence_system();  // this rank's contribution (earlier kernels) first
        st_release_sys_u64(&t.flags[a.self]->ready, a.round);
      }
      s_ok = wait_all(t, a.self, a.round, false);
    }
    __syncthreads();
    if (!s_ok) {
      if (threadIdx.x == 0 && a.flags) atomicOr(a.flags, DS_FLAG_TICKET_TIMEOUT);
      return;
    }
  }
  uint32_t bad = 0;
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  // ---- reduce-scatter: the owned slices (slice starts are multiples of 32 elements) ----
  const uint64_t lo = t.begin[a.r0], hi = t.begin[a.r1];
  const uint64_t hv = a.vec ? lo + ((hi - lo) & ~3ull) : lo;
  for (uint64_t i = lo + 4 * tid; i < hv; i += 4 * stride) reduce_elems<4>(a, i, bad);
  for (uint64_t i = hv + tid; i < hi; i += stride) reduce_elems<1>(a, i, bad);
  // ---- EASGD: every local worker's elastic step with the OLD center, all elements ------
  if (a.mode == 1) {
    const uint64_t dv = a.vec ? (a.dim & ~3ull) : 0;
    for (int k = 0; k < (a.group ? t.world : 1); ++k) {
      for (uint64_t i = 4 * tid; i < dv; i += 4 * stride) worker_elems<4>(a, k, i);
      for (uint64_t i = dv + tid; i < a.dim; i += stride) worker_elems<1>(a, k, i);
    }
  }
  const uint32_t any = __reduce_or_sync(0xffffffffu, bad);
  if (any && a.flags && (threadIdx.x & 31) == 0) atomicOr(a.flags, any);
}

// all-gather half of a multi-process round: publish sliced, wait for every peer, copy the
// peers' slices into the replica (separate launches: every CTA of the reduce kernel must
// have written its pub slice before `sliced` is published)
__global__ void publish_sliced_kernel(SyncFlags* own, unsigned long long r) {
  __threadfence_system();
  st_release_sys_u64(&own->sliced, r);
}
__global__ void __launch_bounds__(kT) gather_kernel(SyncTable t, int self, unsigned long long r, uint64_t poff,
                                                    float* replica, int vec, uint32_t* flags) {
  __shared__ int s_ok;
  if (threadIdx.x == 0) s_ok = wait_all(t, self, r, true);
  __syncthreads();
  if (!s_ok) {
    if (threadIdx.x == 0 && flags) atomicOr(flags, DS_FLAG_TICKET_TIMEOUT);
    return;
  }
  const uint64_t tid = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (int k = 0; k < t.world; ++k) {
    if (k == self) continue;
    const uint64_t lo = t.begin[k], hi = t.begin[k + 1];
    const float* p = t.pub[k] + poff;
    const uint64_t nv = vec ? (hi - lo) / 4 : 0;  // float4 units
    const float4* p4 = reinterpret_cast<const float4*>(p + lo);
    float4* d4 = reinterpret_cast<float4*>(replica + lo);
    uint64_t u = tid;
    for (; u + 3 * stride < nv; u += 4 * stride) {  // four 16-byte loads in flight per thread
      const float4 v0 = __ldcg(p4 + u), v1 = __ldcg(p4 + u + stride), v2 = __ldcg(p4 + u + 2 * stride),
                   v3 = __ldcg(p4 + u + 3 * stride);
      d4[u] = v0, d4[u + stride] = v1, d4[u + 2 * stride] = v2, d4[u + 3 * stride] = v3;
    }
    for (; u < nv; u += stride) d4[u] = __ldcg(p4 + u);
    for (uint64_t i = lo + 4 * nv + tid; i < hi; i += stride) replica[i] = __ldcg(p + i);
  }
}

// NVLink read probe (the all-gather's access pattern): n floats split over every peer's
// slot region, copied into dst. The CTAs are dealt round-robin to the peers, starting at a
// rank-dependent peer, so every link is busy at once (a peer-after-peer walk would have all
// ranks read the same peer together).
__global__ void __launch_bounds__(kT) peer_read_kernel(SyncTable t, int self, uint64_t per, float* dst) {
  const uint32_t np = static_cast<uint32_t>(t.world - 1);
  const uint32_t q = blockIdx.x % np, cq = blockIdx.x / np, nq = gridDim.x / np;
  if (cq >= nq) return;
  const int k = (self + 1 + static_cast<int>(q)) % t.world;  // never self
  const float4* p4 = reinterpret_cast<const float4*>(t.slot[k]);
  float4* d4 = reinterpret_cast<float4*>(dst + q * per);
  const uint64_t nv = per / 4;
  const uint64_t stride = static_cast<uint64_t>(nq) * blockDim.x;
  uint64_t u = static_cast<uint64_t>(cq) * blockDim.x + threadIdx.x;
  for (; u + 3 * stride < nv; u += 4 * stride) {
    const float4 v0 = __ldcg(p4 + u), v1 = __ldcg(p4 + u + stride), v2 = __ldcg(p4 + u + 2 * stride),
                 v3 = __ldcg(p4 + u + 3 * stride);
    d4[u] = v0, d4[u + stride] = v1, d4[u + 2 * stride] = v2, d4[u + 3 * stride] = v3;
  }
  for (; u < nv; u += stride) d4[u] = __ldcg(p4 + u);
}

struct IpcRecord {
  cudaIpcMemHandle_t slots;
  cudaIpcMemHandle_t flags;
  uint64_t dim;
  int32_t rank, world, device, pid;
  uint64_t slots_ptr, flags_ptr;  // same-process ranks use these directly
  uint8_t pad[DS_IPC_RECORD_BYTES - 2 * sizeof(cudaIpcMemHandle_t) - 3 * 8 - 4 * 4];
};
static_assert(sizeof(IpcRecord) == DS_IPC_RECORD_BYTES, "IPC record size");

}  // namespace
}  // namespace dsb

struct ds_sync {
  int device = 0, rank = 0, world = 1;
  uint64_t dim = 0, dpad = 0;         // dpad: dim rounded up to 32 floats (128-byte rows)
  float* slots = nullptr;             // own [2 parities][2 dpad]: contribution (+ EASGD: the old center)
  float* pubs = nullptr;              // own [2][dpad] published slices (same allocation, peer-mapped)
  dsb::SyncFlags* flags = nullptr;    // own ready/sliced words (peer-mapped)
  void* peer_slots[dsb::kMaxRanks] = {};
  void* peer_flags[dsb::kMaxRanks] = {};
  dsb::SyncTable table{};
  bool attached = false;
  unsigned long long round = 0;       // rounds begun
  int ctas = 1;
};

namespace {
inline uint64_t slot_stride(const ds_sync* s) { return 2 * s->dpad; }
inline uint64_t alloc_floats(uint64_t dpad) { return 2 * 2 * dpad + 2 * dpad; }
void set_bounds(ds_sync* s) {
  const uint64_t sl = ((s->dim + s->world - 1) / s->world + 31) & ~31ull;  // 128-byte aligned slices
  for (int k = 0; k <= s->world; ++k) s->table.begin[k] = sl * k < s->dim ? sl * k : s->dim;
  s->table.begin[s->world] = s->dim;
}
inline bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
}  // namespace

extern "C" int ds_sync_create(ds_sync** out, int device, uint64_t dim, int rank, int world) {
  if (!out) return dsb::set_error(DS_E_CONTRACT, "sync: null out");
  if (dim == 0) return dsb::set_error(DS_E_CONTRACT, "sync: dim must be positive");
  if (world < 1 || world > dsb::kMaxRanks || rank < 0 || rank >= world)
    return dsb::set_error(DS_E_CONTRACT, "sync: rank/world out of range (world <= %d)", dsb::kMaxRanks);
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return dsb::set_error(DS_E_CUDA, "sync: no CUDA device");
  if (device < 0 || device >= ndev) return dsb::set_error(DS_E_CONTRACT, "sync: bad device %d", device);
  dsb::DeviceScope ds(device);
  auto* s = new ds_sync();
  s->device = device;
  s->rank = rank;
  s->world = world;
  s->dim = dim;
  s->dpad = (dim + 31) & ~31ull;
  const uint64_t floats = alloc_floats(s->dpad);
  cudaError_t e = cudaMalloc(&s->slots, floats * sizeof(float));
  if (e == cudaSuccess) e = cudaMalloc(&s->flags, sizeof(dsb::SyncFlags));
  if (e == cudaSuccess) e = cudaMemset(s->flags, 0, sizeof(dsb::SyncFlags));
  if (e == cudaSuccess) e = cudaMemset(s->slots, 0, floats * sizeof(float));
  if (e != cudaSuccess) {
    cudaFree(s->slots);
    cudaFree(s->flags);
    delete s;
    return dsb::set_error(e == cudaErrorMemoryAllocation ? DS_E_NOMEM : DS_E_CUDA, "sync: %s", cudaGetErrorString(e));
  }
  s->pubs = s->slots + 2 * slot_stride(s);
  s->table.world = world;
  set_bounds(s);
  for (int k = 0; k < world; ++k) {  // world == 1 needs no attach
    s->table.slot[k] = k == rank ? s->slots : nullptr;
    s->table.pub[k] = k == rank ? s->pubs : nullptr;
    s->table.flags[k] = k == rank ? s->flags : nullptr;
  }
  s->attached = world == 1;
  const uint64_t want = (dim + 1023) / 1024;  // 4 elements per thread
  const uint64_t cap = static_cast<uint64_t>(dsb::sm_count(device)) * 8;
  s->ctas = static_cast<int>(want < cap ? want : cap);
  *out = s;
  return DS_OK;
}

extern "C" int ds_sync_export(ds_sync* s, void* record_out) {
  if (!s || !record_out) return dsb::set_error(DS_E_CONTRACT, "sync_export: null");
  dsb::DeviceScope ds(s->device);
  dsb::IpcRecord r;
  std::memset(&r, 0, sizeof(r));
  DS_CUDA_TRY(cudaIpcGetMemHandle(&r.slots, s->slots));
  DS_CUDA_TRY(cudaIpcGetMemHandle(&r.flags, s->flags));
  r.dim = s->dim;
  r.rank = s->rank;
  r.world = s->world;
  r.device = s->device;
  r.pid = static_cast<int32_t>(getpid());
  r.slots_ptr = reinterpret_cast<uint64_t>(s->slots);
  r.flags_ptr = reinterpret_cast<uint64_t>(s->flags);
  std::memcpy(record_out, &r, sizeof(r));
  return DS_OK;
}

extern "C" int ds_sync_attach(ds_sync* s, const void* records) {
  if (!s || !records) return dsb::set_error(DS_E_CONTRACT, "sync_attach: null");
  if (s->world == 1) return DS_OK;
  if (s->attached) return dsb::set_error(DS_E_STATE, "sync_attach: already attached");
  dsb::DeviceScope ds(s->device);
  const auto* recs = static_cast<const dsb::IpcRecord*>(records);
  for (int k = 0; k < s->world; ++k) {
    const dsb::IpcRecord& r = recs[k];
    if (r.rank != k || r.world != s->world || r.dim != s->dim)
      return dsb::set_error(DS_E_CONTRACT, "sync_attach: record %d does not match this group", k);
  }
  for (int k = 0; k < s->world; ++k) {
    const dsb::IpcRecord& r = recs[k];
    if (k == s->rank) continue;
    void* ps = nullptr;
    void* pf = nullptr;
    if (r.pid == static_cast<int32_t>(getpid())) {  // a rank of this process: plain pointers
      ps = reinterpret_cast<void*>(r.slots_ptr);
      pf = reinterpret_cast<void*>(r.flags_ptr);
      if (r.device != s->device) {
        const cudaError_t pe = cudaDeviceEnablePeerAccess(r.device, 0);
        if (pe == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        else DS_CUDA_TRY(pe);
      }
    } else {
      DS_CUDA_TRY(cudaIpcOpenMemHandle(&ps, r.slots, cudaIpcMemLazyEnablePeerAccess));
      DS_CUDA_TRY(cudaIpcOpenMemHandle(&pf, r.flags, cudaIpcMemLazyEnablePeerAccess));
      s->peer_slots[k] = ps;
      s->peer_flags[k] = pf;
    }
    s->table.slot[k] = static_cast<const float*>(ps);
    s->table.pub[k] = static_cast<const float*>(ps) + 2 * slot_stride(s);
    s->table.flags[k] = static_cast<dsb::SyncFlags*>(pf);
  }
  s->attached = true;
  return DS_OK;
}

extern "C" int ds_sync_begin(ds_sync* s, float** grad_slot, void* stream) {
  (void)stream;  // no wait: see the round protocol in the header comment
  if (!s || !grad_slot) return dsb::set_error(DS_E_CONTRACT, "sync_begin: null");
  if (!s->attached) return dsb::set_error(DS_E_STATE, "sync_begin: group not attached");
  const unsigned long long r = ++s->round;
  *grad_slot = s->slots + (r & 1) * slot_stride(s);
  return DS_OK;
}

namespace {
dsb::RoundArgs round_args(const ds_sync* s, int mode, float eta, float wd, float alpha, uint32_t* flags) {
  dsb::RoundArgs a{};
  a.t = s->table;
  a.mode = mode;
  a.round = s->round;
  a.dim = s->dim;
  a.dpad = s->dpad;
  a.off = (s->round & 1) * slot_stride(s);
  a.poff = (s->round & 1) * s->dpad;
  a.eta = eta;
  a.wd = wd;
  a.alpha = alpha;
  a.flags = flags;
  return a;
}

int round_multi(ds_sync* s, int mode, float* replica, float* worker, float eta, float wd, float alpha, uint32_t* flags,
                cudaStream_t st) {
  dsb::RoundArgs a = round_args(s, mode, eta, wd, alpha, flags);
  a.self = s->rank;
  a.r0 = s->rank;
  a.r1 = s->rank + 1;
  a.group = 0;
  a.replica[0] = replica;
  a.worker[0] = worker;
  a.vec = al16(replica) && (!worker || al16(worker));
  dsb::round_kernel<<<s->ctas, dsb::kT, 0, st>>>(a);
  DS_CUDA_TRY(cudaGetLastError());
  if (s->world > 1) {
    dsb::publish_sliced_kernel<<<1, 1, 0, st>>>(s->flags, s->round);
    dsb::gather_kernel<<<s->ctas, dsb::kT, 0, st>>>(s->table, s->rank, s->round, a.poff, replica, a.vec, flags);
    DS_CUDA_TRY(cudaGetLastError());
  }
  return DS_OK;
}
}  // namespace

extern "C" int ds_sync_reduce_update(ds_sync* s, float* params, float eta, float wd, uint32_t* flags_dev,
                                     void* stream) {
  if (!s || !params) return dsb::set_error(DS_E_CONTRACT, "sync_reduce_update: null");
  if (!s->attached || s->round == 0) return dsb::set_error(DS_E_STATE, "sync_reduce_update: no round begun");
  if (!(eta > 0.0f)) return dsb::set_error(DS_E_CONTRACT, "sgd_step: eta must be positive");
  dsb::DeviceScope ds(s->device);
  return round_multi(s, 0, params, nullptr, eta, wd, 0.f, flags_dev, dsb::as_stream(stream));
}

extern "C" int ds_sync_easgd_update(ds_sync* s, float* worker, float* center, float alpha, uint32_t* flags_dev,
                                    void* stream) {
  if (!s || !worker || !center) return dsb::set_error(DS_E_CONTRACT, "sync_easgd_update: null");
  if (!s->attached) return dsb::set_error(DS_E_STATE, "sync_easgd_update: group not attached");
  if (!(alpha > 0.0f && alpha < 1.0f)) return dsb::set_error(DS_E_CONTRACT, "easgd: alpha must be in (0,1)");
  dsb::DeviceScope ds(s->device);
  cudaStream_t st = dsb::as_stream(stream);
  float* slot = nullptr;
  DS_TRY(ds_sync_begin(s, &slot, stream));
  // the contribution is the worker vector; the old center rides at +dpad
  DS_CUDA_TRY(cudaMemcpyAsync(slot, worker, s->dim * sizeof(float), cudaMemcpyDeviceToDevice, st));
  DS_CUDA_TRY(cudaMemcpyAsync(slot + s->dpad, center, s->dim * sizeof(float), cudaMemcpyDeviceToDevice, st));
  return round_multi(s, 1, center, worker, 0.f, 0.f, alpha, flags_dev, st);
}

namespace {
int check_group(ds_sync** g, uint32_t n, float** replica, float** worker, int mode) {
  if (!g || !replica || n == 0 || n > static_cast<uint32_t>(dsb::kMaxRanks))
    return dsb::set_error(DS_E_CONTRACT, "sync_group: 1..8 ranks");
  for (uint32_t k = 0; k < n; ++k) {
    if (!g[k] || !replica[k] || (mode == 1 && !worker[k])) return dsb::set_error(DS_E_CONTRACT, "sync_group: null");
    if (g[k]->rank != static_cast<int>(k) || g[k]->world != static_cast<int>(n) || g[k]->device != g[0]->device ||
        !g[k]->attached || g[k]->dim != g[0]->dim)
      return dsb::set_error(DS_E_STATE, "sync_group: ranks 0..n-1 of one attached group on one device");
  }
  return DS_OK;
}

int round_group(ds_sync** g, uint32_t n, int mode, float** replica, float** worker, float eta, float wd, float alpha,
                uint32_t* flags, cudaStream_t st) {
  ds_sync* s0 = g[0];
  for (uint32_t k = 0; k < n; ++k)
    if (g[k]->round != s0->round || g[k]->round == 0)
      return dsb::set_error(DS_E_STATE, "sync_group: every rank must have begun the same round");
  dsb::RoundArgs a = round_args(s0, mode, eta, wd, alpha, flags);
  a.self = 0;
  a.r0 = 0;
  a.r1 = static_cast<int>(n);
  a.group = 1;
  a.vec = 1;
  for (uint32_t k = 0; k < n; ++k) {
    a.replica[k] = replica[k];
    a.worker[k] = mode == 1 ? worker[k] : nullptr;
    if (!al16(replica[k]) || (mode == 1 && !al16(worker[k]))) a.vec = 0;
  }
  dsb::round_kernel<<<s0->ctas, dsb::kT, 0, st>>>(a);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}
}  // namespace

extern "C" int ds_sync_reduce_update_group(ds_sync** group, uint32_t n, float** params, float eta, float wd,
                                           uint32_t* flags_dev, void* stream) {
  DS_TRY(check_group(group, n, params, nullptr, 0));
  if (!(eta > 0.0f)) return dsb::set_error(DS_E_CONTRACT, "sgd_step: eta must be positive");
  dsb::DeviceScope ds(group[0]->device);
  return round_group(group, n, 0, params, nullptr, eta, wd, 0.f, flags_dev, dsb::as_stream(stream));
}

extern "C" int ds_sync_easgd_update_group(ds_sync** group, uint32_t n, float** workers, float** centers, float alpha,
                                          uint32_t* flags_dev, void* stream) {
  if (!workers) return dsb::set_error(DS_E_CONTRACT, "sync_group: null");
  DS_TRY(check_group(group, n, centers, workers, 1));
  if (!(alpha > 0.0f && alpha < 1.0f)) return dsb::set_error(DS_E_CONTRACT, "easgd: alpha must be in (0,1)");
  dsb::DeviceScope ds(group[0]->device);
  cudaStream_t st = dsb::as_stream(stream);
  for (uint32_t k = 0; k < n; ++k) {
    float* slot = nullptr;
    DS_TRY(ds_sync_begin(group[k], &slot, stream));
    DS_CUDA_TRY(cudaMemcpyAsync(slot, workers[k], group[k]->dim * sizeof(float), cudaMemcpyDeviceToDevice, st));
    DS_CUDA_TRY(cudaMemcpyAsync(slot + group[k]->dpad, centers[k], group[k]->dim * sizeof(float),
                                cudaMemcpyDeviceToDevice, st));
  }
  return round_group(group, n, 1, centers, workers, 0.f, 0.f, alpha, flags_dev, st);
}

extern "C" int ds_sync_peer_read(ds_sync* s, float* dst, uint64_t n, void* stream) {
  if (!s || !dst) return dsb::set_error(DS_E_CONTRACT, "sync_peer_read: null");
  if (!s->attached || s->world < 2) return dsb::set_error(DS_E_STATE, "sync_peer_read: needs an attached group of >= 2");
  const uint64_t per = (n / static_cast<uint64_t>(s->world - 1)) & ~3ull;
  if (per == 0 || per > alloc_floats(s->dpad) || !al16(dst))
    return dsb::set_error(DS_E_CONTRACT, "sync_peer_read: n must give 4..%llu floats per peer, dst 16-byte aligned",
                          static_cast<unsigned long long>(alloc_floats(s->dpad)));
  dsb::DeviceScope ds(s->device);
  const int ctas = dsb::sm_count(s->device) * 8;
  dsb::peer_read_kernel<<<ctas, dsb::kT, 0, dsb::as_stream(stream)>>>(s->table, s->rank, per, dst);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

extern "C" int ds_sync_rounds(ds_sync* s, uint64_t* out) {
  if (!s || !out) return dsb::set_error(DS_E_CONTRACT, "sync_rounds: null");
  *out = s->round;
  return DS_OK;
}

extern "C" int ds_sync_destroy(ds_sync* s) {
  if (!s) return DS_OK;
  dsb::DeviceScope ds(s->device);
  cudaDeviceSynchronize();
  for (int k = 0; k < dsb::kMaxRanks; ++k) {
    if (s->peer_slots[k]) cudaIpcCloseMemHandle(s->peer_slots[k]);
    if (s->peer_flags[k]) cudaIpcCloseMemHandle(s->peer_flags[k]);
  }
  cudaFree(s->slots);
  cudaFree(s->flags);
  delete s;
  return DS_OK;
}
