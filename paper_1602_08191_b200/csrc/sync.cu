// sync.cu — synchronous data-parallel SGD over GPUs (simulate_sync, simulator.cpp:156-223),
// one process per GPU, with the gradient "allreduce" fused into the update kernel.
//
// Every rank computes its worker's f32 gradient into a peer-mapped slot; one kernel per
// round then reads the `world` slots over NVLink (CUDA IPC mappings), sums them in f64 in
// WORKER ORDER (the reference's gsum loop, simulator.cpp:192-200 — a ring/tree allreduce
// would reorder the additions), divides by n, folds weight decay and applies sgd_step to
// the rank's replica of the master (simulator.cpp:204-209). All replicas perform the same
// arithmetic on the same inputs, so they stay bit-identical without a broadcast.
//
// Round protocol (round r = 1, 2, ...; slot r % 2, double-buffered):
//   ds_sync_begin  : wait until every peer finished round r-2 (its `done` >= r-2), so the
//                    slot this rank is about to overwrite has no reader left.
//   (caller writes its gradient into the slot on the same stream)
//   ds_sync_reduce_update: publish ready = r (system-scope release after the slot writes),
//                    wait for every peer's ready >= r, ordered f64 sum + SGD, then
//                    publish done = r (a trailing one-thread kernel, after every CTA).
#include <cuda_runtime.h>
#include <stdint.h>
#include <unistd.h>

#include <cstring>

#include "ds_common.cuh"
#include "ds_cuda.h"

namespace dsb {
namespace {

constexpr int kMaxRanks = 8;

struct alignas(128) SyncFlags {
  unsigned long long ready;  // last round whose gradient slot is complete
  unsigned long long done;   // last round whose reduction finished reading every slot
  unsigned long long pad[14];
};

struct SyncTable {
  int world;
  const float* slot[kMaxRanks];  // base of each rank's [2][dim] slots (own = local pointer)
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

__global__ void wait_done_kernel(SyncTable t, unsigned long long round) {
  if (threadIdx.x >= static_cast<unsigned>(t.world)) return;
  const unsigned long long* f = &t.flags[threadIdx.x]->done;
  while (ld_acquire_sys_u64(f) < round) __nanosleep(64);
}

__global__ void publish_done_kernel(SyncFlags* own, unsigned long long round) {
  __threadfence_system();
  st_release_sys_u64(&own->done, round);
}

// Grid-stride over the vector. CTA 0 publishes this rank's `ready`; every CTA's thread 0
// waits for all peers' `ready` before its threads read peer slots.
__global__ void __launch_bounds__(256) reduce_update_kernel(SyncTable t, int rank, unsigned long long round,
                                                            uint64_t dim, uint64_t slot_off, float* params,
                                                            float eta, float wd, uint32_t* flags) {
  if (threadIdx.x == 0) {
    if (blockIdx.x == 0) {
      __threadfence_system();  // this rank's gradient (written by earlier kernels) first
      st_release_sys_u64(&t.flags[rank]->ready, round);
    }
    for (int k = 0; k < t.world; ++k)  // own slot: complete by stream order
      if (k != rank)
        while (ld_acquire_sys_u64(&t.flags[k]->ready) < round) __nanosleep(32);
  }
  __syncthreads();
  const double n = static_cast<double>(t.world);
  uint32_t bad = 0;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < dim; i += stride) {
    double gsum = 0.0;  // simulator.cpp:192: std::vector<double> gsum(P, 0.0)
    for (int k = 0; k < t.world; ++k) gsum = dadd(gsum, static_cast<double>(__ldcg(t.slot[k] + slot_off + i)));
    float g = static_cast<float>(__ddiv_rn(gsum, n));
    const float x = params[i];
    if (wd > 0.0f) g = fadd(g, fmul(wd, x));  // simulator.cpp:205-207
    // sgd_step(master, gavg, eta) (param_vector.cpp:21-39)
    if (!isfinite(x)) bad |= DS_FLAG_X_NONFINITE;
    if (!isfinite(g)) bad |= DS_FLAG_G_NONFINITE;
    const float o = fsub(x, fmul(eta, g));
    if (!isfinite(o)) bad |= DS_FLAG_OUT_NONFINITE;
    params[i] = o;
  }
  const uint32_t any = __reduce_or_sync(0xffffffffu, bad);
  if (any && flags && (threadIdx.x & 31) == 0) atomicOr(flags, any);
}

struct IpcRecord {
  cudaIpcMemHandle_t slots;
  cudaIpcMemHandle_t flags;
  uint64_t dim;
  int32_t rank, world, device, pid;
  uint8_t pad[DS_IPC_RECORD_BYTES - 2 * sizeof(cudaIpcMemHandle_t) - 8 - 4 * 4];
};
static_assert(sizeof(IpcRecord) == DS_IPC_RECORD_BYTES, "IPC record size");

}  // namespace
}  // namespace dsb

struct ds_sync {
  int device = 0, rank = 0, world = 1;
  uint64_t dim = 0;
  float* slots = nullptr;             // own [2][dim] gradient slots (peer-mapped)
  dsb::SyncFlags* flags = nullptr;    // own ready/done words (peer-mapped)
  void* peer_slots[dsb::kMaxRanks] = {};
  void* peer_flags[dsb::kMaxRanks] = {};
  dsb::SyncTable table{};
  bool attached = false;
  unsigned long long round = 0;       // rounds begun
  int ctas = 1;
};

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
  cudaError_t e = cudaMalloc(&s->slots, 2 * dim * sizeof(float));
  if (e == cudaSuccess) e = cudaMalloc(&s->flags, sizeof(dsb::SyncFlags));
  if (e == cudaSuccess) e = cudaMemset(s->flags, 0, sizeof(dsb::SyncFlags));
  if (e == cudaSuccess) e = cudaMemset(s->slots, 0, 2 * dim * sizeof(float));
  if (e != cudaSuccess) {
    cudaFree(s->slots);
    cudaFree(s->flags);
    delete s;
    return dsb::set_error(e == cudaErrorMemoryAllocation ? DS_E_NOMEM : DS_E_CUDA, "sync: %s", cudaGetErrorString(e));
  }
  s->table.world = world;
  for (int k = 0; k < world; ++k) {  // world == 1 needs no attach
    s->table.slot[k] = k == rank ? s->slots : nullptr;
    s->table.flags[k] = k == rank ? s->flags : nullptr;
  }
  s->attached = world == 1;
  const uint64_t want = (dim + 255) / 256;
  const uint64_t cap = static_cast<uint64_t>(dsb::sm_count(device)) * 4;
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
  std::memcpy(record_out, &r, sizeof(r));
  return DS_OK;
}

extern "C" int ds_sync_attach(ds_sync* s, const void* records) {
  if (!s || !records) return dsb::set_error(DS_E_CONTRACT, "sync_attach: null");
  if (s->world == 1) return DS_OK;
  dsb::DeviceScope ds(s->device);
  const auto* recs = static_cast<const dsb::IpcRecord*>(records);
  for (int k = 0; k < s->world; ++k) {
    const dsb::IpcRecord& r = recs[k];
    if (r.rank != k || r.world != s->world || r.dim != s->dim)
      return dsb::set_error(DS_E_CONTRACT, "sync_attach: record %d does not match this group", k);
    if (k == s->rank) continue;
    void* ps = nullptr;
    void* pf = nullptr;
    DS_CUDA_TRY(cudaIpcOpenMemHandle(&ps, r.slots, cudaIpcMemLazyEnablePeerAccess));
    DS_CUDA_TRY(cudaIpcOpenMemHandle(&pf, r.flags, cudaIpcMemLazyEnablePeerAccess));
    s->peer_slots[k] = ps;
    s->peer_flags[k] = pf;
    s->table.slot[k] = static_cast<const float*>(ps);
    s->table.flags[k] = static_cast<dsb::SyncFlags*>(pf);
  }
  s->attached = true;
  return DS_OK;
}

extern "C" int ds_sync_begin(ds_sync* s, float** grad_slot, void* stream) {
  if (!s || !grad_slot) return dsb::set_error(DS_E_CONTRACT, "sync_begin: null");
  if (!s->attached) return dsb::set_error(DS_E_STATE, "sync_begin: group not attached");
  dsb::DeviceScope ds(s->device);
  const unsigned long long r = ++s->round;
  if (r > 2 && s->world > 1) {
    dsb::wait_done_kernel<<<1, 32, 0, dsb::as_stream(stream)>>>(s->table, r - 2);
    DS_CUDA_TRY(cudaGetLastError());
  }
  *grad_slot = s->slots + (r & 1) * s->dim;
  return DS_OK;
}

extern "C" int ds_sync_reduce_update(ds_sync* s, float* params, float eta, float wd, uint32_t* flags_dev,
                                     void* stream) {
  if (!s || !params) return dsb::set_error(DS_E_CONTRACT, "sync_reduce_update: null");
  if (!s->attached || s->round == 0) return dsb::set_error(DS_E_STATE, "sync_reduce_update: no round begun");
  if (!(eta > 0.0f)) return dsb::set_error(DS_E_CONTRACT, "sgd_step: eta must be positive");
  dsb::DeviceScope ds(s->device);
  const unsigned long long r = s->round;
  cudaStream_t st = dsb::as_stream(stream);
  dsb::reduce_update_kernel<<<s->ctas, 256, 0, st>>>(s->table, s->rank, r, s->dim, (r & 1) * s->dim, params, eta,
                                                     wd, flags_dev);
  DS_CUDA_TRY(cudaGetLastError());
  if (s->world > 1) {
    dsb::publish_done_kernel<<<1, 1, 0, st>>>(s->flags, r);
    DS_CUDA_TRY(cudaGetLastError());
  }
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
