// master.cu — MasterState (exchanger.cpp:65-122) as a device-resident, optionally
// sharded center variable, and the one-kernel P2P elastic exchange.
//
// Scheduling (north_star 3): the reference's acceptor + FIFO queue + handler pool
// (exchanger.cpp:166-206) becomes stream order plus device flags:
//   LockFree  - the exchange kernel runs wherever it is enqueued; concurrent exchanges
//               interleave per element (lost updates allowed, no torn values).
//   Locked    - single device: every exchange is enqueued on the master's stream under
//               a host mutex (linearizable, FIFO in enqueue order); sharded: a device
//               ticket dispenser orders exchanges globally and each slice admits
//               ticket k only after ticket k-1 completed on it.
//   Ticketed  - deterministic replay of simulate_async's serialization: the caller
//               names the global exchange number.
#include <unistd.h>

#include <cstring>
#include <set>

#include "ds_common.cuh"
#include "master.cuh"

namespace dsb {

namespace {

constexpr int kT = 256;

__device__ __forceinline__ void elastic4(const float4& w, const float4& m, float a, float4& wo, float4& mo) {
  elastic_elem(w.x, m.x, a, wo.x, mo.x);
  elastic_elem(w.y, m.y, a, wo.y, mo.y);
  elastic_elem(w.z, m.z, a, wo.z, mo.z);
  elastic_elem(w.w, m.w, a, wo.w, mo.w);
}

// One kernel over every slice: blockIdx.x % n picks the slice (so resident CTAs hit all
// peers at once), blockIdx.x / n the chunk inside it.
__global__ void __launch_bounds__(kT) exchange_kernel(const float* w, float* out, ShardTable t, float a,
                                                      uint64_t ticket, const unsigned long long* ticket_slot,
                                                      const uint32_t* fire, const uint32_t* gate, int cps,
                                                      int vec) {
  if (fire && *fire == 0) return;  // the policy did not fire: no exchange, no ticket
  // An errored engine (gate) skips the data but still passes an explicit ticket on, so the
  // peers waiting for the next ticket are not left hanging. A dispenser ticket was never
  // taken when gated (take_ticket_kernel skips too).
  const bool gated = gate && *gate;
  if (gated && (ticket_slot || ticket == kNoTicket)) return;
  const int s = blockIdx.x % t.n;
  const int c = blockIdx.x / t.n;
  const uint64_t b0 = t.begin[s], b1 = t.begin[s + 1];
  const uint64_t tk = ticket_slot ? static_cast<uint64_t>(*ticket_slot) : ticket;
  const bool ordered = tk != kNoTicket;
  if (ordered) {
    __shared__ int s_timeout;
    if (threadIdx.x == 0) {
      s_timeout = !wait_seq_eq(reinterpret_cast<const uint64_t*>(&t.flags[s]->seq), tk, 100);
      if (s_timeout) atomicAdd_system(&t.flags[s]->timeouts, 1ull);
    }
    __syncthreads();
    if (s_timeout) return;
  }
  const uint64_t len = gated ? 0 : b1 - b0;
  const uint64_t per = ((len + cps - 1) / cps + 3) & ~3ull;
  const uint64_t lo = b0 + per * c;
  const uint64_t hi = lo + per < b1 ? lo + per : b1;
  float* m = t.ptr[s] - b0;  // indexed by global element number
  if (lo < hi) {
    if (vec) {
      const uint64_t v_end = lo + ((hi - lo) & ~3ull);
      for (uint64_t i = lo + 4ull * threadIdx.x; i < v_end; i += 4ull * kT) {
        const float4 wv = __ldcs(reinterpret_cast<const float4*>(w + i));
        const float4 mv = __ldcg(reinterpret_cast<const float4*>(m + i));
        float4 wo, mo;
        elastic4(wv, mv, a, wo, mo);
        __stcs(reinterpret_cast<float4*>(out + i), wo);
        __stcg(reinterpret_cast<float4*>(m + i), mo);
      }
      for (uint64_t i = v_end + threadIdx.x; i < hi; i += kT) {
        float wo, mo;
        elastic_elem(w[i], m[i], a, wo, mo);
        out[i] = wo;
        m[i] = mo;
      }
    } else {
      for (uint64_t i = lo + threadIdx.x; i < hi; i += kT) {
        float wo, mo;
        elastic_elem(w[i], m[i], a, wo, mo);
        out[i] = wo;
        m[i] = mo;
      }
    }
  }
  if (ordered) {
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      const unsigned long long old = atomicAdd_system(&t.flags[s]->done, 1ull);
      if (old == static_cast<unsigned long long>(cps) - 1) {
        t.flags[s]->done = 0;
        if (s == 0) t.flags[0]->exchanges += 1;
        __threadfence_system();
        st_release_sys(reinterpret_cast<uint64_t*>(&t.flags[s]->seq), tk + 1);
      }
    }
  } else if (blockIdx.x == 0 && threadIdx.x == 0) {
    atomicAdd_system(&t.flags[0]->exchanges, 1ull);
  }
}

__global__ void take_ticket_kernel(ShardFlags* f0, unsigned long long* slot, const uint32_t* fire,
                                   const uint32_t* gate) {
  if (fire && *fire == 0) return;
  if (gate && *gate) return;
  *slot = atomicAdd_system(&f0->next_ticket, 1ull);
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

}  // namespace

int launch_exchange(const ShardTable& t, const float* worker, float* out, float alpha, uint64_t ticket,
                    const unsigned long long* ticket_slot, const uint32_t* fire, const uint32_t* gate,
                    cudaStream_t s, int ctas_per_shard) {
  uint64_t maxlen = 0;
  for (int i = 0; i < t.n; ++i) {
    const uint64_t l = t.begin[i + 1] - t.begin[i];
    maxlen = l > maxlen ? l : maxlen;
  }
  int cps = ctas_per_shard;
  if (cps <= 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t budget = static_cast<uint64_t>(sm_count(dev)) * 8 / t.n;  // ~8 CTAs per SM in total
    const uint64_t want = (maxlen + 8191) / 8192;                          // >= 8K elements per CTA
    cps = static_cast<int>(want < 1 ? 1 : (want > budget ? (budget ? budget : 1) : want));
  }
  const int vec = aligned16(worker) && aligned16(out);
  exchange_kernel<<<cps * t.n, kT, 0, s>>>(worker, out, t, alpha, ticket, ticket_slot, fire, gate, cps, vec);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

namespace {
std::mutex g_live_mu;
std::set<const ds_master*> g_live;  // masters not yet destroyed
}  // namespace

void master_add_client(ds_master* m, cudaStream_t s) {
  if (s == m->stream) return;
  std::lock_guard<std::mutex> lk(m->cmu);
  for (cudaStream_t c : m->clients)
    if (c == s) return;
  m->clients.push_back(s);
}

void master_remove_client(ds_master* m, cudaStream_t s) {
  std::lock_guard<std::mutex> g(g_live_mu);
  if (!g_live.count(m)) return;
  std::lock_guard<std::mutex> lk(m->cmu);
  for (size_t i = 0; i < m->clients.size(); ++i)
    if (m->clients[i] == s) {
      m->clients.erase(m->clients.begin() + static_cast<long>(i));
      return;
    }
}

void master_forget_stream(cudaStream_t s) {
  std::lock_guard<std::mutex> g(g_live_mu);
  for (const ds_master* cm : g_live) {
    ds_master* m = const_cast<ds_master*>(cm);
    std::lock_guard<std::mutex> lk(m->cmu);
    for (size_t i = 0; i < m->clients.size(); ++i)
      if (m->clients[i] == s) {
        m->clients.erase(m->clients.begin() + static_cast<long>(i));
        break;
      }
  }
}

int master_quiesce(ds_master* m) {
  DeviceScope ds(m->device);
  DS_CUDA_TRY(cudaStreamSynchronize(m->stream));
  std::lock_guard<std::mutex> lk(m->cmu);
  for (size_t i = 0; i < m->clients.size();) {
    if (cudaEventRecord(m->ev_q, m->clients[i]) != cudaSuccess) {  // the stream was destroyed
      cudaGetLastError();
      m->clients.erase(m->clients.begin() + static_cast<long>(i));
      continue;
    }
    DS_CUDA_TRY(cudaEventSynchronize(m->ev_q));
    ++i;
  }
  return DS_OK;
}

int master_enqueue_exchange(ds_master* m, const float* worker, float* out, uint64_t ticket, const uint32_t* fire,
                            const uint32_t* gate, cudaStream_t caller) {
  DeviceScope ds(m->device);
  master_add_client(m, caller);
  if (m->sharded && !m->attached) return set_error(DS_E_STATE, "master: sharded master not attached to peers");
  if (m->mode == DS_MODE_LOCKFREE && ticket == kNoTicket) {
    // LockFree: no serialization at all, straight on the caller's stream.
    return launch_exchange(m->table, worker, out, m->alpha, kNoTicket, nullptr, fire, gate, caller);
  }
  std::unique_lock<std::mutex> lk(m->mu);
  if (!m->sharded && ticket != kNoTicket) {
    // single device, deterministic: enqueue strictly in ticket order
    m->cv.wait(lk, [&] { return m->next_host_ticket == ticket; });
  }
  DS_CUDA_TRY(cudaEventRecord(m->ev_in, caller));
  DS_CUDA_TRY(cudaStreamWaitEvent(m->stream, m->ev_in, 0));
  int rc;
  if (!m->sharded) {
    // stream order on one device is the serialization
    rc = launch_exchange(m->table, worker, out, m->alpha, kNoTicket, nullptr, fire, gate, m->stream);
  } else if (ticket != kNoTicket) {
    rc = launch_exchange(m->table, worker, out, m->alpha, ticket, nullptr, fire, gate, m->stream);
  } else {
    take_ticket_kernel<<<1, 1, 0, m->stream>>>(m->table.flags[0], m->ticket_slot, fire, gate);
    rc = launch_exchange(m->table, worker, out, m->alpha, kNoTicket, m->ticket_slot, fire, gate, m->stream);
  }
  if (rc != DS_OK) return rc;
  DS_CUDA_TRY(cudaEventRecord(m->ev_out, m->stream));
  DS_CUDA_TRY(cudaStreamWaitEvent(caller, m->ev_out, 0));
  if (!m->sharded && ticket != kNoTicket) {
    ++m->next_host_ticket;
    lk.unlock();
    m->cv.notify_all();
  }
  ++m->host_exchanges;
  return DS_OK;
}

}  // namespace dsb

// ------------------------------------------------------------------------------------
// C-ABI
// ------------------------------------------------------------------------------------
namespace {

struct IpcRecord {
  cudaIpcMemHandle_t mem;
  cudaIpcMemHandle_t flags;
  uint64_t dim, slice_len, begin, end;
  int32_t rank, world, device, pid;
  uint64_t mem_ptr, flags_ptr;  // same-process peers (shards of one GPU) use these directly
  uint8_t pad[DS_IPC_RECORD_BYTES - 2 * sizeof(cudaIpcMemHandle_t) - 6 * 8 - 4 * 4];
};
static_assert(sizeof(IpcRecord) == DS_IPC_RECORD_BYTES, "IPC record size");

int create_common(ds_master** out, int device, uint64_t dim, float alpha, int mode, int rank, int world,
                  const float* init) {
  if (!out) return dsb::set_error(DS_E_CONTRACT, "master: null out");
  if (dim == 0 || dim > 0xFFFFFFFFull) return dsb::set_error(DS_E_CONTRACT, "master: dim must be in [1, 2^32)");
  if (!(alpha > 0.0f && alpha < 1.0f)) return dsb::set_error(DS_E_CONTRACT, "exchanger: alpha must be in (0,1)");
  if (mode != DS_MODE_LOCKED && mode != DS_MODE_LOCKFREE) return dsb::set_error(DS_E_CONTRACT, "master: bad mode");
  if (world < 1 || world > dsb::kMaxShards || rank < 0 || rank >= world)
    return dsb::set_error(DS_E_CONTRACT, "master: rank/world out of range (world <= %d)", dsb::kMaxShards);
  if (!init) return dsb::set_error(DS_E_CONTRACT, "master initial params: null");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return dsb::set_error(DS_E_CUDA, "master: no CUDA device");
  if (device < 0 || device >= ndev) return dsb::set_error(DS_E_CONTRACT, "master: bad device %d", device);
  dsb::DeviceScope ds(device);
  auto* m = new ds_master();
  m->device = device;
  m->dim = dim;
  m->alpha = alpha;
  m->mode = mode;
  m->rank = rank;
  m->world = world;
  m->sharded = world > 1;
  m->slice_len = ((dim + world - 1) / world + 31) & ~31ull;  // 128-byte aligned slices
  m->begin = m->slice_len * rank < dim ? m->slice_len * rank : dim;
  m->end = m->begin + m->slice_len < dim ? m->begin + m->slice_len : dim;
  const uint64_t own = m->end - m->begin;
  auto fail = [&](int rc) {
    if (m->local) cudaFree(m->local);
    if (m->flags) cudaFree(m->flags);
    if (m->ticket_slot) cudaFree(m->ticket_slot);
    delete m;
    return rc;
  };
  dsb::warm_master_kernels();  // no first exchange pays lazy module loading
  cudaError_t e = cudaMalloc(&m->local, (own ? own : 1) * sizeof(float));
  if (e == cudaSuccess) e = cudaMalloc(&m->flags, sizeof(dsb::ShardFlags));
  if (e == cudaSuccess) e = cudaMalloc(&m->ticket_slot, sizeof(unsigned long long));
  if (e == cudaSuccess) e = cudaMemset(m->flags, 0, sizeof(dsb::ShardFlags));
  if (e == cudaSuccess && own) e = cudaMemcpy(m->local, init + m->begin, own * sizeof(float), cudaMemcpyDefault);
  if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&m->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&m->ev_in, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&m->ev_out, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&m->ev_q, cudaEventDisableTiming);
  if (e != cudaSuccess)
    return fail(dsb::set_error(e == cudaErrorMemoryAllocation ? DS_E_NOMEM : DS_E_CUDA, "master: %s", cudaGetErrorString(e)));
  // require_finite(initial) (exchanger.cpp:72), checked on the host copy of our slice
  {
    float* h = static_cast<float*>(malloc((own ? own : 1) * sizeof(float)));
    cudaMemcpy(h, m->local, own * sizeof(float), cudaMemcpyDeviceToHost);
    bool ok = true;
    for (uint64_t i = 0; i < own && ok; ++i) ok = std::isfinite(h[i]);
    free(h);
    if (!ok) return fail(dsb::set_error(DS_E_CONTRACT, "master initial params contains a non-finite value"));
  }
  m->table.n = 1;
  m->table.begin[0] = 0;
  m->table.begin[1] = dim;
  m->table.ptr[0] = m->local;
  m->table.flags[0] = m->flags;
  {
    std::lock_guard<std::mutex> g(dsb::g_live_mu);
    dsb::g_live.insert(m);
  }
  *out = m;
  return DS_OK;
}

}  // namespace

extern "C" int ds_master_create(ds_master** out, int device, uint64_t dim, float alpha, int mode,
                                const float* init_host) {
  return create_common(out, device, dim, alpha, mode, 0, 1, init_host);
}

extern "C" int ds_master_create_sharded(ds_master** out, int device, uint64_t dim, float alpha, int mode, int rank,
                                        int world, const float* init_host) {
  return create_common(out, device, dim, alpha, mode, rank, world, init_host);
}

extern "C" int ds_master_export(ds_master* m, void* record_out) {
  if (!m || !record_out) return dsb::set_error(DS_E_CONTRACT, "master_export: null");
  dsb::DeviceScope ds(m->device);
  IpcRecord r;
  std::memset(&r, 0, sizeof(r));
  DS_CUDA_TRY(cudaIpcGetMemHandle(&r.mem, m->local));
  DS_CUDA_TRY(cudaIpcGetMemHandle(&r.flags, m->flags));
  r.dim = m->dim;
  r.slice_len = m->slice_len;
  r.begin = m->begin;
  r.end = m->end;
  r.rank = m->rank;
  r.world = m->world;
  r.device = m->device;
  r.pid = static_cast<int32_t>(getpid());
  r.mem_ptr = reinterpret_cast<uint64_t>(m->local);
  r.flags_ptr = reinterpret_cast<uint64_t>(m->flags);
  std::memcpy(record_out, &r, sizeof(r));
  return DS_OK;
}

extern "C" int ds_master_attach(ds_master* m, const void* records) {
  if (!m || !records) return dsb::set_error(DS_E_CONTRACT, "master_attach: null");
  if (!m->sharded) return DS_OK;
  dsb::DeviceScope ds(m->device);
  const auto* recs = static_cast<const IpcRecord*>(records);
  m->table.n = m->world;
  for (int k = 0; k < m->world; ++k) {
    const IpcRecord& r = recs[k];
    if (r.rank != k || r.world != m->world || r.dim != m->dim || r.slice_len != m->slice_len)
      return dsb::set_error(DS_E_CONTRACT, "master_attach: record %d does not match this master", k);
    m->table.begin[k] = r.begin;
    if (k == m->rank) {
      m->table.ptr[k] = m->local;
      m->table.flags[k] = m->flags;
      continue;
    }
    void* pm = nullptr;
    void* pf = nullptr;
    if (r.pid == static_cast<int32_t>(getpid())) {
      // a shard of this process (several ranks emulated in one process): plain pointers;
      // CUDA IPC handles cannot be opened by the process that exported them
      pm = reinterpret_cast<void*>(r.mem_ptr);
      pf = reinterpret_cast<void*>(r.flags_ptr);
      if (r.device != m->device) {
        int can = 0;
        cudaDeviceCanAccessPeer(&can, m->device, r.device);
        if (!can) return dsb::set_error(DS_E_CUDA, "master_attach: no peer access from device %d to %d", m->device, r.device);
        const cudaError_t pe = cudaDeviceEnablePeerAccess(r.device, 0);
        if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled)
          return dsb::set_error(DS_E_CUDA, "master_attach: %s", cudaGetErrorString(pe));
        cudaGetLastError();
      }
    } else {
      DS_CUDA_TRY(cudaIpcOpenMemHandle(&pm, r.mem, cudaIpcMemLazyEnablePeerAccess));
      DS_CUDA_TRY(cudaIpcOpenMemHandle(&pf, r.flags, cudaIpcMemLazyEnablePeerAccess));
      m->peer_mem[k] = pm;  // opened here: closed by destroy
      m->peer_flags[k] = pf;
    }
    m->table.ptr[k] = static_cast<float*>(pm);
    m->table.flags[k] = static_cast<dsb::ShardFlags*>(pf);
  }
  m->table.begin[m->world] = m->dim;
  m->attached = true;
  return DS_OK;
}

extern "C" int ds_master_destroy(ds_master* m) {
  if (!m) return DS_OK;
  dsb::DeviceScope ds(m->device);
  {
    std::lock_guard<std::mutex> g(dsb::g_live_mu);
    dsb::g_live.erase(m);
  }
  cudaStreamSynchronize(m->stream);
  for (int k = 0; k < dsb::kMaxShards; ++k) {
    if (m->peer_mem[k]) cudaIpcCloseMemHandle(m->peer_mem[k]);
    if (m->peer_flags[k]) cudaIpcCloseMemHandle(m->peer_flags[k]);
  }
  cudaFree(m->local);
  cudaFree(m->flags);
  cudaFree(m->ticket_slot);
  cudaEventDestroy(m->ev_in);
  cudaEventDestroy(m->ev_out);
  cudaEventDestroy(m->ev_q);
  cudaStreamDestroy(m->stream);
  delete m;
  return DS_OK;
}

extern "C" int ds_master_exchange(ds_master* m, const float* worker, float* out, void* stream) {
  if (!m || !worker || !out) return dsb::set_error(DS_E_CONTRACT, "master_exchange: null");
  return dsb::master_enqueue_exchange(m, worker, out, dsb::kNoTicket, nullptr, nullptr, dsb::as_stream(stream));
}

extern "C" int ds_master_exchange_ticketed(ds_master* m, const float* worker, float* out, uint64_t ticket,
                                           void* stream) {
  if (!m || !worker || !out) return dsb::set_error(DS_E_CONTRACT, "master_exchange: null");
  if (ticket == dsb::kNoTicket) return dsb::set_error(DS_E_CONTRACT, "master_exchange: bad ticket");
  return dsb::master_enqueue_exchange(m, worker, out, ticket, nullptr, nullptr, dsb::as_stream(stream));
}

extern "C" int ds_master_snapshot(ds_master* m, float* host_out) {
  if (!m || !host_out) return dsb::set_error(DS_E_CONTRACT, "master_snapshot: null");
  dsb::DeviceScope ds(m->device);
  DS_TRY(dsb::master_quiesce(m));
  if (m->sharded && !m->attached) return dsb::set_error(DS_E_STATE, "master: sharded master not attached to peers");
  for (int k = 0; k < m->table.n; ++k) {
    const uint64_t b = m->table.begin[k], e = m->table.begin[k + 1];
    if (e > b) DS_CUDA_TRY(cudaMemcpy(host_out + b, m->table.ptr[k], (e - b) * sizeof(float), cudaMemcpyDefault));
  }
  return DS_OK;
}

extern "C" int ds_master_local_slice(ds_master* m, float** dev_ptr, uint64_t* begin, uint64_t* end) {
  if (!m) return dsb::set_error(DS_E_CONTRACT, "master: null");
  if (dev_ptr) *dev_ptr = m->local;
  if (begin) *begin = m->begin;
  if (end) *end = m->end;
  return DS_OK;
}

extern "C" int ds_master_exchange_count(ds_master* m, uint64_t* count) {
  if (!m || !count) return dsb::set_error(DS_E_CONTRACT, "master: null");
  dsb::DeviceScope ds(m->device);
  DS_TRY(dsb::master_quiesce(m));
  dsb::ShardFlags f;
  for (int k = 0; k < m->table.n; ++k) {
    DS_CUDA_TRY(cudaMemcpy(&f, m->table.flags[k], sizeof(f), cudaMemcpyDefault));
    if (f.timeouts)
      return dsb::set_error(DS_E_STATE, "master: %llu ordered exchange(s) on shard %d timed out waiting for their "
                            "ticket (a peer worker stopped early or died)", f.timeouts, k);
  }
  DS_CUDA_TRY(cudaMemcpy(&f, m->table.flags[0], sizeof(f), cudaMemcpyDefault));
  *count = f.exchanges;
  return DS_OK;
}

extern "C" int ds_master_dim(ds_master* m, uint64_t* dim) {
  if (!m || !dim) return dsb::set_error(DS_E_CONTRACT, "master: null");
  *dim = m->dim;
  return DS_OK;
}

extern "C" int ds_master_reset_tickets(ds_master* m) {
  if (!m) return dsb::set_error(DS_E_CONTRACT, "master: null");
  dsb::DeviceScope ds(m->device);
  DS_TRY(dsb::master_quiesce(m));
  DS_CUDA_TRY(cudaMemset(m->flags, 0, sizeof(dsb::ShardFlags)));
  std::lock_guard<std::mutex> lk(m->mu);
  m->next_host_ticket = 0;
  return DS_OK;
}

void dsb::warm_master_kernels() { dsb::load_kernels(dsb::exchange_kernel, dsb::take_ticket_kernel); }
