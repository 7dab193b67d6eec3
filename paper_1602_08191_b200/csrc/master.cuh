// master.cuh — the center variable x~ (MasterState, exchanger.hpp:40-72) on B200s.
//
// One device holds the whole center (world == 1), or each of `world` processes owns a
// contiguous, 128-byte aligned slice and maps its peers' slices over NVLink (CUDA IPC).
// An exchange is ONE kernel that streams the worker vector from local HBM and
// read-modify-writes every slice where it lives — plain 32-bit loads/stores, so a
// LockFree exchange can lose updates but never tears a value (the reference's
// relaxed std::atomic<float> contract, exchanger.cpp:76-92).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <condition_variable>
#include <mutex>
#include <vector>

#include "ds_cuda.h"

namespace dsb {

constexpr int kMaxShards = 8;

// Per-shard control words, in the shard owner's memory, peer-mapped to every rank.
struct alignas(128) ShardFlags {
  unsigned long long seq;        // next ticket allowed to touch this shard
  unsigned long long done;       // CTAs finished for the current ticket
  unsigned long long next_ticket;  // ticket dispenser (Locked mode; rank 0's copy is used)
  unsigned long long exchanges;  // completed exchanges (counted on shard 0)
  unsigned long long timeouts;   // ticket waits on this shard that gave up (wait_seq_eq)
  unsigned long long pad[11];
};

// What an exchange kernel needs to reach every slice.
struct ShardTable {
  int n;
  uint64_t begin[kMaxShards + 1];
  float* ptr[kMaxShards];
  ShardFlags* flags[kMaxShards];
};

// Kernel-side conditional: exchange only if *fire != 0 (nullptr = unconditional).
// ticket: explicit ticket (deterministic), or read from *ticket_slot (Locked), or
// none (LockFree) when both are "unset".
constexpr uint64_t kNoTicket = ~0ull;

int launch_exchange(const ShardTable& t, const float* worker, float* out, float alpha,
                    uint64_t ticket, const unsigned long long* ticket_slot,
                    const uint32_t* fire, const uint32_t* gate, cudaStream_t s,
                    int ctas_per_shard = 0);

}  // namespace dsb

struct ds_master {
  int device = 0;
  uint64_t dim = 0;
  float alpha = 0.1f;
  int mode = DS_MODE_LOCKED;
  int rank = 0, world = 1;
  bool sharded = false, attached = false;
  uint64_t slice_len = 0, begin = 0, end = 0;
  float* local = nullptr;              // own slice
  dsb::ShardFlags* flags = nullptr;    // own control words
  unsigned long long* ticket_slot = nullptr;  // device scratch for a taken ticket
  dsb::ShardTable table{};
  void* peer_mem[dsb::kMaxShards] = {};    // IPC-opened peer slices (to close)
  void* peer_flags[dsb::kMaxShards] = {};
  cudaStream_t stream = nullptr;       // all exchanges issued by this process
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  std::mutex mu;                       // host-side serialization of enqueues
  std::condition_variable cv;
  uint64_t next_host_ticket = 0;       // single-device deterministic ordering
  uint64_t host_exchanges = 0;
  // streams that may carry work touching this center (callers' exchange streams, attached
  // engines): snapshot / count / reset wait for these and the master stream only, never
  // for the whole device
  std::mutex cmu;
  std::vector<cudaStream_t> clients;
  cudaEvent_t ev_q = nullptr;
};

namespace dsb {
// Enqueue an exchange of `worker` (device, on caller stream `caller`) against master m.
// fire/gate as in launch_exchange. Orders the work on the master stream when the mode
// needs serialization and joins back into `caller`.
int master_enqueue_exchange(ds_master* m, const float* worker, float* out, uint64_t ticket,
                            const uint32_t* fire, const uint32_t* gate, cudaStream_t caller);
// client-stream registry (see ds_master::clients); remove is a no-op for a destroyed master
void master_add_client(ds_master* m, cudaStream_t s);
void master_remove_client(ds_master* m, cudaStream_t s);
// drop `s` from every live master's registry (the stream is about to be destroyed)
void master_forget_stream(cudaStream_t s);
// wait for the master stream and every client stream's work enqueued so far
int master_quiesce(ds_master* m);
}  // namespace dsb
