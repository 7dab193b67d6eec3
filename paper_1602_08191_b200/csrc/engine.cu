// engine.cu — the worker's local SGD loop on one B200 (engine.cpp:10-113).
//
// SgdEngine keeps its shard, parameters, gradients, policy state and TrainLog in HBM.
// The host contributes only what is inherently sequential and value-independent: the
// per-epoch Fisher-Yates order of ShardSweeper (engine.cpp:19-33, seeded mt19937_64
// bit-identical to the reference), uploaded as a batch plan once per run() call. Each
// iteration then runs without host round trips:
//
//   fused path   (<= 1 hidden layer): ONE persistent kernel executes all steps of the
//                run — forward, softmax-CE, backward, SGD, ExchangePolicy and the
//                elastic exchange into the (possibly peer-resident) center — with one
//                grid barrier per step (mlp_fused.cu).
//   layered path (any depth): per-layer f64 kernels (model.cu) + SGD + a one-thread
//                policy kernel + a conditional exchange kernel, stream-ordered.
//
// The policy is evaluated on the device (engine.cpp:35-48) so adaptive exchanges need
// no host sync; the exchange kernels test the device-side fire flag themselves.
#include <atomic>
#include <chrono>
#include <algorithm>
#include <cmath>
#include <cstring>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <numeric>
#include <set>
#include <string>
#include <new>
#include <thread>
#include <vector>

#include "deepspark/rng.hpp"
#include "ds_common.cuh"
#include "elementwise.cuh"
#include "engine.cuh"

namespace dsb {
namespace {

// run_training_loop body after the step: policy, TrainLog row (engine.cpp:97-110).
__global__ void policy_kernel(DevState* st, DevLog log) {
  if (st->err) return;
  if (st->flags) {
    st->err = st->flags;
    st->bad_iter = st->iter + 1;
    st->fire = 0;
    return;
  }
  const double loss = st->loss;
  st->cum = dadd(st->cum, loss);
  st->since += 1;
  const bool fire = st->adaptive ? (st->cum > st->cut) : (st->since == st->tau);
  st->period = fire ? st->since : 0u;
  if (fire) {
    st->cum = 0.0;
    st->since = 0;
    st->exchanges += 1;
  }
  st->fire = fire ? 1u : 0u;
  const unsigned long long row = st->iter;
  if (row < log.cap) {
    log.loss[row] = loss;
    log.cum[row] = st->cum;
    log.exchanged[row] = fire ? 1 : 0;
    log.period[row] = st->period;
  }
  st->iter = row + 1;
}

}  // namespace
}  // namespace dsb

struct ds_engine {
  int device = 0;
  cudaStream_t stream = nullptr;
  dsb::ModelInfo model;
  ds_hyper hp{};
  uint64_t shard_n = 0;
  uint32_t shard_classes = 0;
  float* X = nullptr;
  uint32_t* y = nullptr;
  float* params[2] = {nullptr, nullptr};
  int cur = 0;
  float* grad = nullptr;
  double* ws = nullptr;
  double* act = nullptr;   // fused: [2][H x B]
  double* xb64 = nullptr;  // fused MLP: [3][chunks][B][CW] f64 batch rows
  dsb::DevState* st = nullptr;
  dsb::DevLog log{};
  unsigned int* bar = nullptr;
  // batch plan (device) and its pinned staging copy
  uint32_t* plan = nullptr;
  uint32_t* plan_rows = nullptr;
  uint32_t* h_plan = nullptr;
  uint32_t* h_rows = nullptr;
  uint64_t plan_cap = 0;  // steps
  cudaEvent_t plan_ev = nullptr;
  bool plan_ev_armed = false;
  // ShardSweeper (host, bit-identical order)
  std::vector<uint32_t> order;
  uint64_t pos = 0, epoch = 0, seed = 0;
  // host mirror of the fixed-period policy and of queued work
  uint32_t host_since = 0;
  uint64_t queued = 0;
  uint64_t host_exchanges = 0;
  ds_master* master = nullptr;
  std::vector<uint64_t> tickets;
  uint64_t* d_tickets = nullptr;
  int kind = DS_ENGINE_AUTO;
  bool fused = false;
  bool tc = false;   // DS_ENGINE_TC: run_fused launches the tensor-core step (mlp_tc.cu)
  int tc_nc = 0;     // its cluster size
  // tensor-core step: bf16 copies of the batch sources ([rows][tc_pitch(F)]) + TMA maps
  void* tc_shard = nullptr;   // the resident shard
  void* tc_stage = nullptr;   // host-fed rows (ds_engine_step_host)
  void* tc_ring = nullptr;    // stream-mode ring slots
  CUtensorMap tm_shard{}, tm_stage{}, tm_ring{};
  int fused_grid = 0;
  uint64_t launches = 0;
  // host-fed batches (ds_engine_step_host): staging rows, identity plan, row count
  float* Xb = nullptr;              // current slot (one of Xb2)
  uint32_t* yb = nullptr;
  uint32_t* iota = nullptr;
  uint32_t* rows_dev = nullptr;
  float* Xb2[2] = {};               // double-buffered staging for ds_engine_step_host_async
  uint32_t* yb2[2] = {};
  uint32_t* rows2[2] = {};
  cudaEvent_t slot_ev[2] = {};
  bool slot_armed[2] = {};
  int slot = 0;
  // stream mode (ds_engine_stream_*): host-fed ring consumed by one persistent launch
  static constexpr uint32_t kRing = DS_STREAM_RING;  // host may run this many steps ahead
  float* ring_X = nullptr;              // [kRing][B][F]
  uint32_t* ring_y = nullptr;           // [kRing][B]
  uint32_t* ring_words = nullptr;       // [kRing] rows, [kRing] ready sequence
  uint32_t* ring_src = nullptr;         // pinned host: the same words' sources
  unsigned long long* ring_consumed = nullptr;  // pinned host, written by the kernel
  cudaStream_t copy_stream = nullptr;
  bool ring_active = false;
  uint64_t ring_steps = 0, ring_pushed = 0;
  float* ring_hX = nullptr;      // engine-owned pinned staging [kRing][B][F] (ds_engine_stream_push_rows)
  // tensor-core engines: the stream ring tc_ring is [kTcRing][B + 1][tc_pitch(F)] bf16 in
  // HBM (row B of a slot holds its labels). The host gathers each step's rows straight into
  // a pinned twin as bf16 and the copy engine moves a group of slots per DMA, then the
  // group's sequence words (ring_words): two CUDA calls per group of steps
  static constexpr uint32_t kTcRing = 16, kTcGroup = 4;
  uint16_t* tch_ring = nullptr;   // pinned host twin of tc_ring
  uint32_t* tch_words = nullptr;  // pinned host sources of ring_words
  // ds_engine_stream_cache_host_shard: a bf16 copy of a host shard (rows of F), so the
  // per-step gather of rows from that shard is a row copy instead of a read + cast
  const float* hb_src = nullptr;
  uint64_t hb_rows = 0;
  std::vector<uint16_t> hb;
  // a DS_FUSED_PROFILE buffer of a stream-mode launch, reported at ds_engine_stream_end
  unsigned long long* prof_pending = nullptr;
  uint64_t prof_steps = 0, prof_n = 0;
  const char* prof_path = nullptr;
  uint32_t* ring_hy = nullptr;
  double* ring_loss = nullptr;
  float mu = 0.0f;            // momentum (layered path), ds_engine_set_momentum
  float* velocity = nullptr;
  // layered path: one full-batch iteration captured as a CUDA graph (set_idx + loss/grad +
  // update + policy), replayed per step; keyed by the pointers it captured
  cudaGraphExec_t step_graph = nullptr;
  const void* graph_key[3] = {};
  uint32_t* cur_idx = nullptr;             // [B] the step's shard rows (set_idx_kernel)
  ds_sync* sync = nullptr;                 // synchronous data-parallel mode (ds_engine_attach_sync)
  // sync mode: the gradient pass captured once per gradient slot (the group alternates two
  // slots), replayed between the eager round kernels (wait / reduce+update / publish)
  cudaGraphExec_t sync_graph[2] = {};
  float* sync_slot[2] = {};
  bool sync_eager[2] = {};
  const void* sync_key[4] = {};
  unsigned long long* step_ctr = nullptr;  // device step counter within a run
  uint32_t hostfed_rows = 0;
  bool hostfed = false;
};

namespace dsb {
namespace {

void reshuffle(ds_engine* e) {  // ShardSweeper::reshuffle (engine.cpp:19-23)
  deepspark::Rng rng(deepspark::mix_seed(e->seed, e->epoch));
  rng.shuffle(e->order);
  e->pos = 0;
}

uint32_t sweeper_next(ds_engine* e, uint32_t* dst) {  // ShardSweeper::next (engine.cpp:25-33)
  if (e->pos >= e->order.size()) {
    ++e->epoch;
    reshuffle(e);
  }
  const uint64_t take = std::min<uint64_t>(e->hp.batch_size, e->order.size() - e->pos);
  std::memcpy(dst, e->order.data() + e->pos, take * sizeof(uint32_t));
  e->pos += take;
  return static_cast<uint32_t>(take);
}

int ensure_plan(ds_engine* e, uint64_t steps) {
  if (steps <= e->plan_cap) return DS_OK;
  uint64_t cap = std::max<uint64_t>(steps, 2 * e->plan_cap);
  if (e->plan_ev_armed) cudaEventSynchronize(e->plan_ev);
  DS_CUDA_TRY(cudaStreamSynchronize(e->stream));
  cudaFree(e->plan);
  cudaFree(e->plan_rows);
  cudaFreeHost(e->h_plan);
  cudaFreeHost(e->h_rows);
  e->plan = nullptr;
  e->plan_rows = nullptr;
  e->h_plan = nullptr;
  e->h_rows = nullptr;
  const uint64_t B = e->hp.batch_size;
  DS_CUDA_TRY(cudaMalloc(&e->plan, cap * B * sizeof(uint32_t)));
  DS_CUDA_TRY(cudaMalloc(&e->plan_rows, cap * sizeof(uint32_t)));
  DS_CUDA_TRY(cudaMallocHost(&e->h_plan, cap * B * sizeof(uint32_t)));
  DS_CUDA_TRY(cudaMallocHost(&e->h_rows, cap * sizeof(uint32_t)));
  e->plan_cap = cap;
  e->plan_ev_armed = false;
  return DS_OK;
}

int ensure_log(ds_engine* e, uint64_t rows) {
  if (rows <= e->log.cap) return DS_OK;
  uint64_t cap = std::max<uint64_t>(rows, 2 * e->log.cap);
  cap = std::max<uint64_t>(cap, 1024);
  DevLog n{};
  DS_CUDA_TRY(cudaMalloc(&n.loss, cap * sizeof(double)));
  DS_CUDA_TRY(cudaMalloc(&n.cum, cap * sizeof(double)));
  DS_CUDA_TRY(cudaMalloc(&n.exchanged, cap));
  DS_CUDA_TRY(cudaMalloc(&n.period, cap * sizeof(uint32_t)));
  n.cap = cap;
  if (e->log.cap) {
    const uint64_t c = e->log.cap;
    DS_CUDA_TRY(cudaMemcpyAsync(n.loss, e->log.loss, c * sizeof(double), cudaMemcpyDeviceToDevice, e->stream));
    DS_CUDA_TRY(cudaMemcpyAsync(n.cum, e->log.cum, c * sizeof(double), cudaMemcpyDeviceToDevice, e->stream));
    DS_CUDA_TRY(cudaMemcpyAsync(n.exchanged, e->log.exchanged, c, cudaMemcpyDeviceToDevice, e->stream));
    DS_CUDA_TRY(cudaMemcpyAsync(n.period, e->log.period, c * sizeof(uint32_t), cudaMemcpyDeviceToDevice, e->stream));
    DS_CUDA_TRY(cudaStreamSynchronize(e->stream));
    cudaFree(e->log.loss);
    cudaFree(e->log.cum);
    cudaFree(e->log.exchanged);
    cudaFree(e->log.period);
  }
  e->log = n;
  return DS_OK;
}

// Upload the sweep plan for `steps` iterations; returns per-step row counts on host.
int upload_plan(ds_engine* e, uint64_t steps) {
  DS_TRY(ensure_plan(e, steps));
  if (e->plan_ev_armed) DS_CUDA_TRY(cudaEventSynchronize(e->plan_ev));  // staging buffer free again
  const uint64_t B = e->hp.batch_size;
  for (uint64_t j = 0; j < steps; ++j) e->h_rows[j] = sweeper_next(e, e->h_plan + j * B);
  DS_CUDA_TRY(cudaMemcpyAsync(e->plan, e->h_plan, steps * B * sizeof(uint32_t), cudaMemcpyHostToDevice, e->stream));
  DS_CUDA_TRY(cudaMemcpyAsync(e->plan_rows, e->h_rows, steps * sizeof(uint32_t), cudaMemcpyHostToDevice, e->stream));
  DS_CUDA_TRY(cudaEventRecord(e->plan_ev, e->stream));
  e->plan_ev_armed = true;
  return DS_OK;
}

// Next exchange ticket of this worker, or kNoTicket.
uint64_t next_ticket(ds_engine* e) {
  if (e->tickets.empty()) return kNoTicket;
  return e->host_exchanges < e->tickets.size() ? e->tickets[e->host_exchanges] : kNoTicket;
}

bool in_kernel_ok(const ds_engine* e) {
  // the fused kernel may exchange itself when no host-side ordering is needed
  const ds_master* m = e->master;
  if (e->tc) return m != nullptr;  // tickets / dispenser / plain stores, all in-kernel
  return m && (m->sharded || (m->mode == DS_MODE_LOCKFREE && e->tickets.empty()));
}

int enqueue_exchange(ds_engine* e, float* p) {
  const uint64_t tk = next_ticket(e);
  if (!e->tickets.empty() && tk == kNoTicket)
    return set_error(DS_E_STATE, "engine: ran out of deterministic exchange tickets");
  DS_TRY(master_enqueue_exchange(e->master, p, p, tk, &e->st->fire, &e->st->err, e->stream));
  e->launches += (e->master->sharded && e->master->mode == DS_MODE_LOCKED && tk == kNoTicket) ? 2 : 1;
  return DS_OK;
}

// Layered iterations; with_master = perform fired exchanges against e->master.
// cur_idx = plan[ctr*B .. +B); ++ctr (one CTA)
__global__ void set_idx_kernel(const uint32_t* __restrict__ plan, uint32_t B, unsigned long long* ctr,
                               uint32_t* __restrict__ cur_idx) {
  const unsigned long long c = *reinterpret_cast<volatile unsigned long long*>(ctr);
  for (uint32_t r = threadIdx.x; r < B; r += blockDim.x) cur_idx[r] = plan[c * B + r];
  __syncthreads();
  if (threadIdx.x == 0) *ctr = c + 1;
}

// One layered iteration (everything but the exchange) on e->stream.
bool graphs_enabled();

int layered_step(ds_engine* e, const float* X, const uint32_t* y, const uint32_t* idx, uint32_t R, bool set_idx) {
  const uint64_t B = e->hp.batch_size;
  const float eta = static_cast<float>(e->hp.eta);
  const float wd = static_cast<float>(e->hp.weight_decay);
  float* p = e->params[e->cur];
  if (set_idx) {
    set_idx_kernel<<<1, B < 1024 ? static_cast<unsigned>(B) : 1024u, 0, e->stream>>>(e->plan, static_cast<uint32_t>(B),
                                                                                     e->step_ctr, e->cur_idx);
    idx = e->cur_idx;
  }
  if (e->sync) {  // simulate_sync (simulator.cpp:156-223) across the group's GPUs
    float* slot = nullptr;
    DS_TRY(ds_sync_begin(e->sync, &slot, e->stream));
    int k = -1;  // which captured gradient pass (per slot) applies, if any
    if (set_idx && !e->hostfed && R == e->hp.batch_size && graphs_enabled()) {
      const void* key[4] = {X, y, p, e->ws};
      if (std::memcmp(key, e->sync_key, sizeof(key)) != 0) {  // buffers moved: drop the old captures
        for (int q = 0; q < 2; ++q) {
          if (e->sync_graph[q]) cudaGraphExecDestroy(e->sync_graph[q]);
          e->sync_graph[q] = nullptr;
          e->sync_slot[q] = nullptr;
          e->sync_eager[q] = false;
        }
        std::memcpy(e->sync_key, key, sizeof(key));
      }
      for (int q = 0; q < 2 && k < 0; ++q)
        if (e->sync_slot[q] == slot || !e->sync_slot[q]) k = q, e->sync_slot[q] = slot;
    }
    if (k >= 0 && e->sync_graph[k]) {
      DS_CUDA_TRY(cudaGraphLaunch(e->sync_graph[k], e->stream));
    } else {
      DS_TRY(launch_loss_and_grad(e->model, p, X, idx, y, R, slot, &e->st->loss, e->ws, &e->st->flags, &e->st->err,
                                  e->stream));
      if (k >= 0 && e->sync_eager[k]) {  // second use of this slot: record the pass for replay
        cudaGraph_t g = nullptr;
        DS_CUDA_TRY(cudaStreamBeginCapture(e->stream, cudaStreamCaptureModeThreadLocal));
        const int rc = launch_loss_and_grad(e->model, p, X, idx, y, R, slot, &e->st->loss, e->ws, &e->st->flags,
                                            &e->st->err, e->stream);
        const cudaError_t ce = cudaStreamEndCapture(e->stream, &g);
        if (rc != DS_OK) return rc;
        if (ce != cudaSuccess) return set_error(DS_E_CUDA, "engine: sync capture: %s", cudaGetErrorString(ce));
        const cudaError_t ie = cudaGraphInstantiate(&e->sync_graph[k], g, 0);
        cudaGraphDestroy(g);
        if (ie != cudaSuccess) return set_error(DS_E_CUDA, "engine: sync graph: %s", cudaGetErrorString(ie));
      } else if (k >= 0) {
        e->sync_eager[k] = true;
      }
    }
    DS_TRY(ds_sync_reduce_update(e->sync, p, eta, wd, &e->st->flags, e->stream));
    policy_kernel<<<1, 1, 0, e->stream>>>(e->st, e->log);
    DS_CUDA_TRY(cudaGetLastError());
    return DS_OK;
  }
  DS_TRY(launch_loss_and_grad(e->model, p, X, idx, y, R, e->grad, &e->st->loss, e->ws, &e->st->flags, &e->st->err,
                              e->stream));
  if (e->mu > 0.0f)
    DS_TRY(launch_momentum(p, p, e->velocity, e->grad, e->model.P, eta, e->mu, wd, &e->st->flags, e->stream,
                           &e->st->err));
  else
    DS_TRY(launch_sgd(p, p, e->grad, e->model.P, eta, wd, &e->st->flags, e->stream, &e->st->err));
  policy_kernel<<<1, 1, 0, e->stream>>>(e->st, e->log);
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

bool graphs_enabled() {
  const char* v = std::getenv("DS_ENGINE_NO_GRAPH");
  return !(v && v[0] == '1');
}

int run_layered(ds_engine* e, uint64_t steps, bool with_master) {
  if (!e->hostfed) DS_TRY(upload_plan(e, steps));
  const uint64_t B = e->hp.batch_size;
  const float* X = e->hostfed ? e->Xb : e->X;
  const uint32_t* y = e->hostfed ? e->yb : e->y;
  float* p = e->params[e->cur];
  const bool xm = with_master && e->master;
  const uint64_t per_step = (e->model.kind == DS_MODEL_CIFAR10_QUICK ? 31 : 3 * e->model.layers.size() + 1) + 2;
  if (!e->hostfed) {
    if (!e->cur_idx) {
      DS_CUDA_TRY(cudaMalloc(&e->cur_idx, B * sizeof(uint32_t)));
      DS_CUDA_TRY(cudaMalloc(&e->step_ctr, sizeof(unsigned long long)));
    }
    DS_CUDA_TRY(cudaMemsetAsync(e->step_ctr, 0, sizeof(unsigned long long), e->stream));
  }
  const void* key[3] = {e->plan, p, e->velocity};
  if (e->step_graph && (key[0] != e->graph_key[0] || key[1] != e->graph_key[1] || key[2] != e->graph_key[2] ||
                        !graphs_enabled())) {
    cudaGraphExecDestroy(e->step_graph);
    e->step_graph = nullptr;
  }
  for (uint64_t j = 0; j < steps; ++j) {
    const uint32_t R = e->hostfed ? e->hostfed_rows : e->h_rows[j];
    if (e->hostfed) {
      DS_TRY(layered_step(e, X, y, e->iota, R, false));
    } else if (R == B && e->step_graph && !e->sync) {
      DS_CUDA_TRY(cudaGraphLaunch(e->step_graph, e->stream));
    } else {
      DS_TRY(layered_step(e, X, y, nullptr, R, true));
      if (R == B && graphs_enabled() && !e->sync) {  // first full batch ran eagerly; capture the next ones
        cudaGraph_t g = nullptr;
        DS_CUDA_TRY(cudaStreamBeginCapture(e->stream, cudaStreamCaptureModeThreadLocal));
        const int rc = layered_step(e, X, y, nullptr, R, true);
        const cudaError_t ce = cudaStreamEndCapture(e->stream, &g);
        if (rc != DS_OK) return rc;
        if (ce != cudaSuccess) return set_error(DS_E_CUDA, "engine: step capture: %s", cudaGetErrorString(ce));
        const cudaError_t ie = cudaGraphInstantiate(&e->step_graph, g, 0);
        cudaGraphDestroy(g);
        if (ie != cudaSuccess) return set_error(DS_E_CUDA, "engine: step graph: %s", cudaGetErrorString(ie));
        for (int k = 0; k < 3; ++k) e->graph_key[k] = key[k];
      }
    }
    e->launches += (e->model.kind == DS_MODEL_ALEXNET ? dsb::alex_last_launches() + 2 : per_step) + (e->hostfed ? 0 : 1);
    if (e->hp.adaptive) {
      if (xm) DS_TRY(enqueue_exchange(e, p));  // conditional on the device fire flag
    } else if (++e->host_since == e->hp.tau) {
      e->host_since = 0;
      if (xm) DS_TRY(enqueue_exchange(e, p));
      ++e->host_exchanges;
    }
  }
  DS_CUDA_TRY(cudaGetLastError());
  return DS_OK;
}

// The step kernels' arguments for the next `steps` iterations (uploads the batch plan).
int fused_args(ds_engine* e, uint64_t steps, bool in_kernel_exchange, FusedArgs& a) {
  if (!e->hostfed && !e->ring_active) DS_TRY(upload_plan(e, steps));
  a = FusedArgs{};
  a.F = e->model.n_features;
  a.H = e->model.hidden.empty() ? 0 : e->model.hidden[0];
  a.C = e->model.n_classes;
  a.P = e->model.P;
  a.X = e->hostfed ? e->Xb : e->X;
  a.y = e->hostfed ? e->yb : e->y;
  a.plan = (e->hostfed || e->ring_active) ? e->iota : e->plan;
  a.plan_rows = (e->hostfed || e->ring_active) ? e->rows_dev : e->plan_rows;
  a.B = e->hp.batch_size;
  a.steps = steps;
  a.params[0] = e->params[0];
  a.params[1] = e->params[1];
  a.cur = e->cur;
  a.act = e->act;
  a.xb64 = e->xb64;
  a.eta = static_cast<float>(e->hp.eta);
  a.wd = static_cast<float>(e->hp.weight_decay);
  a.alpha = e->master ? e->master->alpha : static_cast<float>(e->hp.alpha);
  a.st = e->st;
  a.log = e->log;
  a.bar = e->bar;
  a.has_master = (e->master && in_kernel_exchange) ? 1 : 0;
  if (a.has_master) {
    a.table = e->master->table;
    a.center_local = (!e->master->sharded && e->master->world == 1) ? 1 : 0;
    a.lockfree = e->master->mode == DS_MODE_LOCKFREE && e->tickets.empty();
    a.tickets = e->tickets.empty() ? nullptr : e->d_tickets + e->host_exchanges;
    if (a.tickets) {
      // the kernel reads one ticket per exchange of this run: never past the array
      const uint64_t need = (e->host_since + steps) / e->hp.tau;
      if (e->host_exchanges + need > e->tickets.size())
        return set_error(DS_E_STATE, "engine: ran out of deterministic exchange tickets (%llu needed, %llu left)",
                         static_cast<unsigned long long>(need),
                         static_cast<unsigned long long>(e->tickets.size() - std::min<uint64_t>(e->host_exchanges, e->tickets.size())));
    }
    a.ticket_src = (!a.lockfree && !a.tickets) ? &e->master->table.flags[0]->next_ticket : nullptr;
  }
  if (e->ring_active) {
    a.ring = 1;
    a.ring_slots = ds_engine::kRing;
    a.ring_X = e->ring_X;
    a.ring_y = e->ring_y;
    a.ring_rows = e->ring_words;
    a.ring_ready = e->ring_words + ds_engine::kRing;
    a.ring_slot_rows = static_cast<uint32_t>(e->hp.batch_size);
    a.ring_y_stride = static_cast<uint32_t>(e->hp.batch_size);
    if (e->tc) {  // bf16 slots of B + 1 rows, the labels in the last row
      const uint64_t B = e->hp.batch_size, pitch = tc_pitch(e->model.n_features);
      a.ring_slots = ds_engine::kTcRing;
      a.ring_slot_rows = static_cast<uint32_t>(B + 1);
      a.ring_y = reinterpret_cast<const uint32_t*>(static_cast<const char*>(e->tc_ring) + B * pitch * 2);
      a.ring_y_stride = static_cast<uint32_t>((B + 1) * pitch / 2);
      a.ring_ready = e->ring_words;
    }
    a.ring_consumed = e->ring_consumed;
    a.ring_loss = e->ring_loss;
  }
  return DS_OK;
}

// Per-phase medians of a DS_FUSED_PROFILE run (stream mode: at stream_end, once the
// launch is done).
int dump_profile(ds_engine* e, unsigned long long* prof, uint64_t steps, uint64_t prof_n, const char* prof_path) {
  const uint64_t G = static_cast<uint64_t>(e->fused_grid);
    std::vector<unsigned long long> h(prof_n);
    DS_CUDA_TRY(cudaMemcpyAsync(h.data(), prof, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, e->stream));
    DS_CUDA_TRY(cudaStreamSynchronize(e->stream));
    cudaFree(prof);
    const char* fnames[] = {"x_staged", "forward", "grid_barrier", "acts_staged", "logits", "softmax_loss",
                            "backward_update", "policy_exchange", "bwd_head", "bwd_dW1"};
    const int fpairs[][2] = {{0, 1}, {1, 2}, {2, 3}, {3, 4}, {4, 5}, {5, 6}, {6, 7}, {7, 8}, {6, 9}, {9, 7}};
    // tensor-core step (mlp_tc.cu): forward MMAs, tanh + partial logits, R phase, softmax +
    // G phase, deltas + dW1 MMAs, W1 SGD, policy + exchange (then the next step's start)
    const char* tnames[] = {"wait_fwd", "tanh_logits", "R_phase", "softmax_G", "unpack_delta1", "w2b_dW1_sgd",
                            "exchange", "-", "start_to_G", "G_to_end"};
    const int tpairs[][2] = {{0, 1}, {1, 2}, {2, 3}, {3, 4}, {4, 5}, {5, 6}, {6, 7}, {7, 7}, {0, 4}, {4, 7}};
    const char* const* names = e->tc ? tnames : fnames;
    const int(*pairs)[2] = e->tc ? tpairs : fpairs;
    static const int xpairs[][2] = {{0, 1}, {1, 6}, {6, 7}, {7, 8}, {8, 2}, {2, 3}, {3, 4}, {4, 5}, {1, 2}, {0, 5}};
    static const char* xnames[] = {"arm", "round0_first_tile", "round0_rest", "round1", "wait_st", "small_fence",
                                   "cbar", "release", "w1_all", "exchange_all"};
    if (e->tc && std::getenv("DS_TC_PROF_X")) pairs = xpairs, names = xnames;
    // the one-shard bulk exchange: ticket, bulk load landed, W1 updated, stored, rest
    static const int bpairs[][2] = {{0, 1}, {1, 6}, {6, 7}, {7, 8}, {8, 3}, {3, 5}, {0, 5}, {0, 0}, {0, 0}, {0, 0}};
    static const char* bnames[] = {"ticket", "bulk_load", "w1_update", "small_store", "fence_sync", "b2_release",
                                   "exchange_all", "-", "-", "-"};
    if (e->tc && std::getenv("DS_TC_PROF_B")) pairs = bpairs, names = bnames;
    // MMA warp timeline: fwd(s) tiles (stamps 2,3,4 at sgdd waits of tiles 0,3,last; 5 commit),
    // logits (6), delta1 ready (0) and dW1 issued (1); pairs are within the MMA loop's step s
    static const int mpairs[][2] = {{2, 3}, {3, 4}, {4, 5}, {5, 6}, {6, 0}, {0, 1}, {2, 5}, {2, 0}, {0, 0}, {0, 0}};
    static const char* mnames[] = {"fwd_t0_t3", "fwd_t3_t6", "fwd_last_commit", "logits_wait_a1",
                                   "a1_to_d1rdy", "dW1_issue", "fwd_all", "fwd_to_d1", "-", "-"};
    if (e->tc && std::getenv("DS_TC_PROF_M")) pairs = mpairs, names = mnames;
    // TMA warp timeline (DS_TC_PROF_T build): poll word, labels, wait for the X buffer,
    // issue, and the MMA warp's arrival of the gathered rows
    static const int tpairs2[][2] = {{0, 1}, {1, 2}, {2, 3}, {3, 4}, {4, 5}, {3, 5}, {0, 5}, {0, 3}, {0, 0}, {0, 0}};
    static const char* tnames2[] = {"poll_word", "labels", "wait_xbuf", "issue", "issue_to_landed", "stage_to_landed",
                                    "start_to_landed", "start_to_stage", "-", "-"};
    if (e->tc && std::getenv("DS_TC_PROF_T")) pairs = tpairs2, names = tnames2;
    if (FILE* f = std::fopen(prof_path, "a")) {
      std::fprintf(f, "steps=%llu", (unsigned long long)steps);
      if (e->tc && h[steps * kProfSlots])
        std::fprintf(f, " sm_clock=%.0fMHz", 1e3 * static_cast<double>(h[steps * kProfSlots + 1]) /
                                                 static_cast<double>(h[steps * kProfSlots]));
      for (int k = 0; k < 10; ++k) {
        std::vector<double> d;
        for (uint64_t s = 2; s < steps; ++s) {
          const unsigned long long t0 = h[s * kProfSlots + pairs[k][0]], t1 = h[s * kProfSlots + pairs[k][1]];
          if (t0 && t1 >= t0) d.push_back(static_cast<double>(t1 - t0));
        }
        std::sort(d.begin(), d.end());
        std::fprintf(f, " %s=%.0fns", names[k], d.empty() ? -1.0 : d[d.size() / 2]);
      }
      std::vector<double> tot;
      for (uint64_t s = 3; s < steps; ++s) tot.push_back(static_cast<double>(h[s * kProfSlots] - h[(s - 1) * kProfSlots]));
      uint64_t worst = 3;
      double sum = 0.0, wmax = 0.0;
      for (uint64_t s = 3; s < steps; ++s) {
        const double d = static_cast<double>(h[s * kProfSlots] - h[(s - 1) * kProfSlots]);
        sum += d;
        if (d > wmax) wmax = d, worst = s - 1;
      }
      std::sort(tot.begin(), tot.end());
      std::fprintf(f, " step=%.0fns", tot.empty() ? -1.0 : tot[tot.size() / 2]);
      if (!tot.empty())
        std::fprintf(f, " step_mean=%.0fns step_p90=%.0fns step_max=%.0fns worst_step=%llu worst_phases:", sum / tot.size(),
                     tot[tot.size() * 9 / 10], wmax, (unsigned long long)worst);
      for (int k = 0; k < 10 && !tot.empty(); ++k) {
        const unsigned long long t0 = h[worst * kProfSlots + pairs[k][0]], t1 = h[worst * kProfSlots + pairs[k][1]];
        std::fprintf(f, " %s=%lld", names[k], static_cast<long long>(t1 - t0));
      }
      {  // grid-barrier anatomy: CTA skew at the forward's end vs the barrier itself
        std::vector<double> skew, mech;
        const unsigned long long* hc = h.data() + steps * kProfSlots;
        for (uint64_t s = 2; s < steps; ++s) {
          unsigned long long lo = ~0ull, hi = 0, exit0 = hc[(s * G) * 2 + 1];
          for (uint64_t g = 0; g < G; ++g) {
            const unsigned long long t = hc[(s * G + g) * 2];
            lo = t < lo ? t : lo;
            hi = t > hi ? t : hi;
          }
          if (lo && exit0 >= hi) {
            skew.push_back(static_cast<double>(hi - lo));
            mech.push_back(static_cast<double>(exit0 - hi));
          }
        }
        std::sort(skew.begin(), skew.end());
        std::sort(mech.begin(), mech.end());
        if (!skew.empty())
          std::fprintf(f, " | fwd_end_skew=%.0fns barrier_after_last=%.0fns", skew[skew.size() / 2], mech[mech.size() / 2]);
      }
      std::fprintf(f, "\n");
      std::fclose(f);
    }
  return DS_OK;
}

int run_fused(ds_engine* e, uint64_t steps, bool in_kernel_exchange) {
  FusedArgs a;
  DS_TRY(fused_args(e, steps, in_kernel_exchange, a));
  // DS_FUSED_PROFILE=<file>: per-phase globaltimer stamps of CTA 0, medians appended
  const char* prof_path = std::getenv("DS_FUSED_PROFILE");
  unsigned long long* prof = nullptr;
  const uint64_t G = static_cast<uint64_t>(e->fused_grid);
  const uint64_t prof_n = steps * (kProfSlots + 2 * G) + 8;
  if (prof_path && steps >= 8) DS_CUDA_TRY(cudaMalloc(&prof, prof_n * sizeof(unsigned long long)));
  if (prof) DS_CUDA_TRY(cudaMemsetAsync(prof, 0, prof_n * sizeof(unsigned long long), e->stream));
  a.prof = prof;
  a.prof_cta = prof ? prof + steps * kProfSlots : nullptr;
  if (e->tc) {
    const CUtensorMap* tm = &e->tm_shard;
    if (e->ring_active) {
      tm = &e->tm_ring;
    } else if (e->hostfed) {  // this step's rows (staged f32 by step_host) as bf16
      DS_TRY(tc_rows_to_bf16(e->Xb, e->hostfed_rows, e->model.n_features, e->tc_stage, e->stream));
      tm = &e->tm_stage;
    }
    DS_TRY(launch_tc(a, e->tc_nc, *tm, e->stream));
  }
  else
    DS_TRY(launch_fused(a, e->fused_grid, e->stream));
  e->launches += 1;
  e->cur ^= static_cast<int>(steps & 1);
  if (prof && e->ring_active) {  // the launch waits on host pushes: report at stream_end
    e->prof_pending = prof;
    e->prof_steps = steps;
    e->prof_n = prof_n;
    e->prof_path = prof_path;
  } else if (prof) {
    DS_TRY(dump_profile(e, prof, steps, prof_n, prof_path));
  }
  return DS_OK;
}

}  // namespace
}  // namespace dsb

using dsb::set_error;
namespace dsb {
int run_group(ds_engine** engines, uint32_t n, uint64_t steps);
}

// ds_engine_create / ds_engine_create_from_shard: the shard comes from host arrays, or
// (shard_path != nullptr) from a DSHD file streamed straight into e->X / e->y.
// Load the step kernels once per device at engine creation, so no timed step pays CUDA's
// lazy module loading (the reference's TrainLog wall_ms would otherwise differ between a
// cold and a warm run of the same training).
static void warm_step_kernels(int device) {
  static std::mutex mu;
  static std::set<int> done;
  std::lock_guard<std::mutex> lk(mu);
  if (!done.insert(device).second) return;
  dsb::DeviceScope ds(device);
  dsb::load_kernels(dsb::policy_kernel, dsb::set_idx_kernel);
  dsb::warm_model_kernels();
  dsb::warm_elementwise_kernels();
  dsb::warm_fused_kernels();
  dsb::warm_tc_kernels();
  dsb::warm_master_kernels();
}

static int engine_create(ds_engine** out, int device, const ds_model_desc* model, const float* X_host,
                         const uint32_t* y_host, uint64_t shard_n, uint32_t shard_classes, const ds_hyper* hp,
                         uint64_t sweep_seed, const float* init_host, int kind, const char* shard_path) {
  if (!out || !hp || (!shard_path && (!X_host || !y_host)) || !init_host)
    return set_error(DS_E_CONTRACT, "engine: null argument");
  dsb::ModelInfo m;
  DS_TRY(dsb::model_from_desc(model, m));
  if (device >= 0) warm_step_kernels(device);
  // Hyperparams::validate (hyperparams.cpp:7-18)
  if (!(hp->eta > 0.0)) return set_error(DS_E_CONTRACT, "hyperparams: eta must be positive");
  if (!(hp->alpha > 0.0 && hp->alpha < 1.0)) return set_error(DS_E_CONTRACT, "hyperparams: alpha must lie in (0,1)");
  if (hp->batch_size == 0) return set_error(DS_E_CONTRACT, "hyperparams: batch_size must be positive");
  if (hp->i_max == 0) return set_error(DS_E_CONTRACT, "hyperparams: i_max must be positive");
  if (hp->weight_decay < 0.0) return set_error(DS_E_CONTRACT, "hyperparams: weight_decay must be nonnegative");
  if (!hp->adaptive && hp->tau == 0) return set_error(DS_E_CONTRACT, "hyperparams: tau must be positive in Fixed mode");
  if (hp->adaptive && !(hp->loss_cut > 0.0))
    return set_error(DS_E_CONTRACT, "hyperparams: loss_cut must be positive in Adaptive mode");
  if (shard_n == 0) return set_error(DS_E_CONTRACT, "dataset: no samples");
  if (shard_n > 0xFFFFFFFFull) return set_error(DS_E_CONTRACT, "engine: shard too large for u32 row indices");
  if (shard_classes == 0) return set_error(DS_E_CONTRACT, "dataset: n_classes must be positive");
  if (shard_classes > m.n_classes) return set_error(DS_E_CONTRACT, "engine: shard dims do not match model");
  if (!shard_path)  // a shard file's labels are range-checked on the device as they land
    for (uint64_t i = 0; i < shard_n; ++i)
      if (y_host[i] >= shard_classes) return set_error(DS_E_CONTRACT, "dataset: label out of range");
  for (uint64_t i = 0; i < m.P; ++i)
    if (!std::isfinite(init_host[i])) {
      // sgd_step's require_finite(x) would reject the first step (param_vector.cpp:29)
      break;
    }
  if (hp->batch_size > 65535) return set_error(DS_E_CONTRACT, "engine: batch_size above 65535");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) return set_error(DS_E_CUDA, "engine: no CUDA device");
  if (device < 0 || device >= ndev) return set_error(DS_E_CONTRACT, "engine: bad device %d", device);
  dsb::DeviceScope ds(device);
  auto* e = new ds_engine();
  e->device = device;
  e->model = m;
  e->hp = *hp;
  e->shard_n = shard_n;
  e->shard_classes = shard_classes;
  e->seed = sweep_seed;
  e->kind = kind;
  auto fail = [&](int rc) {
    ds_engine_destroy(e);
    return rc;
  };
  const uint64_t F = m.n_features, B = hp->batch_size;
  cudaError_t err = cudaStreamCreateWithFlags(&e->stream, cudaStreamNonBlocking);
  if (err == cudaSuccess) err = cudaMalloc(&e->X, shard_n * F * sizeof(float));
  if (err == cudaSuccess) err = cudaMalloc(&e->y, shard_n * sizeof(uint32_t));
  if (err == cudaSuccess) err = cudaMalloc(&e->params[0], m.P * sizeof(float));
  if (err == cudaSuccess) err = cudaMalloc(&e->params[1], m.P * sizeof(float));
  if (err == cudaSuccess) err = cudaMalloc(&e->grad, m.P * sizeof(float));
  if (err == cudaSuccess) err = cudaMalloc(&e->ws, dsb::layered_workspace_doubles(m, static_cast<uint32_t>(B)) * sizeof(double));
  if (err == cudaSuccess) err = cudaMalloc(&e->st, sizeof(dsb::DevState));
  if (err == cudaSuccess) err = cudaMalloc(&e->bar, 64 * sizeof(unsigned int));
  if (err == cudaSuccess) err = cudaEventCreateWithFlags(&e->plan_ev, cudaEventDisableTiming);
  for (int k = 0; k < 2; ++k) {
    if (err == cudaSuccess) err = cudaMalloc(&e->Xb2[k], B * F * sizeof(float));
    if (err == cudaSuccess) err = cudaMalloc(&e->yb2[k], B * sizeof(uint32_t));
    if (err == cudaSuccess) err = cudaMalloc(&e->rows2[k], sizeof(uint32_t));
    if (err == cudaSuccess) err = cudaEventCreateWithFlags(&e->slot_ev[k], cudaEventDisableTiming);
  }
  e->Xb = e->Xb2[0];
  e->yb = e->yb2[0];
  e->rows_dev = e->rows2[0];
  if (err == cudaSuccess) err = cudaMalloc(&e->iota, B * sizeof(uint32_t));
  if (err == cudaSuccess) {
    std::vector<uint32_t> id(B);
    std::iota(id.begin(), id.end(), 0u);
    err = cudaMemcpy(e->iota, id.data(), B * sizeof(uint32_t), cudaMemcpyHostToDevice);
  }
  if (err == cudaSuccess && !shard_path) err = cudaMemcpy(e->X, X_host, shard_n * F * sizeof(float), cudaMemcpyDefault);
  if (err == cudaSuccess && !shard_path) err = cudaMemcpy(e->y, y_host, shard_n * sizeof(uint32_t), cudaMemcpyDefault);
  if (err == cudaSuccess) err = cudaMemcpy(e->params[0], init_host, m.P * sizeof(float), cudaMemcpyDefault);
  if (err == cudaSuccess) err = cudaMemcpy(e->params[1], init_host, m.P * sizeof(float), cudaMemcpyDefault);
  if (err == cudaSuccess) err = cudaMemset(e->bar, 0, 64 * sizeof(unsigned int));
  if (err != cudaSuccess)
    return fail(set_error(err == cudaErrorMemoryAllocation ? DS_E_NOMEM : DS_E_CUDA, "engine: %s", cudaGetErrorString(err)));
  if (shard_path) {
    ds_shard_info info{};
    const int rc = ds_shard_load(shard_path, e->X, e->y, shard_n, &info, e->stream);
    if (rc != DS_OK) return fail(rc);
    if (info.n_samples != shard_n || info.n_features != F)
      return fail(set_error(DS_E_FORMAT, "%s: changed while loading", shard_path));
  }
  dsb::DevState s0{};
  s0.cut = hp->loss_cut;
  s0.tau = hp->tau;
  s0.adaptive = hp->adaptive ? 1 : 0;
  err = cudaMemcpy(e->st, &s0, sizeof(s0), cudaMemcpyHostToDevice);
  if (err != cudaSuccess) return fail(set_error(DS_E_CUDA, "engine: %s", cudaGetErrorString(err)));
  // ShardSweeper ctor: identity order, reshuffled for epoch 0 (engine.cpp:10-17)
  e->order.resize(shard_n);
  std::iota(e->order.begin(), e->order.end(), 0u);
  dsb::reshuffle(e);
  int rc = dsb::ensure_log(e, hp->i_max);
  if (rc != DS_OK) return fail(rc);
  const char* why = nullptr;
  if (kind == DS_ENGINE_TC) {
    if (dsb::tc_supported(m, static_cast<uint32_t>(B), device, &why) != DS_OK)
      return fail(set_error(DS_E_CONTRACT, "engine: tensor-core path unavailable: %s", why));
    e->fused = true;
    e->tc = true;
    e->tc_nc = dsb::tc_cluster(m);
    const uint64_t pitch = dsb::tc_pitch(static_cast<uint32_t>(F));
    err = cudaMalloc(&e->tc_shard, shard_n * pitch * 2);
    if (err == cudaSuccess) err = cudaMalloc(&e->tc_stage, B * pitch * 2);
    if (err == cudaSuccess) err = cudaMemset(e->tc_stage, 0, B * pitch * 2);
    if (err != cudaSuccess) return fail(set_error(DS_E_NOMEM, "engine: %s", cudaGetErrorString(err)));
    rc = dsb::tc_rows_to_bf16(e->X, shard_n, static_cast<uint32_t>(F), e->tc_shard, e->stream);
    if (rc == DS_OK) rc = dsb::tc_make_map(&e->tm_shard, e->tc_shard, shard_n, static_cast<uint32_t>(F));
    if (rc == DS_OK) rc = dsb::tc_make_map(&e->tm_stage, e->tc_stage, B, static_cast<uint32_t>(F));
    if (rc != DS_OK) return fail(rc);
    *out = e;
    return DS_OK;
  }
  const bool can_fuse = dsb::fused_supported(m, static_cast<uint32_t>(B), device, &why) == DS_OK;
  if (kind == DS_ENGINE_FUSED && !can_fuse) return fail(set_error(DS_E_CONTRACT, "engine: fused path unavailable: %s", why));
  e->fused = (kind == DS_ENGINE_FUSED) || (kind == DS_ENGINE_AUTO && can_fuse);
  if (e->fused) {
    e->fused_grid = dsb::fused_grid(m, device);
    const uint64_t H = m.hidden.empty() ? 0 : m.hidden[0];
    err = cudaMalloc(&e->act, 2 * B * (H ? H : 1) * sizeof(double));
    const size_t xbd = dsb::fused_xb_doubles(m, static_cast<uint32_t>(B), device);
    if (err == cudaSuccess && xbd) err = cudaMalloc(&e->xb64, xbd * sizeof(double));
    if (err != cudaSuccess) return fail(set_error(DS_E_NOMEM, "engine: %s", cudaGetErrorString(err)));
  }
  *out = e;
  return DS_OK;
}

extern "C" int ds_engine_create(ds_engine** out, int device, const ds_model_desc* model, const float* X_host,
                                const uint32_t* y_host, uint64_t shard_n, uint32_t shard_classes, const ds_hyper* hp,
                                uint64_t sweep_seed, const float* init_host, int kind) {
  return engine_create(out, device, model, X_host, y_host, shard_n, shard_classes, hp, sweep_seed, init_host, kind,
                       nullptr);
}

extern "C" int ds_engine_create_from_shard(ds_engine** out, int device, const ds_model_desc* model, const char* path,
                                           const ds_hyper* hp, uint64_t sweep_seed, const float* init_host, int kind) {
  if (!path) return set_error(DS_E_CONTRACT, "engine: null argument");
  ds_shard_info info{};
  DS_TRY(ds_shard_info_read(path, &info));
  dsb::ModelInfo m;
  DS_TRY(dsb::model_from_desc(model, m));
  if (info.n_features != m.n_features)
    return set_error(DS_E_CONTRACT, "engine: shard has %u features, model expects %u", info.n_features, m.n_features);
  return engine_create(out, device, model, nullptr, nullptr, info.n_samples, info.n_classes, hp, sweep_seed, init_host,
                       kind, path);
}

extern "C" int ds_engine_destroy(ds_engine* e) {
  if (!e) return DS_OK;
  dsb::DeviceScope ds(e->device);
  if (e->stream) cudaStreamSynchronize(e->stream);
  if (e->stream) dsb::master_forget_stream(e->stream);
  cudaFree(e->X);
  cudaFree(e->y);
  cudaFree(e->params[0]);
  cudaFree(e->params[1]);
  cudaFree(e->grad);
  cudaFree(e->ws);
  cudaFree(e->act);
  cudaFree(e->xb64);
  cudaFree(e->tc_shard);
  cudaFree(e->tc_stage);
  cudaFree(e->tc_ring);
  cudaFree(e->st);
  cudaFree(e->bar);
  cudaFree(e->plan);
  cudaFree(e->plan_rows);
  cudaFree(e->d_tickets);
  cudaFree(e->velocity);
  if (e->ring_hX) cudaFreeHost(e->ring_hX);
  if (e->tch_ring) cudaFreeHost(e->tch_ring);
  if (e->tch_words) cudaFreeHost(e->tch_words);
  if (e->ring_hy) cudaFreeHost(e->ring_hy);
  if (e->step_graph) cudaGraphExecDestroy(e->step_graph);
  for (auto& g : e->sync_graph)
    if (g) cudaGraphExecDestroy(g);
  cudaFree(e->cur_idx);
  cudaFree(e->step_ctr);
  cudaFree(e->ring_X);
  cudaFree(e->ring_y);
  cudaFree(e->ring_words);
  cudaFreeHost(e->ring_src);
  cudaFreeHost(e->ring_consumed);
  if (e->copy_stream) cudaStreamDestroy(e->copy_stream);
  for (int k = 0; k < 2; ++k) {
    cudaFree(e->Xb2[k]);
    cudaFree(e->yb2[k]);
    cudaFree(e->rows2[k]);
    if (e->slot_ev[k]) cudaEventDestroy(e->slot_ev[k]);
  }
  cudaFree(e->iota);
  if (e->h_plan) cudaFreeHost(e->h_plan);
  if (e->h_rows) cudaFreeHost(e->h_rows);
  cudaFree(e->log.loss);
  cudaFree(e->log.cum);
  cudaFree(e->log.exchanged);
  cudaFree(e->log.period);
  if (e->plan_ev) cudaEventDestroy(e->plan_ev);
  if (e->stream) cudaStreamDestroy(e->stream);
  delete e;
  return DS_OK;
}

extern "C" int ds_engine_attach_master(ds_engine* e, ds_master* m) {
  if (!e) return set_error(DS_E_CONTRACT, "engine: null");
  if (m) {
    uint64_t dim = 0;
    ds_master_dim(m, &dim);
    if (dim != e->model.P) return set_error(DS_E_CONTRACT, "engine: master dim %llu != model dim %llu",
                                            (unsigned long long)dim, (unsigned long long)e->model.P);
    if (m->device != e->device) return set_error(DS_E_CONTRACT, "engine: master lives on another device");
    if (e->sync) return set_error(DS_E_CONTRACT, "engine: synchronous mode replaces the EASGD master");
  }
  if (e->master && e->master != m) dsb::master_remove_client(e->master, e->stream);
  if (m) dsb::master_add_client(m, e->stream);  // in-kernel exchanges run on the engine stream
  e->master = m;
  return DS_OK;
}

extern "C" int ds_engine_set_tickets(ds_engine* e, const uint64_t* tickets, uint64_t count) {
  if (!e) return set_error(DS_E_CONTRACT, "engine: null");
  if (count && e->hp.adaptive)
    return set_error(DS_E_CONTRACT, "engine: deterministic tickets need a Fixed period (adaptive order is value-dependent)");
  dsb::DeviceScope ds(e->device);
  DS_CUDA_TRY(cudaStreamSynchronize(e->stream));
  cudaFree(e->d_tickets);
  e->d_tickets = nullptr;
  e->tickets.assign(tickets, tickets + count);
  if (count) {
    DS_CUDA_TRY(cudaMalloc(&e->d_tickets, count * sizeof(uint64_t)));
    DS_CUDA_TRY(cudaMemcpy(e->d_tickets, tickets, count * sizeof(uint64_t), cudaMemcpyHostToDevice));
  }
  e->host_exchanges = 0;
  return DS_OK;
}

extern "C" int ds_engine_reserve(ds_engine* e, uint64_t steps) {
  if (!e) return set_error(DS_E_CONTRACT, "engine: null");
  dsb::DeviceScope ds(e->device);
  DS_TRY(dsb::ensure_log(e, e->queued + steps));
  if (!e->hostfed) DS_TRY(dsb::ensure_plan(e, steps));
  return DS_OK;
}

extern "C" int ds_engine_run(ds_engine* e, uint64_t steps, int stop_at_exchange, uint64_t* ran_out) {
  if (!e) return set_error(DS_E_CONTRACT, "engine: null");
  dsb::DeviceScope ds(e->device);
  uint64_t done = 0;
  DS_TRY(dsb::ensure_log(e, e->queued + steps));
  const bool ik = dsb::in_kernel_ok(e);
  if (e->hp.adaptive) {
    if (stop_at_exchange) {
      // value-dependent: one iteration at a time, stop once the device policy fired
      while (done < steps) {
        DS_TRY(e->fused ? dsb::run_fused(e, 1, false) : dsb::run_layered(e, 1, false));
        ++done;
        ++e->queued;
        uint32_t fire = 0;
        DS_CUDA_TRY(cudaMemcpyAsync(&fire, &e->st->fire, sizeof(fire), cudaMemcpyDeviceToHost, e->stream));
        DS_CUDA_TRY(cudaStreamSynchronize(e->stream));
        if (fire) break;
      }
    } else if (e->fused && e->master && !ik) {
      for (; done < steps; ++done, ++e->queued) {  // host-ordered master: exchange between launches
        DS_TRY(dsb::run_fused(e, 1, false));
        DS_TRY(dsb::enqueue_exchange(e, e->params[e->cur]));
      }
    } else {
      DS_TRY(e->fused ? dsb::run_fused(e, steps, e->master != nullptr) : dsb::run_layered(e, steps, true));
      done = steps;
      e->queued += steps;
    }
  } else if (!stop_at_exchange && (!e->fused || !e->master || ik)) {
    if (e->fused) {
      DS_TRY(dsb::run_fused(e, steps, e->master != nullptr));
      const uint64_t total = e->host_since + steps;
      e->host_exchanges += total / e->hp.tau;
      e->host_since = static_cast<uint32_t>(total % e->hp.tau);
    } else {
      DS_TRY(dsb::run_layered(e, steps, true));
    }
    done = steps;
    e->queued += steps;
  } else {
    // fixed period, split at the exchange points the host can predict
    while (done < steps) {
      const uint64_t to_fire = e->hp.tau - e->host_since;
      const uint64_t chunk = std::min<uint64_t>(to_fire, steps - done);
      const bool fires = chunk == to_fire;
      if (e->fused) {
        DS_TRY(dsb::run_fused(e, chunk, false));
        e->host_since = fires ? 0 : e->host_since + static_cast<uint32_t>(chunk);
        if (fires) {
          if (!stop_at_exchange && e->master) DS_TRY(dsb::enqueue_exchange(e, e->params[e->cur]));
          ++e->host_exchanges;
        }
      } else {
        DS_TRY(dsb::run_layered(e, chunk, !stop_at_exchange));
      }
      done += chunk;
      e->queued += chunk;
      if (fires && stop_at_exchange) break;
    }
  }
  if (ran_out) *ran_out = done;
  return DS_OK;
}

namespace dsb {
int run_group(ds_engine** engines, uint32_t n, uint64_t steps) {
  if (!engines || n == 0) return set_error(DS_E_CONTRACT, "engine_run_group: no engines");
  if (n > 8) return set_error(DS_E_CONTRACT, "engine_run_group: at most 8 engines per launch");
  ds_engine* e0 = engines[0];
  for (uint32_t i = 0; i < n; ++i) {
    ds_engine* e = engines[i];
    if (!e) return set_error(DS_E_CONTRACT, "engine_run_group: null engine");
    for (uint32_t k = 0; k < i; ++k)
      if (engines[k] == e) return set_error(DS_E_CONTRACT, "engine_run_group: engine listed twice");
    if (!e->tc) return set_error(DS_E_CONTRACT, "engine_run_group: needs tensor-core engines (DS_ENGINE_TC)");
    if (e->device != e0->device || e->model.n_features != e0->model.n_features ||
        e->model.hidden != e0->model.hidden || e->model.n_classes != e0->model.n_classes ||
        e->hp.batch_size != e0->hp.batch_size)
      return set_error(DS_E_CONTRACT, "engine_run_group: engines differ in device, model or batch size");
    if (e->hostfed || e->ring_active != e0->ring_active)
      return set_error(DS_E_STATE, "engine_run_group: engines differ in stream mode");
  }
  if (steps == 0) return DS_OK;
  dsb::DeviceScope ds(e0->device);
  std::vector<dsb::FusedArgs> a(n);
  std::vector<CUtensorMap> tm(n);
  cudaEvent_t ev = nullptr;
  DS_CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  struct EvGuard {
    cudaEvent_t e;
    ~EvGuard() { cudaEventDestroy(e); }
  } guard{ev};
  for (uint32_t i = 0; i < n; ++i) {
    ds_engine* e = engines[i];
    DS_TRY(dsb::ensure_log(e, e->queued + steps));
    DS_TRY(dsb::fused_args(e, steps, e->master != nullptr, a[i]));
    tm[i] = e->ring_active ? e->tm_ring : e->tm_shard;
    if (i) {  // the launch (on engine 0's stream) follows every engine's queued work
      DS_CUDA_TRY(cudaEventRecord(ev, e->stream));
      DS_CUDA_TRY(cudaStreamWaitEvent(e0->stream, ev, 0));
    }
  }
  // DS_FUSED_PROFILE=<file>: per-phase stamps of worker 0's CTA 0 (as run_fused)
  const char* prof_path = std::getenv("DS_FUSED_PROFILE");
  unsigned long long* prof = nullptr;
  const uint64_t prof_n = steps * (kProfSlots + 2 * static_cast<uint64_t>(e0->fused_grid)) + 8;
  if (prof_path && steps >= 8 && !e0->ring_active) {
    DS_CUDA_TRY(cudaMalloc(&prof, prof_n * sizeof(unsigned long long)));
    DS_CUDA_TRY(cudaMemsetAsync(prof, 0, prof_n * sizeof(unsigned long long), e0->stream));
    a[0].prof = prof;
    a[0].prof_cta = prof + steps * kProfSlots;
  }
  DS_TRY(dsb::launch_tc_group(a.data(), tm.data(), n, e0->tc_nc, e0->stream));
  if (prof) DS_TRY(dump_profile(e0, prof, steps, prof_n, prof_path));
  DS_CUDA_TRY(cudaEventRecord(ev, e0->stream));
  for (uint32_t i = 0; i < n; ++i) {
    ds_engine* e = engines[i];
    if (i) DS_CUDA_TRY(cudaStreamWaitEvent(e->stream, ev, 0));  // later work on each engine's stream
    e->launches += 1;
    e->cur ^= static_cast<int>(steps & 1);
    if (!e->hp.adaptive) {
      const uint64_t total = e->host_since + steps;
      e->host_exchanges += total / e->hp.tau;
      e->host_since = static_cast<uint32_t>(total % e->hp.tau);
    }
    e->queued += steps;
  }
  return DS_OK;
}
}  // namespace dsb

extern "C" int ds_engine_run_group(ds_engine** engines, uint32_t n, uint64_t steps) {
  for (uint32_t i = 0; engines && i < n; ++i)
    if (engines[i] && engines[i]->ring_active)
      return set_error(DS_E_STATE, "engine_run_group: an engine is in stream mode");
  return dsb::run_group(engines, n, steps);
}

namespace {
int engine_error(ds_engine* e) {
  dsb::DevState s;
  DS_CUDA_TRY(cudaMemcpy(&s, e->st, sizeof(s), cudaMemcpyDeviceToHost));
  if (!s.err) return DS_OK;
  const unsigned long long it = s.bad_iter;
  const uint32_t f = s.err;
  // the reference's check order: check_inputs, loss/grad finiteness, then sgd_step
  if (f & DS_FLAG_LABEL_RANGE) return set_error(DS_E_CONTRACT, "loss_and_grad: label out of range (iteration %llu)", it);
  if (f & DS_FLAG_LOSS_NONFINITE) return set_error(DS_E_NUMERIC, "loss_and_grad: non-finite loss (iteration %llu)", it);
  if (f & DS_FLAG_GRAD_NONFINITE) return set_error(DS_E_NUMERIC, "loss_and_grad: non-finite gradient (iteration %llu)", it);
  if (f & DS_FLAG_X_NONFINITE) return set_error(DS_E_CONTRACT, "sgd_step: x contains a non-finite value (iteration %llu)", it);
  if (f & DS_FLAG_G_NONFINITE) return set_error(DS_E_CONTRACT, "sgd_step: grad contains a non-finite value (iteration %llu)", it);
  if (f & DS_FLAG_OUT_NONFINITE) return set_error(DS_E_NUMERIC, "sgd_step: non-finite result (iteration %llu)", it);
  if (f & DS_FLAG_TICKET_TIMEOUT)
    return set_error(DS_E_STATE, "exchange: timed out waiting for the previous ticket (a peer worker stopped early "
                     "or died; iteration %llu)", it);
  if (f & DS_FLAG_STREAM_TIMEOUT) return set_error(DS_E_STATE, "stream: no batch from the host for 20 s (iteration %llu)", it);
  return set_error(DS_E_NUMERIC, "engine: failure flags 0x%x (iteration %llu)", f, it);
}
}  // namespace

extern "C" int ds_engine_sync(ds_engine* e) {
  if (!e) return set_error(DS_E_CONTRACT, "engine: null");
  dsb::DeviceScope ds(e->device);
  DS_CUDA_TRY(cudaStreamSynchronize(e->stream));
  return engine_error(e);
}

extern "C" int ds_engine_stream(ds_engine* e, void** stream) {
  if (!e || !stream) return set_error(DS_E_CONTRACT, "engine: null");
  *stream = e->stream;
  return DS_OK;
}

extern "C" int ds_engine_log(ds_engine* e, uint64_t first, uint64_t count, double* batch_loss, double* cumulated,
                             uint8_t* exchanged, uint32_t* period_len) {
  if (!e) return set_error(DS_E_CONTRACT, "engine: null");
  dsb::DeviceScope ds(e->device);
  DS_CUDA_TRY(cudaStreamSynchronize(e->stream));
  if (first + count > e->log.cap) return set_error(DS_E_CONTRACT, "engine_log: rows beyond the log");
  if (batch_loss) DS_CUDA_TRY(cudaMemcpy(batch_loss, e->log.loss + first, count * sizeof(double), cudaMemcpyDeviceToHost));
  if (cumulated) DS_CUDA_TRY(cudaMemcpy(cumulated, e->log.cum + first, count * sizeof(double), cudaMemcpyDeviceToHost));
  if (exchanged) DS_CUDA_TRY(cudaMemcpy(exchanged, e->log.exchanged + first, count, cudaMemcpyDeviceToHost));
  if (period_len) DS_CUDA_TRY(cudaMemcpy(period_len, e->log.period + first, count * sizeof(uint32_t), cudaMemcpyDeviceToHost));
  return DS_OK;
}

extern "C" int ds_engine_iterations(ds_engine* e, uint64_t* iters) {
  if (!e || !iters) return set_error(DS_E_CONTRACT, "engine: null");
  dsb::DeviceScope ds(e->device);
  DS_CUDA_TRY(cudaStreamSynchronize(e->stream));
  dsb::DevState s;
  DS_CUDA_TRY(cudaMemcpy(&s, e->st, sizeof(s), cudaMemcpyDeviceToHost));
  *iters = s.iter;
  return DS_OK;
}

extern "C" int ds_engine_get_params(ds_engine* e, float* host_out) {
  if (!e || !host_out) return set_error(DS_E_CONTRACT, "engine: null");
  dsb::DeviceScope ds(e->device);
  DS_CUDA_TRY(cudaMemcpyAsync(host_out, e->params[e->cur], e->model.P * sizeof(float), cudaMemcpyDeviceToHost, e->stream));
  DS_CUDA_TRY(cudaStreamSynchronize(e->stream));
  return DS_OK;
}

extern "C" int ds_engine_set_params(ds_engine* e, const float* host_in) {
  if (!e || !host_in) return set_error(DS_E_CONTRACT, "engine: null");
  dsb::DeviceScope ds(e->device);
  DS_CUDA_TRY(cudaMemcpyAsync(e->params[e->cur], host_in, e->model.P * sizeof(float), cudaMemcpyDefault, e->stream));
  DS_CUDA_TRY(cudaStreamSynchronize(e->stream));
  return DS_OK;
}

extern "C" int ds_engine_params_device(ds_engine* e, float** dev_ptr) {
  if (!e || !dev_ptr) return set_error(DS_E_CONTRACT, "engine: null");
  *dev_ptr = e->params[e->cur];
  return DS_OK;
}

extern "C" int ds_engine_policy(ds_engine* e, double* cumulated, uint32_t* since_exchange, double* loss_cut) {
  if (!e) return set_error(DS_E_CONTRACT, "engine: null");
  dsb::DeviceScope ds(e->device);
  DS_CUDA_TRY(cudaStreamSynchronize(e->stream));
  dsb::DevState s;
  DS_CUDA_TRY(cudaMemcpy(&s, e->st, sizeof(s), cudaMemcpyDeviceToHost));
  if (cumulated) *cumulated = s.cum;
  if (since_exchange) *since_exchange = s.since;
  if (loss_cut) *loss_cut = s.cut;
  return DS_OK;
}

extern "C" int ds_engine_launches(ds_engine* e, uint64_t* launches) {
  if (!e || !launches) return set_error(DS_E_CONTRACT, "engine: null");
  *launches = e->launches;
  return DS_OK;
}

namespace {
// One host-fed iteration on the next staging slot. Waits (host) only when the slot's
// previous user — the iteration two calls back — has not finished on the device.
int step_host_enqueue(ds_engine* e, const float* X_host, const uint32_t* y_host, uint32_t rows, double* loss_host) {
  if (!e || !X_host || !y_host) return set_error(DS_E_CONTRACT, "engine_step_host: null");
  if (rows == 0) return set_error(DS_E_CONTRACT, "loss_and_grad: empty batch");
  if (rows > e->hp.batch_size) return set_error(DS_E_CONTRACT, "engine_step_host: more rows than batch_size");
  const int k = e->slot;
  e->slot ^= 1;
  if (e->slot_armed[k]) DS_CUDA_TRY(cudaEventSynchronize(e->slot_ev[k]));
  e->Xb = e->Xb2[k];
  e->yb = e->yb2[k];
  e->rows_dev = e->rows2[k];
  const uint64_t F = e->model.n_features;
  DS_CUDA_TRY(cudaMemcpyAsync(e->Xb, X_host, rows * F * sizeof(float), cudaMemcpyDefault, e->stream));
  DS_CUDA_TRY(cudaMemcpyAsync(e->yb, y_host, rows * sizeof(uint32_t), cudaMemcpyDefault, e->stream));
  DS_CUDA_TRY(cudaMemcpyAsync(e->rows_dev, &rows, sizeof(uint32_t), cudaMemcpyHostToDevice, e->stream));
  e->hostfed = true;
  e->hostfed_rows = rows;
  const int rc = ds_engine_run(e, 1, 0, nullptr);
  e->hostfed = false;
  if (rc != DS_OK) return rc;
  DS_CUDA_TRY(cudaEventRecord(e->slot_ev[k], e->stream));
  e->slot_armed[k] = true;
  if (loss_host)  // the loss row of this iteration: st->iter was advanced by the step
    DS_CUDA_TRY(cudaMemcpyAsync(loss_host, e->log.loss + (e->queued - 1), sizeof(double), cudaMemcpyDeviceToHost,
                                e->stream));
  return DS_OK;
}
}  // namespace

extern "C" int ds_engine_step_host(ds_engine* e, const float* X_host, const uint32_t* y_host, uint32_t rows,
                                   double* loss_host) {
  if (!e) return set_error(DS_E_CONTRACT, "engine_step_host: null");
  dsb::DeviceScope ds(e->device);
  DS_TRY(step_host_enqueue(e, X_host, y_host, rows, loss_host));
  if (loss_host) DS_CUDA_TRY(cudaStreamSynchronize(e->stream));
  return DS_OK;
}

extern "C" int ds_engine_step_host_async(ds_engine* e, const float* X_host, const uint32_t* y_host, uint32_t rows,
                                         double* loss_host) {
  if (!e) return set_error(DS_E_CONTRACT, "engine_step_host: null");
  dsb::DeviceScope ds(e->device);
  return step_host_enqueue(e, X_host, y_host, rows, loss_host);
}

// ---- stream mode --------------------------------------------------------------------
extern "C" int ds_engine_attach_sync(ds_engine* e, ds_sync* sg) {
  if (!e) return set_error(DS_E_CONTRACT, "engine: null");
  if (sg && e->fused) return set_error(DS_E_CONTRACT, "engine: synchronous mode needs the layered engine");
  if (sg && e->master) return set_error(DS_E_CONTRACT, "engine: synchronous mode replaces the EASGD master");
  if (sg && e->mu > 0.0f) return set_error(DS_E_CONTRACT, "engine: synchronous mode has no momentum");
  e->sync = sg;
  return DS_OK;
}

extern "C" int ds_engine_set_momentum(ds_engine* e, float mu) {
  if (!e) return set_error(DS_E_CONTRACT, "engine: null");
  if (!(mu >= 0.0f && mu < 1.0f)) return set_error(DS_E_CONTRACT, "sgd_momentum: mu must be in [0,1)");
  if (mu > 0.0f && e->fused) return set_error(DS_E_CONTRACT, "engine: momentum needs the layered engine");
  dsb::DeviceScope ds(e->device);
  if (mu > 0.0f && !e->velocity) {
    DS_CUDA_TRY(cudaMalloc(&e->velocity, e->model.P * sizeof(float)));
    DS_CUDA_TRY(cudaMemsetAsync(e->velocity, 0, e->model.P * sizeof(float), e->stream));
  }
  e->mu = mu;
  return DS_OK;
}

namespace {
// stream mode set-up of one engine (everything but the launch)
int stream_prepare(ds_engine* e, uint64_t steps, double* loss_host) {
  if (!e) return set_error(DS_E_CONTRACT, "engine_stream: null");
  if (e->ring_active) return set_error(DS_E_STATE, "engine_stream: a stream is already open");
  if (!e->fused || e->model.hidden.size() != 1 || (e->model.n_features % 4) != 0)
    return set_error(DS_E_CONTRACT, "engine_stream: needs the fused one-hidden-layer engine and n_features %% 4 == 0");
  // the adaptive policy (engine.cpp:35-48) runs in the kernel; it needs the exchange to be
  // in-kernel too (a host-ordered master would split the launch at value-dependent points)
  if (e->hp.adaptive && e->master && !dsb::in_kernel_ok(e))
    return set_error(DS_E_CONTRACT, "engine_stream: an adaptive policy needs an in-kernel exchange (LockFree or "
                     "sharded master, or a tensor-core engine)");
  if (loss_host) {  // the kernel stores into it directly: it must be mapped (pinned) host memory
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, loss_host) != cudaSuccess || pa.type != cudaMemoryTypeHost) {
      cudaGetLastError();
      return set_error(DS_E_CONTRACT, "engine_stream: loss_host must be pinned host memory (cudaHostAlloc / "
                       "cudaHostRegister), the kernel writes it directly");
    }
  }
  if (steps == 0) return DS_OK;
  dsb::DeviceScope ds(e->device);
  const uint64_t B = e->hp.batch_size, F = e->model.n_features, K = ds_engine::kRing;
  if (!e->ring_consumed)
    DS_CUDA_TRY(cudaHostAlloc(&e->ring_consumed, sizeof(unsigned long long), cudaHostAllocMapped));
  if (!e->tc && !e->ring_X) {
    DS_CUDA_TRY(cudaMalloc(&e->ring_X, K * B * F * sizeof(float)));
    DS_CUDA_TRY(cudaMalloc(&e->ring_y, K * B * sizeof(uint32_t)));
    DS_CUDA_TRY(cudaMalloc(&e->ring_words, 2 * K * sizeof(uint32_t)));
    DS_CUDA_TRY(cudaMallocHost(&e->ring_src, 2 * K * sizeof(uint32_t)));
    DS_CUDA_TRY(cudaStreamCreateWithFlags(&e->copy_stream, cudaStreamNonBlocking));
  }
  if (e->tc && !e->tc_ring) {
    const uint64_t KT = ds_engine::kTcRing, pitch = dsb::tc_pitch(static_cast<uint32_t>(F));
    const uint64_t sb = (B + 1) * pitch * 2;  // bytes per slot
    DS_CUDA_TRY(cudaMalloc(&e->tc_ring, KT * sb));
    DS_CUDA_TRY(cudaMemset(e->tc_ring, 0, KT * sb));
    DS_CUDA_TRY(cudaMalloc(&e->ring_words, KT * sizeof(uint32_t)));
    DS_CUDA_TRY(cudaHostAlloc(&e->tch_ring, KT * sb, cudaHostAllocDefault));
    DS_CUDA_TRY(cudaHostAlloc(&e->tch_words, KT * sizeof(uint32_t), cudaHostAllocDefault));
    std::memset(e->tch_ring, 0, KT * sb);
    DS_CUDA_TRY(cudaStreamCreateWithFlags(&e->copy_stream, cudaStreamNonBlocking));
    DS_TRY(dsb::tc_make_map(&e->tm_ring, e->tc_ring, KT * (B + 1), static_cast<uint32_t>(F)));
  }
  DS_CUDA_TRY(cudaStreamSynchronize(e->stream));
  DS_CUDA_TRY(cudaMemsetAsync(e->ring_words, 0, (e->tc ? ds_engine::kTcRing : 2 * K) * sizeof(uint32_t), e->stream));
  *reinterpret_cast<volatile unsigned long long*>(e->ring_consumed) = 0;
  DS_TRY(dsb::ensure_log(e, e->queued + steps));
  e->ring_active = true;
  e->ring_steps = steps;
  e->ring_pushed = 0;
  e->ring_loss = loss_host;
  return DS_OK;
}
}  // namespace

extern "C" int ds_engine_stream_begin(ds_engine* e, uint64_t steps, double* loss_host) {
  DS_TRY(stream_prepare(e, steps, loss_host));
  if (steps == 0) return DS_OK;
  dsb::DeviceScope ds(e->device);
  const int rc = ds_engine_run(e, steps, 0, nullptr);  // the launch waits on the ring
  if (rc != DS_OK) e->ring_active = false;
  return rc;
}

extern "C" int ds_engine_stream_begin_group(ds_engine** engines, uint32_t n, uint64_t steps, double** loss_host) {
  if (!engines || n == 0 || n > 8) return set_error(DS_E_CONTRACT, "engine_stream_group: 1..8 engines");
  for (uint32_t i = 0; i < n; ++i)
    if (!engines[i] || !engines[i]->tc)
      return set_error(DS_E_CONTRACT, "engine_stream_group: needs tensor-core engines (DS_ENGINE_TC)");
  for (uint32_t i = 0; i < n; ++i) {
    const int rc = stream_prepare(engines[i], steps, loss_host ? loss_host[i] : nullptr);
    if (rc != DS_OK) {
      for (uint32_t k = 0; k < i; ++k) engines[k]->ring_active = false;
      return rc;
    }
  }
  if (steps == 0) return DS_OK;
  const int rc = dsb::run_group(engines, n, steps);
  if (rc != DS_OK)
    for (uint32_t k = 0; k < n; ++k) engines[k]->ring_active = false;
  return rc;
}

namespace {
// stream mode: validate a push and wait until ring slot (step % kRing) is free again (its
// previous step has been read by every CTA, which also means its H2D copy completed)
// wait until ring slot (step % kRing) is free again: step - kRing has been read by every
// CTA (which also means its H2D copy completed)
int wait_slot(ds_engine* e, uint64_t step) {
  const uint64_t K = e->tc ? ds_engine::kTcRing : ds_engine::kRing;
  if (step < K) return DS_OK;
  const auto t0 = std::chrono::steady_clock::now();
  for (uint64_t spin = 0; *reinterpret_cast<volatile unsigned long long*>(e->ring_consumed) < step - K + 1; ++spin) {
    if ((spin & 1023) != 1023) continue;  // the CUDA / clock checks are rare: the word is hot
    if (cudaStreamQuery(e->stream) != cudaErrorNotReady)
      return set_error(DS_E_STATE, "engine_stream_push: the stream kernel is no longer running");
    if (std::chrono::steady_clock::now() - t0 > std::chrono::seconds(30))
      return set_error(DS_E_CUDA, "engine_stream_push: device stopped consuming");
  }
  return DS_OK;
}

// stream mode: validate a push and wait for its slot
int stream_slot_ready(ds_engine* e, uint32_t rows) {
  if (!e->ring_active) return set_error(DS_E_STATE, "engine_stream_push: no open stream");
  if (e->ring_pushed >= e->ring_steps) return set_error(DS_E_STATE, "engine_stream_push: all steps already pushed");
  if (rows == 0 || rows > e->hp.batch_size) return set_error(DS_E_CONTRACT, "engine_stream_push: bad row count");
  return wait_slot(e, e->ring_pushed);
}

// tensor-core engines: gather step `step`'s rows (X + idx[r] * F, or X + r * F when idx is
// null) as bf16 into its slot of the pinned twin, labels in the slot's last row, and set
// the slot's word. The caller waited for the slot; tc_flush moves it to the device.
void tc_fill(ds_engine* e, uint64_t step, const float* X, const uint32_t* y, const uint32_t* idx, uint32_t rows) {
  const uint64_t KT = ds_engine::kTcRing, B = e->hp.batch_size;
  const uint32_t F = e->model.n_features;
  const uint64_t slot = step % KT, pitch = dsb::tc_pitch(F);
  uint16_t* base = e->tch_ring + slot * (B + 1) * pitch;
  if (X == e->hb_src && !e->hb.empty()) {  // the cached bf16 shard: gather_batch as row copies
    for (uint32_t r = 0; r < rows; ++r)
      std::memcpy(base + r * pitch, e->hb.data() + static_cast<uint64_t>(idx ? idx[r] : r) * F, F * sizeof(uint16_t));
  } else {
    dsb::gather_rows_bf16_host(X, F, idx, rows, base, pitch);  // gather_batch + the bf16 operand cast
  }
  uint32_t* lab = reinterpret_cast<uint32_t*>(base + B * pitch);
  for (uint32_t r = 0; r < rows; ++r) lab[r] = y[idx ? idx[r] : r];
  e->tch_words[slot] = (rows << 20) | (static_cast<uint32_t>(step + 1) & 0xFFFFFu);
}

// DMA steps [s0, s1) (one group: contiguous slots) and then their words, on the copy stream
int tc_flush(ds_engine* e, uint64_t s0, uint64_t s1) {
  const uint64_t KT = ds_engine::kTcRing, B = e->hp.batch_size;
  const uint64_t sb = (B + 1) * dsb::tc_pitch(e->model.n_features) * 2, slot0 = s0 % KT, n = s1 - s0;
  DS_CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(e->tc_ring) + slot0 * sb, reinterpret_cast<char*>(e->tch_ring) + slot0 * sb,
                              n * sb, cudaMemcpyHostToDevice, e->copy_stream));
  DS_CUDA_TRY(cudaMemcpyAsync(e->ring_words + slot0, e->tch_words + slot0, n * sizeof(uint32_t), cudaMemcpyHostToDevice,
                              e->copy_stream));
  return DS_OK;
}

int stream_enqueue(ds_engine* e, const float* X_host, const uint32_t* y_host, uint32_t rows) {
  const uint64_t s = e->ring_pushed, K = ds_engine::kRing, B = e->hp.batch_size, F = e->model.n_features;
  if (e->tc) {
    tc_fill(e, s, X_host, y_host, nullptr, rows);
    DS_TRY(tc_flush(e, s, s + 1));
    ++e->ring_pushed;
    return DS_OK;
  }
  const uint64_t slot = s % K;
  // one word carries the row count and the step (mod 2^20; slots are reused kRing steps apart)
  e->ring_src[K + slot] = (rows << 20) | (static_cast<uint32_t>(s + 1) & 0xFFFFFu);
  cudaStream_t cs = e->copy_stream;
  DS_CUDA_TRY(cudaMemcpyAsync(e->ring_X + slot * B * F, X_host, rows * F * sizeof(float), cudaMemcpyDefault, cs));
  DS_CUDA_TRY(cudaMemcpyAsync(e->ring_y + slot * B, y_host, rows * sizeof(uint32_t), cudaMemcpyDefault, cs));
  DS_CUDA_TRY(cudaMemcpyAsync(e->ring_words + K + slot, e->ring_src + K + slot, sizeof(uint32_t),
                              cudaMemcpyHostToDevice, cs));
  ++e->ring_pushed;
  return DS_OK;
}

int push_rows_one(ds_engine* e, const float* X_host, const uint32_t* y_host, const uint32_t* idx, uint32_t rows) {
  DS_TRY(stream_slot_ready(e, rows));
  const uint64_t K = ds_engine::kRing, B = e->hp.batch_size, F = e->model.n_features;
  if (e->tc) {  // gather + bf16 cast straight into the pinned twin, then one DMA
    tc_fill(e, e->ring_pushed, X_host, y_host, idx, rows);
    DS_TRY(tc_flush(e, e->ring_pushed, e->ring_pushed + 1));
    ++e->ring_pushed;
    return DS_OK;
  }
  if (!e->ring_hX) {
    DS_CUDA_TRY(cudaHostAlloc(&e->ring_hX, K * B * F * sizeof(float), cudaHostAllocDefault));
    DS_CUDA_TRY(cudaHostAlloc(&e->ring_hy, K * B * sizeof(uint32_t), cudaHostAllocDefault));
  }
  const uint64_t slot = e->ring_pushed % K;  // free: its previous copy has been consumed
  float* hx = e->ring_hX + slot * B * F;
  uint32_t* hy = e->ring_hy + slot * B;
  for (uint32_t r = 0; r < rows; ++r) {  // gather_batch (model.cpp:12-21) into pinned staging
    std::memcpy(hx + static_cast<uint64_t>(r) * F, X_host + static_cast<uint64_t>(idx[r]) * F, F * sizeof(float));
    hy[r] = y_host[idx[r]];
  }
  return stream_enqueue(e, hx, hy, rows);
}
}  // namespace

extern "C" int ds_engine_stream_push(ds_engine* e, const float* X_host, const uint32_t* y_host, uint32_t rows) {
  if (!e || !X_host || !y_host) return set_error(DS_E_CONTRACT, "engine_stream_push: null");
  dsb::DeviceScope ds(e->device);
  DS_TRY(stream_slot_ready(e, rows));
  return stream_enqueue(e, X_host, y_host, rows);
}

extern "C" int ds_engine_stream_push_rows(ds_engine* e, const float* X_host, const uint32_t* y_host,
                                          const uint32_t* idx, uint32_t rows) {
  if (!e || !X_host || !y_host || !idx) return set_error(DS_E_CONTRACT, "engine_stream_push_rows: null");
  dsb::DeviceScope ds(e->device);
  return push_rows_one(e, X_host, y_host, idx, rows);
}

extern "C" int ds_engine_stream_push_rows_n(ds_engine* e, const float* X_host, const uint32_t* y_host,
                                            const uint32_t* idx, const uint32_t* rows, uint64_t nsteps) {
  if (!e || !X_host || !y_host || !idx || !rows) return set_error(DS_E_CONTRACT, "engine_stream_push_rows_n: null");
  dsb::DeviceScope ds(e->device);
  const uint64_t B = e->hp.batch_size, K = ds_engine::kRing;
  if (!e->ring_active) return set_error(DS_E_STATE, "engine_stream_push: no open stream");
  if (e->ring_pushed + nsteps > e->ring_steps)
    return set_error(DS_E_STATE, "engine_stream_push_rows_n: %llu steps exceed the %llu the stream was opened for",
                     static_cast<unsigned long long>(e->ring_pushed + nsteps),
                     static_cast<unsigned long long>(e->ring_steps));
  for (uint64_t s = 0; s < nsteps; ++s)
    if (rows[s] == 0 || rows[s] > B) return set_error(DS_E_CONTRACT, "engine_stream_push: bad row count at step %llu",
                                                      static_cast<unsigned long long>(s));
  if (!e->tc) {
    for (uint64_t s = 0; s < nsteps; ++s) DS_TRY(push_rows_one(e, X_host, y_host, idx + s * B, rows[s]));
    return DS_OK;
  }
  // groups of kTcGroup steps, one DMA each; T producer threads take groups g = t, t + T, ...
  // (the host's gather is memory-latency bound: one thread cannot keep up with the kernel)
  const uint64_t G = ds_engine::kTcGroup, base = e->ring_pushed;
  uint32_t T = 2;
  if (const char* env = std::getenv("DS_STREAM_FEED_THREADS")) T = static_cast<uint32_t>(std::max(1, std::atoi(env)));
  // groups in flight <= ring slots / G; a group starts at a multiple of G so it never wraps
  const uint64_t first = std::min<uint64_t>(nsteps, (G - base % G) % G);  // steps before the next boundary
  for (uint64_t s = 0; s < first; ++s) DS_TRY(push_rows_one(e, X_host, y_host, idx + s * B, rows[s]));
  const uint64_t rest = nsteps - first, b0 = base + first, ngroups = (rest + G - 1) / G;
  T = static_cast<uint32_t>(std::min<uint64_t>({T, ds_engine::kTcRing / G, std::max<uint64_t>(ngroups, 1)}));
  std::vector<int> rc(T, DS_OK);
  std::vector<std::string> msg(T);
  auto work = [&](uint32_t t) {
    for (uint64_t g = t; g < ngroups; g += T) {
      const uint64_t s0 = b0 + g * G, s1 = std::min(s0 + G, base + nsteps);
      int r = wait_slot(e, s1 - 1);
      for (uint64_t s = s0; r == DS_OK && s < s1; ++s) tc_fill(e, s, X_host, y_host, idx + (s - base) * B, rows[s - base]);
      if (r == DS_OK) r = tc_flush(e, s0, s1);
      if (r != DS_OK) {
        rc[t] = r;
        msg[t] = ds_last_error();
        return;
      }
    }
  };
  std::vector<std::thread> th;
  for (uint32_t t = 1; t < T; ++t) th.emplace_back(work, t);
  work(0);
  for (auto& x : th) x.join();
  e->ring_pushed = base + nsteps;
  for (uint32_t t = 0; t < T; ++t)
    if (rc[t] != DS_OK) return set_error(rc[t], "%s", msg[t].c_str());
  return DS_OK;
}

extern "C" int ds_engine_stream_cache_host_shard(ds_engine* e, const float* X_host, uint64_t n_rows) {
  if (!e) return set_error(DS_E_CONTRACT, "engine_stream_cache_host_shard: null engine");
  if (e->ring_active) return set_error(DS_E_STATE, "engine_stream_cache_host_shard: not while a stream is open");
  if (!X_host || n_rows == 0) {  // drop the cache
    e->hb_src = nullptr;
    e->hb_rows = 0;
    std::vector<uint16_t>().swap(e->hb);
    return DS_OK;
  }
  if (!e->tc) return set_error(DS_E_CONTRACT, "engine_stream_cache_host_shard: needs a tensor-core engine");
  const uint32_t F = e->model.n_features;
  try {
    e->hb.resize(n_rows * F);
  } catch (const std::bad_alloc&) {
    e->hb_src = nullptr;
    return set_error(DS_E_NOMEM, "engine_stream_cache_host_shard: %llu bf16 rows do not fit in host memory",
                     static_cast<unsigned long long>(n_rows));
  }
  // the same cast as the per-step path (gather_rows_bf16_host: RNE, NaN, denormals), split
  // over a few threads
  uint32_t T = 4;
  if (const char* env = std::getenv("DS_STREAM_FEED_THREADS")) T = static_cast<uint32_t>(std::max(1, std::atoi(env)));
  T = static_cast<uint32_t>(std::min<uint64_t>(T, n_rows));
  auto work = [&](uint32_t t) {
    const uint64_t r0 = n_rows * t / T, r1 = n_rows * (t + 1) / T;
    for (uint64_t r = r0; r < r1; r += 65536) {
      const uint32_t n = static_cast<uint32_t>(std::min<uint64_t>(65536, r1 - r));
      dsb::gather_rows_bf16_host(X_host + r * F, F, nullptr, n, e->hb.data() + r * F, F);
    }
  };
  std::vector<std::thread> th;
  for (uint32_t t = 1; t < T; ++t) th.emplace_back(work, t);
  work(0);
  for (auto& x : th) x.join();
  e->hb_src = X_host;
  e->hb_rows = n_rows;
  return DS_OK;
}

extern "C" int ds_engine_stream_end(ds_engine* e) {
  if (!e) return set_error(DS_E_CONTRACT, "engine_stream_end: null");
  if (!e->ring_active) return DS_OK;
  dsb::DeviceScope ds(e->device);
  if (e->ring_pushed < e->ring_steps)
    return set_error(DS_E_STATE, "engine_stream_end: %llu of %llu steps pushed",
                     static_cast<unsigned long long>(e->ring_pushed), static_cast<unsigned long long>(e->ring_steps));
  const cudaError_t err = cudaStreamSynchronize(e->stream);
  if (e->copy_stream) cudaStreamSynchronize(e->copy_stream);
  e->ring_active = false;
  if (e->prof_pending && err == cudaSuccess) {
    unsigned long long* p = e->prof_pending;
    e->prof_pending = nullptr;
    DS_TRY(dsb::dump_profile(e, p, e->prof_steps, e->prof_n, e->prof_path));
  }
  e->ring_loss = nullptr;
  if (err != cudaSuccess) return set_error(DS_E_CUDA, "engine_stream_end: %s", cudaGetErrorString(err));
  return DS_OK;
}
