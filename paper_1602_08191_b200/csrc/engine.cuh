// engine.cuh — device-resident SgdEngine / run_training_loop state (engine.hpp:17-105).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "ds_cuda.h"
#include "master.cuh"
#include "model.cuh"

namespace dsb {

// ExchangePolicy + loop bookkeeping, resident on the device (engine.hpp:40-59).
struct DevState {
  double cum;              // cumulated loss L since the last exchange
  double cut;              // resolved loss_cut (Adaptive)
  double loss;             // batch loss of the step in flight
  unsigned long long iter; // completed iterations (TrainRecord.iter of the last row)
  unsigned long long bad_iter;  // first failing iteration (1-based); 0 = none
  unsigned long long exchanges; // exchanges this worker performed
  uint32_t since;          // iterations since the last exchange
  uint32_t fire;           // the policy fired on the step in flight
  uint32_t flags;          // DS_FLAG_* raised by the step in flight
  uint32_t err;            // sticky copy of the first failing step's flags (gate)
  uint32_t tau;
  int32_t adaptive;
  uint32_t period;
  uint32_t pad;
};

struct DevLog {
  double* loss;
  double* cum;
  uint8_t* exchanged;
  uint32_t* period;
  unsigned long long cap;
};

// Arguments of the fused persistent step kernel (mlp_fused.cu).
struct FusedArgs {
  // model: n_hidden == 0 (softmax) or 1 (one tanh layer)
  uint32_t F, H, C;     // features, hidden width (0 = softmax regression), classes
  uint64_t P;
  const float* X;       // shard, row-major [shard_n x F]
  const uint32_t* y;
  const uint32_t* plan; // steps x B shard-local row indices
  const uint32_t* plan_rows;  // rows per step
  uint32_t B;           // batch stride of the plan
  uint64_t steps;
  float* params[2];     // ping-pong parameter buffers; step s reads [cur], writes [cur^1]
  int cur;
  double* act;          // [2][H x B] hidden activations (ping-pong), f64, unit-major
  double* xb64;         // [3][nck][B][CW] f64 copies of the batch rows (MLP kernel)
  float eta, wd, alpha;
  DevState* st;
  DevLog log;
  // exchange
  int has_master;
  ShardTable table;
  int lockfree;               // plain stores, no tickets
  int center_local;           // the center and its control words are touched by this GPU only (gpu-scope fences)
  const uint64_t* tickets;    // per-exchange global tickets (deterministic), or null
  unsigned long long* ticket_src;  // Locked: dispenser (shard 0 flags.next_ticket)
  int stop_at_exchange;
  unsigned int* bar;          // grid barrier words [2]
  unsigned long long* prof;   // optional: kProfSlots globaltimer stamps per step (CTA 0)
  unsigned long long* prof_cta;  // optional: [step][CTA][2] forward-done / grid-barrier-exit stamps
  // stream mode (host-fed ring; MLP kernel only)
  int ring;
  uint32_t ring_slots;
  const float* ring_X;              // [slots][B][F]
  const uint32_t* ring_y;           // [slots][B]
  const uint32_t* ring_rows;        // [slots]
  const uint32_t* ring_ready;       // [slots] sequence words (step + 1), written by the copy engine
  uint32_t ring_slot_rows;          // TC ring: rows per slot (B + 1: the labels ride in the last)
  uint32_t ring_y_stride;           // TC ring: u32 stride between slots' labels
  unsigned long long* ring_consumed;  // pinned host: steps whose ring slot is free again
  double* ring_loss;                // pinned host: per-step batch loss (zero-copy), or null
};

constexpr int kProfSlots = 10;

int fused_supported(const ModelInfo& m, uint32_t batch, int device, const char** why);
// mlp_tc.cu: the tensor-core (bf16 tcgen05, tolerance) fast step, one cluster per worker.
int tc_supported(const ModelInfo& m, uint32_t batch, int device, const char** why);
int tc_cluster(const ModelInfo& m);
size_t tc_smem_bytes(const ModelInfo& m, uint32_t batch);
int launch_tc(const FusedArgs& a, int nc, const CUtensorMap& batch_rows, cudaStream_t s);
// n workers (engines) in one cooperative launch, one cluster each (n <= 8)
int launch_tc_group(const FusedArgs* a, const CUtensorMap* batch_rows, uint32_t n, int nc, cudaStream_t s);
// the tensor-core step reads batches as bf16 rows of tc_pitch(F) elements through a TMA map
uint32_t tc_pitch(uint32_t F);
// host_rows.cpp: gather + bf16 cast of host rows (the zero-copy stream ring's producer);
// idx == nullptr: X is the batch itself
void gather_rows_bf16_host(const float* X, uint32_t F, const uint32_t* idx, uint32_t rows, uint16_t* dst,
                           uint64_t pitch);
int tc_rows_to_bf16(const float* src, uint64_t rows, uint32_t F, void* dst, cudaStream_t s);
int tc_make_map(CUtensorMap* m, const void* base, uint64_t rows, uint32_t F);
// Doubles of the f64 batch buffer (A.xb64) the MLP kernel needs.
size_t fused_xb_doubles(const ModelInfo& m, uint32_t batch, int device);
int launch_fused(const FusedArgs& a, int grid, cudaStream_t s);
int fused_grid(const ModelInfo& m, int device);
size_t fused_smem_bytes(const ModelInfo& m, uint32_t batch);

}  // namespace dsb
