/*
 * deepspark_c.h — plain-C entry points of the reference-compatible C++ API
 * (libdeepspark_b200.so over include/deepspark/), for FFI hosts (ctypes, cgo, JNI).
 *
 * These mirror the reference's public C++ functions one for one (the names after the
 * dsx_ prefix), exchanging flat caller-owned buffers instead of STL containers. All
 * compute runs on the B200 through include/ds_cuda.h. Status codes are ds_status
 * (0 ok, 1 ContractError, 2 NumericError, 3 CUDA, ...); dsx_last_error() explains.
 */
#ifndef DEEPSPARK_C_H
#define DEEPSPARK_C_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct { /* deepspark::Model (model.hpp) */
  int32_t kind;  /* 0 SoftmaxRegression, 1 Mlp */
  uint32_t n_features;
  uint32_t n_classes;
  uint32_t n_hidden;
  const uint32_t* hidden;
} dsx_model;

typedef struct { /* deepspark::Hyperparams (hyperparams.hpp) */
  double eta;
  double alpha;
  uint32_t tau;
  uint32_t batch_size;
  uint64_t i_max;
  double loss_cut;
  double weight_decay;
  int32_t adaptive;
} dsx_hyper;

typedef struct { /* deepspark::Dataset view */
  const float* X;
  const uint32_t* y;
  uint64_t n;
  uint32_t n_features;
  uint32_t n_classes;
} dsx_data;

typedef struct { /* deepspark::SimConfig (simulator.hpp) */
  uint32_t n_workers;
  dsx_hyper hyper;
  dsx_model model;
  dsx_data data;
  int32_t sync_mode;
  double batch_cost_C;
  double comm_cost_S;
  const double* cost_multipliers;
  uint64_t schedule_seed;
  uint64_t init_seed;
  uint64_t data_seed;
  uint32_t eval_every;
  double holdout_frac;
  int32_t replicate_shards;
  int32_t record_master_snaps;
} dsx_sim_cfg;

typedef struct { /* deepspark::SimResult, flattened (P params, n workers, I = i_max) */
  float* final_master;
  float* worker_final;
  double* batch_loss;
  double* cumulated;
  uint8_t* exchanged;
  uint32_t* period_len;
  int64_t* wall_ms;
  uint64_t snap_cap;
  uint64_t n_snaps;
  uint32_t* snap_worker;
  double* snap_time;
  float* snap_params;
  uint64_t eval_cap;
  uint64_t n_eval;
  double* eval_time;
  uint64_t* eval_iter;
  double* eval_acc;
  double virtual_total;
} dsx_sim_out;

typedef struct { /* LocalRunResult (engine.hpp) */
  float* final_params;
  double* batch_loss;
  double* cumulated;
  uint8_t* exchanged;
  uint32_t* period_len;
} dsx_loop_out;

const char* dsx_last_error(void);
uint64_t dsx_mix_seed(uint64_t seed, uint64_t stream);
void dsx_rng_draws(uint64_t seed, uint64_t n, uint64_t* u64, double* uni, double* nrm, uint64_t bound,
                   uint64_t* below);
uint64_t dsx_param_dim(const dsx_model* m);
uint64_t dsx_fingerprint(const dsx_model* m);
int dsx_init_params(const dsx_model* m, uint64_t seed, float* out);
int dsx_loss_and_grad(const dsx_model* m, const float* params, const float* X, const uint32_t* y, uint32_t rows,
                      float* grad, double* loss);
int dsx_predict(const dsx_model* m, const float* params, const float* X, uint64_t rows, uint32_t* out);
int dsx_accuracy(const dsx_model* m, const float* params, const dsx_data* d, double* acc);
int dsx_sgd_step(const float* x, const float* g, uint64_t n, double eta, float* out);
int dsx_easgd_update(const float* w, const float* m, uint64_t n, double alpha, float* w_out, float* m_out);
int dsx_gen_synthetic(uint32_t n, uint32_t f, uint32_t c, double sep, double sigma, uint64_t seed, float* X,
                      uint32_t* y);
int dsx_split_holdout_order(uint64_t n, double frac, uint64_t seed, uint32_t* order, uint64_t* n_hold);
int dsx_partition_order(uint64_t n, uint32_t k, uint64_t seed, uint32_t* order);
int dsx_sweep_batches(uint64_t shard_n, uint32_t batch, uint64_t seed, uint64_t n_batches, uint32_t* idx,
                      uint32_t* sizes);
int dsx_engine_steps(const dsx_model* m, const dsx_data* shard, const dsx_hyper* hp, uint64_t sweep_seed,
                     const float* init, uint64_t steps, float* params, double* losses);
/* exchange_mode: 0 none, 1 identity ExchangeFn (host callback path), 2 device MasterState
 * (Locked, alpha = f32(hp.alpha)) initialised from / written back to master_inout. */
int dsx_run_training_loop(const dsx_model* m, const dsx_data* shard, const dsx_hyper* hp, uint64_t sweep_seed,
                          const float* init, int exchange_mode, float* master_inout, dsx_loop_out* out);
/* run_worker (worker.hpp) against a device center: the center is created from
 * master_init with the model `master_model` bound to it (its handshake config: dim,
 * fingerprint, alpha = f32(master_alpha)), mode 0 Locked / 1 LockFree. worker_model NULL
 * = infer softmax from the shard. metrics_path NULL or "" = no dump. On return (also on
 * the handshake errors, which leave the center untouched) master_out receives the
 * center's snapshot and *master_exchanges its exchange count (either may be NULL). */
int dsx_run_worker(const dsx_model* master_model, double master_alpha, int master_mode, const float* master_init,
                   const dsx_model* worker_model, const char* shard_path, const dsx_hyper* hp, uint32_t worker_id,
                   uint64_t rng_seed, const char* metrics_path, float* master_out, uint64_t* master_exchanges,
                   dsx_loop_out* out);
int dsx_resolve_loss_cut(const dsx_model* m, const dsx_data* shard, const dsx_hyper* hp, uint64_t sweep_seed,
                         const float* init, double* cut);
int dsx_simulate(const dsx_sim_cfg* cfg, dsx_sim_out* out);
/* exchange_order (simulator.hpp): the global (worker, iteration) exchange sequence of
 * simulate_async for a Fixed period; *count = total (entries beyond cap not written). */
int dsx_exchange_order(uint32_t n_workers, double batch_cost_C, double comm_cost_S, const double* mults,
                       uint32_t tau, uint64_t i_max, uint64_t schedule_seed, uint32_t* worker, uint64_t* iteration,
                       uint64_t cap, uint64_t* count);

#ifdef __cplusplus
}
#endif

#endif /* DEEPSPARK_C_H */
