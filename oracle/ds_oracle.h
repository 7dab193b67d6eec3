/*
 * ds_oracle.h — TEST INFRASTRUCTURE ONLY (not product code).
 *
 * The C interface shared by the two CPU checkers of the DeepSpark EASGD hot path:
 *
 *   dso_*   — ds_oracle.c, a plain-C restatement of the reference algorithm
 *             (/root/reference/proj/src/{param_vector,model,engine,dataset,simulator}.cpp).
 *   dsref_* — ref_capi.cpp, a thin extern "C" wrapper over the UNMODIFIED reference
 *             library compiled from /root/reference into oracle/_ref/ (see Makefile).
 *
 * Both implement the same functions with the same meaning, so tests can pin the
 * restatement against the reference bit for bit and then use either as the checker.
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load these libraries; the product (paper_1602_08191_b200/) never does.
 *
 * Status codes: 0 ok, 1 ContractError, 2 NumericError, 3 other. The message of the
 * last failure is available from <prefix>_last_error().
 */
#ifndef DS_ORACLE_H
#define DS_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Model structure (reference: model.hpp:32-56). kind 0 = softmax regression, 1 = MLP. */
typedef struct {
  int32_t kind;
  uint32_t n_features;
  uint32_t n_classes;
  uint32_t n_hidden;
  const uint32_t* hidden;
} dso_model;

/* Hyperparams (reference: hyperparams.hpp:10-21). */
typedef struct {
  double eta;
  double alpha;
  uint32_t tau;
  uint32_t batch_size;
  uint64_t i_max;
  double loss_cut;
  double weight_decay;
  int32_t adaptive; /* PeriodMode::Adaptive when nonzero */
} dso_hyper;

/* Row-major dataset view (reference: dataset.hpp:12-23). */
typedef struct {
  const float* X;
  const uint32_t* y;
  uint64_t n;
  uint32_t n_features;
  uint32_t n_classes;
} dso_data;

/* SimConfig (reference: simulator.hpp:24-54). */
typedef struct {
  uint32_t n_workers;
  dso_hyper hyper;
  dso_model model;
  dso_data data;
  int32_t sync_mode; /* SimMode::Synchronous when nonzero, else AsyncEASGD */
  double batch_cost_C;
  double comm_cost_S;
  const double* cost_multipliers; /* n_workers entries or NULL */
  uint64_t schedule_seed;
  uint64_t init_seed;
  uint64_t data_seed;
  uint32_t eval_every;
  double holdout_frac;
  int32_t replicate_shards;
  int32_t record_master_snaps;
} dso_sim_cfg;

/* SimResult, flattened into caller-owned buffers (reference: simulator.hpp:73-82).
 * P = param_dim, n = n_workers, I = i_max. Any pointer may be NULL to skip it. */
typedef struct {
  float* final_master;  /* P */
  float* worker_final;  /* n*P */
  double* batch_loss;   /* n*I, per-worker TrainLog rows */
  double* cumulated;    /* n*I */
  uint8_t* exchanged;   /* n*I */
  uint32_t* period_len; /* n*I */
  int64_t* wall_ms;     /* n*I */
  uint64_t snap_cap;    /* capacity of the snap arrays */
  uint64_t n_snaps;     /* out: total snaps (may exceed snap_cap; extra not stored) */
  uint32_t* snap_worker;
  double* snap_time;
  float* snap_params;   /* snap_cap*P */
  uint64_t eval_cap;
  uint64_t n_eval;      /* out */
  double* eval_time;
  uint64_t* eval_iter;
  double* eval_acc;
  double virtual_total; /* out */
} dso_sim_out;

/* run_training_loop (reference: engine.cpp:84-113). exchange_mode: 0 = nullptr
 * ExchangeFn, 1 = identity, 2 = in-process master with elastic_update_elem at
 * float(alpha) (the local-master oracle of test_worker.cpp:131-137 /
 * test_simulator.cpp:117-124); master_inout holds the master (P floats) for mode 2. */
typedef struct {
  float* final_params;  /* P */
  double* batch_loss;   /* I */
  double* cumulated;    /* I */
  uint8_t* exchanged;   /* I */
  uint32_t* period_len; /* I */
} dso_loop_out;

#define DSO_DECLARE(P)                                                                        \
  const char* P##_last_error(void);                                                          \
  uint64_t P##_mix_seed(uint64_t seed, uint64_t stream);                                      \
  /* first n draws of Rng(seed): next_u64, uniform(), normal(), below(bound) */               \
  void P##_rng_draws(uint64_t seed, uint64_t n, uint64_t* u64, double* uni, double* nrm,      \
                     uint64_t bound, uint64_t* below);                                        \
  uint64_t P##_param_dim(const dso_model* m);                                                 \
  uint64_t P##_fingerprint(const dso_model* m);                                               \
  int P##_init_params(const dso_model* m, uint64_t seed, float* out);                         \
  int P##_loss_and_grad(const dso_model* m, const float* params, const float* X,              \
                        const uint32_t* y, uint32_t rows, float* grad, double* loss);         \
  int P##_predict(const dso_model* m, const float* params, const float* X, uint64_t rows,     \
                  uint32_t* out);                                                             \
  int P##_accuracy(const dso_model* m, const float* params, const dso_data* d, double* acc);  \
  int P##_sgd_step(const float* x, const float* g, uint64_t n, double eta, float* out);       \
  int P##_easgd_update(const float* w, const float* m, uint64_t n, double alpha, float* w_out, \
                       float* m_out);                                                         \
  int P##_gen_synthetic(uint32_t n, uint32_t f, uint32_t c, double sep, double sigma,         \
                        uint64_t seed, float* X, uint32_t* y);                                \
  /* split_holdout: order[0:n_hold) -> holdout rows, order[n_hold:) -> train rows */          \
  int P##_split_holdout_order(uint64_t n, double frac, uint64_t seed, uint32_t* order,        \
                              uint64_t* n_hold);                                              \
  /* partition: shard k takes order[pos_k : pos_k + count_k) */                               \
  int P##_partition_order(uint64_t n, uint32_t k, uint64_t seed, uint32_t* order);            \
  /* ShardSweeper: n_batches successive batches; idx[b*batch + j], sizes[b] */                \
  int P##_sweep_batches(uint64_t shard_n, uint32_t batch, uint64_t seed, uint64_t n_batches,  \
                        uint32_t* idx, uint32_t* sizes);                                      \
  int P##_engine_steps(const dso_model* m, const dso_data* shard, const dso_hyper* hp,        \
                       uint64_t sweep_seed, const float* init, uint64_t steps, float* params, \
                       double* losses);                                                       \
  int P##_run_training_loop(const dso_model* m, const dso_data* shard, const dso_hyper* hp,   \
                            uint64_t sweep_seed, const float* init, int exchange_mode,        \
                            float* master_inout, dso_loop_out* out);                          \
  int P##_resolve_loss_cut(const dso_model* m, const dso_data* shard, const dso_hyper* hp,    \
                           uint64_t sweep_seed, const float* init, double* cut);              \
  int P##_simulate(const dso_sim_cfg* cfg, dso_sim_out* out);

DSO_DECLARE(dso)
DSO_DECLARE(dsref)

/* Reference-only timing helpers (used by bench.py --impl reference / cpu_baseline). */
/* MasterState::exchange (exchanger.cpp:76-92) on `threads` host threads, each doing
 * `iters` exchanges of a P-float worker vector; returns seconds elapsed. */
double dsref_master_exchange_time(uint64_t P, int lockfree, int threads, int iters);
/* n worker threads (SgdEngine + ExchangePolicy + one in-process MasterState): wall
 * seconds of `steps` timed iterations per worker after `warmup`; -1 on error. */
double dsref_workers_time(const dso_model* m, const dso_data* shards, uint32_t n_workers,
                          const dso_hyper* hp, const float* init, int lockfree, uint64_t warmup,
                          uint64_t steps, double* losses_out);

#ifdef __cplusplus
}
#endif

#endif /* DS_ORACLE_H */
