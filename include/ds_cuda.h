/*
 * ds_cuda.h — the C-ABI drop-in boundary of the B200-native DeepSpark EASGD hot path.
 *
 * Plain C: no exceptions, no STL, no torch types. Device pointers are CUDA device
 * addresses (local or peer-mapped); `stream` is a cudaStream_t passed as void* (NULL =
 * the legacy default stream). Every entry point returns a ds_status; the message of
 * the last failure on the calling thread is available from ds_last_error(). The C++
 * API in include/deepspark/ (the reference's own headers' surface) sits on top of this
 * and maps DS_E_CONTRACT -> deepspark::ContractError and DS_E_NUMERIC ->
 * deepspark::NumericError, as the reference throws them.
 *
 * Each entry point names the reference interface it replaces (file:line under
 * /root/reference/proj/). There is no CPU fallback behind any of them: a missing GPU
 * or a CUDA failure is DS_E_CUDA.
 */
#ifndef DS_CUDA_H
#define DS_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------------------------- */
/* Status                                                                             */
/* ---------------------------------------------------------------------------------- */
typedef enum {
  DS_OK = 0,
  DS_E_CONTRACT = 1, /* deepspark::ContractError  (errors.hpp:10-13)  */
  DS_E_NUMERIC = 2,  /* deepspark::NumericError   (errors.hpp:16-19)  */
  DS_E_CUDA = 3,     /* CUDA runtime / driver failure, or no device      */
  DS_E_NOMEM = 4,    /* device allocation failed                         */
  DS_E_STATE = 5,    /* handle used in a state that does not allow it    */
  DS_E_FORMAT = 6,   /* deepspark::FormatError    (errors.hpp:33-36)  */
  DS_E_IO = 7        /* deepspark::IoError        (errors.hpp:56-59)  */
} ds_status;

const char* ds_last_error(void);
const char* ds_version(void);
/* Number of visible CUDA devices (0 when none); DS_E_CUDA if the runtime fails. */
int ds_device_count(int* count);

/* Finiteness flags written by the update kernels (OR-ed, device uint32). */
#define DS_FLAG_X_NONFINITE 1u    /* sgd_step: x contains a non-finite value   (param_vector.cpp:29) */
#define DS_FLAG_G_NONFINITE 2u    /* sgd_step: grad contains a non-finite value (param_vector.cpp:30) */
#define DS_FLAG_OUT_NONFINITE 4u  /* sgd_step: non-finite result              (param_vector.cpp:34-35) */
#define DS_FLAG_LOSS_NONFINITE 8u /* loss_and_grad: non-finite loss            (model.cpp:256) */
#define DS_FLAG_GRAD_NONFINITE 16u /* loss_and_grad: non-finite gradient       (model.cpp:259) */
#define DS_FLAG_LABEL_RANGE 32u   /* loss_and_grad: label out of range         (model.cpp:176-180) */
#define DS_FLAG_STREAM_TIMEOUT 64u /* stream mode: no batch from the host for 20 s                  */
#define DS_FLAG_TICKET_TIMEOUT 128u /* ordered exchange: the previous ticket never completed (30 s) */

/* ---------------------------------------------------------------------------------- */
/* Elementwise updates — param_vector.hpp:21-38                                       */
/* ---------------------------------------------------------------------------------- */

/* In-place elastic update, one fused pass: e = a*(w-m); w -= e; m += e, each step one
 * f32 rounding (no FMA contraction) — elastic_update_elem (param_vector.hpp:34-38) over
 * a vector, i.e. easgd_update (param_vector.cpp:41-57) without the allocations.
 * alpha is the f32 moving rate; callers holding a double convert with (float)alpha as
 * the reference does (param_vector.cpp:50). 16 bytes of HBM traffic per element. */
int ds_elastic_update(float* w, float* m, uint64_t n, float alpha, void* stream);

/* MasterState::exchange (exchanger.cpp:76-92) against a plain device vector `master`:
 * out[i] = w'[i], master[i] = m'[i]. `out` may equal `worker` (in place). */
int ds_elastic_exchange(const float* worker, float* master, float* out, uint64_t n, float alpha,
                        void* stream);

/* SGD with the engine's optional L2 fold (engine.cpp:75-79 + param_vector.cpp:21-39):
 *   g' = wd > 0 ? g + f32(wd)*x : g;   out = x - f32(eta)*g'
 * in f32 with separate roundings. `out` may equal `x`. Non-finite conditions are OR-ed
 * into *flags_dev (DS_FLAG_*); the vector is still written, the caller decides. */
int ds_sgd_update(float* out, const float* x, const float* g, uint64_t n, float eta, float wd,
                  uint32_t* flags_dev, void* stream);

/* Synchronous helper with the reference's exact error behaviour for one sgd_step call:
 * DS_E_CONTRACT on eta <= 0 or non-finite x/g, DS_E_NUMERIC on non-finite output. */
int ds_sgd_step_checked(float* out, const float* x, const float* g, uint64_t n, double eta,
                        void* stream);

/* Momentum SGD — NOT IN THE REFERENCE (Hyperparams has no momentum), the
 * Caffe solver's form: g' = g + f32(wd)*x; v = mu*v + g'; out = x - f32(eta)*v, f32 with
 * separate roundings. mu == 0 is bit-identical to ds_sgd_update. `velocity` (device,
 * n floats, zero-initialised by the caller) is updated in place. */
int ds_sgd_momentum_update(float* out, const float* x, float* velocity, const float* g, uint64_t n,
                           float eta, float mu, float wd, uint32_t* flags_dev, void* stream);

/* ---------------------------------------------------------------------------------- */
/* Synchronous data-parallel SGD — simulator.cpp:156-223 (and its NCCL form)          */
/* ---------------------------------------------------------------------------------- */

/* gsum[i] += (double)g[i] — the f64 gradient sum of simulate_sync (simulator.cpp:195). */
int ds_grad_accumulate(double* gsum, const float* g, uint64_t n, void* stream);
/* out[i] = (float)(gsum[i] / n_workers), then out[i] += f32(wd)*x[i] when wd > 0
 * (simulator.cpp:204-208). x may be NULL when wd == 0. */
int ds_grad_average(float* out, const double* gsum, uint64_t n, uint32_t n_workers, float wd,
                    const float* x, void* stream);

/* Multi-GPU synchronous SGD, one process per GPU (simulate_sync, simulator.cpp:156-223,
 * as the reference's "allreduce each iteration"), as a worker-ordered reduce-scatter +
 * all-gather over NVLink fused with the update: rank r owns the 128-byte aligned slice r;
 * ds_sync_reduce_update sums every rank's gradient for that slice in f64 in worker order
 * (simulator.cpp:192-200), divides by world, folds f32(wd)*x (205-207), applies sgd_step to
 * its slice of `params` (the rank's replica of the master) and publishes it; then every
 * rank copies the peers' new slices. Bit-identical to the single-process reference and on
 * all ranks. NVLink bytes per rank and round: 2 (world-1)/world x 4 dim.
 *   create -> export (256-byte record) -> all-gather records -> attach
 *   per round: ds_sync_begin -> write the local gradient into *grad_slot on `stream` ->
 *   ds_sync_reduce_update(params, ...) on the same stream.
 * Peer waits are bounded (30 s -> DS_FLAG_TICKET_TIMEOUT). Non-finite conditions are
 * OR-ed into *flags_dev (DS_FLAG_*). world <= 8. Ranks of one process may share a device
 * only through the *_group entry points (one kernel for all of them — never separate
 * launches that wait on each other). */
typedef struct ds_sync ds_sync;
int ds_sync_create(ds_sync** out, int device, uint64_t dim, int rank, int world);
int ds_sync_export(ds_sync* s, void* record_out);
int ds_sync_attach(ds_sync* s, const void* records);
int ds_sync_begin(ds_sync* s, float** grad_slot, void* stream);
int ds_sync_reduce_update(ds_sync* s, float* params, float eta, float wd, uint32_t* flags_dev, void* stream);
/* Synchronous EASGD (EXTENSION — not in the reference; the EASGD paper's synchronous
 * variant, sharing the async path's elastic arithmetic param_vector.cpp:41-61): every
 * rank holds a replica of the center `center` and its worker vector `worker`; one round:
 *   e_k = f32(alpha * f32(x_k - c))        (all k, the OLD center)
 *   x_k' = x_k - e_k                       (each rank its own worker)
 *   c'   = c + f32(sum_k e_k in f64, worker order)
 * Begins its own round (no ds_sync_begin). */
int ds_sync_easgd_update(ds_sync* s, float* worker, float* center, float alpha, uint32_t* flags_dev, void* stream);
/* Ranks 0..n-1 of one group living in THIS process on ONE device: one launch reduces every
 * slice and writes every replica (params[k] / centers[k], workers[k]). Each rank's round
 * must have been begun (ds_sync_begin, gradients written) for the SGD form. */
int ds_sync_reduce_update_group(ds_sync** group, uint32_t n, float** params, float eta, float wd,
                                uint32_t* flags_dev, void* stream);
int ds_sync_easgd_update_group(ds_sync** group, uint32_t n, float** workers, float** centers, float alpha,
                               uint32_t* flags_dev, void* stream);
/* NVLink read probe with the all-gather's access pattern: n floats split evenly over every
 * peer's exported region (<= 6 dim per peer), copied into dst (16-byte aligned). Timing
 * it on all ranks concurrently gives the in-run NVLink peak the round is judged against. */
int ds_sync_peer_read(ds_sync* s, float* dst, uint64_t n, void* stream);
int ds_sync_rounds(ds_sync* s, uint64_t* out);
int ds_sync_destroy(ds_sync* s);

/* Row gather for host-free minibatches (model.cpp:12-21 gather_batch on the device):
 * dst[r, :] = X[idx[r], :] for r < rows, f32 rows of `features`; y_dst[r] = y[idx[r]]. */
int ds_gather_rows(float* dst, uint32_t* y_dst, const float* X, const uint32_t* y, const uint32_t* idx,
                   uint32_t rows, uint32_t features, void* stream);

/* ---------------------------------------------------------------------------------- */
/* Device plumbing for hosts that do not link the CUDA runtime (C++/Go/Java/Python)   */
/* D[M x N] = relu?( scale * A[M x K] . B[N x K]^T + bias_n[col] + bias_m[row] ) on the
 * tcgen05 tensor cores (kind::tf32, f32 accumulation in TMEM; TMA SWIZZLE_128B tiles).
 * A, B row-major with leading dimensions lda, ldb (multiples of 4, 16-byte aligned).
 * Biases and ReLU optional (NULL / 0). splits > 1 cuts K into that many ranges whose
 * partials (part: splits*M*N floats) are summed in a fixed order; D dense then. The
 * contraction of the AlexNet-shaped convnet's convolution and FC layers (config 4; no
 * reference counterpart). */
int ds_gemm_tf32(const float* A, uint64_t lda, const float* B, uint64_t ldb, float* D, uint64_t ldd, uint32_t M,
                 uint32_t N, uint32_t K, float scale, const float* bias_n, const float* bias_m, int relu,
                 uint32_t splits, float* part, void* stream);

/* ---------------------------------------------------------------------------------- */
/* DSHD shards (shard.hpp:9-35, shard.cpp:75-125)                                     */
/* ---------------------------------------------------------------------------------- */
typedef struct ds_shard_info {
  uint32_t n_samples;
  uint32_t n_features;
  uint32_t n_classes;
  uint64_t seed; /* provenance seed (ShardData::seed) */
} ds_shard_info;
/* Header of a DSHD file, validated like read_shard (magic, version, dimensions, size
 * arithmetic against the file length): DS_E_FORMAT / DS_E_IO with the reference's messages. */
int ds_shard_info_read(const char* path, ds_shard_info* info);
/* read_shard straight into device memory on the calling thread's current device: X_dev
 * f32 [n x F] row-major, y_dev u32 [n] (capacity_rows >= n). The body streams through
 * pinned double buffers and async copies and is unpacked and label-checked on the GPU;
 * returns after the data is resident. A label >= n_classes is DS_E_FORMAT ("label L out
 * of range at sample i"). */
int ds_shard_load(const char* path, float* X_dev, uint32_t* y_dev, uint64_t capacity_rows, ds_shard_info* info_out,
                  void* stream);

/* ---------------------------------------------------------------------------------- */
int ds_device_alloc(int device, uint64_t bytes, void** out);
int ds_device_free(void* p);
/* Copy in any direction (unified addressing). stream == NULL: synchronous. */
int ds_memcpy(void* dst, const void* src, uint64_t bytes, void* stream);
int ds_memset(void* dst, int value, uint64_t bytes, void* stream);
int ds_stream_create(int device, void** stream);
int ds_stream_destroy(void* stream);
int ds_stream_sync(void* stream);

/* ---------------------------------------------------------------------------------- */
/* Model — model.hpp:32-76                                                            */
/* ---------------------------------------------------------------------------------- */
/* kind 2: Caffe cifar10_quick on CHW 3x32x32 rows (n_features 3072, n_hidden 0) —
 * NOT IN THE REFERENCE; same flat W-then-b layout, init and loss
 * conventions, f32 arithmetic (tolerance parity vs the f64 oracle, not bit-exact). */
#define DS_MODEL_CIFAR10_QUICK 2
/* AlexNet-shaped convnet (BASELINE config 4, NOT IN THE REFERENCE): n_features = 3*S*S
 * (S = 224 for the config; S >= 55), n_hidden = 0; tf32 tensor-core GEMMs (alexnet.cu). */
#define DS_MODEL_ALEXNET 3
typedef struct {
  int32_t kind;          /* 0 = SoftmaxRegression, 1 = Mlp (model.hpp:13), 2 = cifar10_quick */
  uint32_t n_features;
  uint32_t n_classes;
  uint32_t n_hidden;     /* number of tanh hidden layers                            */
  const uint32_t* hidden; /* host array of n_hidden layer widths                    */
} ds_model_desc;

/* Model::param_dim (model.cpp:123-129); DS_E_CONTRACT on an invalid model (model.cpp:44-57). */
int ds_param_dim(const ds_model_desc* model, uint64_t* dim);

/* Bytes of device workspace loss_and_grad needs for `rows` samples. */
int ds_loss_and_grad_workspace(const ds_model_desc* model, uint32_t rows, uint64_t* bytes);

/* loss_and_grad / loss_only (model.cpp:242-275), f64 internals with the reference's
 * per-element summation order, gradient rounded once to f32. All pointers are device
 * pointers: params[P], X[rows*n_features] row-major f32, y[rows] u32, grad[P] (NULL =
 * loss_only semantics), loss_out one double. Asynchronous; label-range and finiteness
 * violations are OR-ed into *flags_dev (may be NULL). `workspace` must hold
 * ds_loss_and_grad_workspace bytes. */
int ds_loss_and_grad(const ds_model_desc* model, const float* params, const float* X,
                     const uint32_t* y, uint32_t rows, float* grad, double* loss_out,
                     void* workspace, uint32_t* flags_dev, void* stream);

/* predict (model.cpp:303-318) for `rows` samples, and the hit count behind accuracy
 * (model.cpp:320-328): *hits_out (device u64) += #{r : predict(X_r) == y_r}. */
int ds_predict(const ds_model_desc* model, const float* params, const float* X, uint64_t rows,
               uint32_t* pred_out, void* stream);
int ds_count_hits(const ds_model_desc* model, const float* params, const float* X,
                  const uint32_t* y, uint64_t rows, unsigned long long* hits_out, void* stream);

/* ---------------------------------------------------------------------------------- */
/* Master — exchanger.hpp:40-72 (MasterState), center variable x~                     */
/* ---------------------------------------------------------------------------------- */
typedef struct ds_master ds_master;

#define DS_MODE_LOCKED 0   /* UpdateMode::Locked: exchanges linearized (ticketed)    */
#define DS_MODE_LOCKFREE 1 /* UpdateMode::LockFree: per-element plain ld/st, lost updates allowed */

/* MasterState(dim, alpha, mode, initial) (exchanger.cpp:65-74) on one device.
 * init_host: dim floats (must be finite: ContractError otherwise). */
int ds_master_create(ds_master** out, int device, uint64_t dim, float alpha, int mode,
                     const float* init_host);
/* Sharded center: this process owns slice `rank` of `world` (128-byte aligned
 * contiguous slices). Peers are attached with ds_master_export/ds_master_attach. */
int ds_master_create_sharded(ds_master** out, int device, uint64_t dim, float alpha, int mode,
                             int rank, int world, const float* init_host);
#define DS_IPC_RECORD_BYTES 256
/* Write this shard's IPC record (DS_IPC_RECORD_BYTES) for the peers. */
int ds_master_export(ds_master* m, void* record_out);
/* Attach all `world` records (index = rank; this rank's own is ignored). */
int ds_master_attach(ds_master* m, const void* records);
int ds_master_destroy(ds_master* m);

/* MasterState::exchange (exchanger.cpp:76-92): worker/out are device pointers on the
 * master's device (dim floats each; out may equal worker). Locked mode takes the next
 * ticket so concurrent exchanges linearize; LockFree streams straight through. */
int ds_master_exchange(ds_master* m, const float* worker, float* out, void* stream);
/* Deterministic mode: perform exchange number `ticket` (0-based, global order) only
 * after exchange ticket-1 completed on every shard; used to replay simulate_async's
 * serialization (simulator.cpp:105-143) across GPUs. */
int ds_master_exchange_ticketed(ds_master* m, const float* worker, float* out, uint64_t ticket,
                                void* stream);
/* MasterState::snapshot (exchanger.cpp:94-106) into host memory (synchronous). */
int ds_master_snapshot(ds_master* m, float* host_out);
/* Device pointer to this process's slice and its [begin,end) element range. */
int ds_master_local_slice(ds_master* m, float** dev_ptr, uint64_t* begin, uint64_t* end);
int ds_master_exchange_count(ds_master* m, uint64_t* count);
int ds_master_dim(ds_master* m, uint64_t* dim);
/* Reset the ticket sequence and exchange counter (all ranks, quiescent). */
int ds_master_reset_tickets(ds_master* m);

/* ---------------------------------------------------------------------------------- */
/* Engine — engine.hpp:17-105 (ShardSweeper, ExchangePolicy, SgdEngine, loop)        */
/* ---------------------------------------------------------------------------------- */
typedef struct ds_engine ds_engine;

typedef struct {
  double eta;
  double alpha;
  uint32_t tau;
  uint32_t batch_size;
  uint64_t i_max;
  double loss_cut;
  double weight_decay;
  int32_t adaptive;
} ds_hyper; /* Hyperparams (hyperparams.hpp:10-21) */

#define DS_ENGINE_AUTO 0    /* fused persistent kernel when the model allows, else layered */
#define DS_ENGINE_LAYERED 1 /* one kernel per layer pass; any depth                        */
#define DS_ENGINE_FUSED 2   /* persistent single-kernel step (<= 1 hidden layer)            */
/* Fast mode (NOT the reference's f64 order): the one-hidden-layer MLP step with its two
 * dense contractions (forward X.W1^T, weight gradient X^T.delta1) on the tcgen05 tensor
 * cores in bf16 with f32 accumulation, everything else f32; one thread-block cluster per
 * worker (16 hidden units per CTA), so several engines train concurrently on one GPU.
 * Every master mode exchanges in-kernel. Tolerance parity (tests/test_gpu_tc.py). */
#define DS_ENGINE_TC 3

/* SgdEngine(model, shard, hp, sweep_seed, initial) (engine.cpp:50-65): uploads the
 * shard (X row-major f32 [shard_n x n_features], y u32) to `device` once, keeps the
 * parameters, gradients and sweep order resident. hp is validated like
 * Hyperparams::validate (hyperparams.cpp:7-18). */
int ds_engine_create(ds_engine** out, int device, const ds_model_desc* model, const float* X_host,
                     const uint32_t* y_host, uint64_t shard_n, uint32_t shard_classes,
                     const ds_hyper* hp, uint64_t sweep_seed, const float* init_host, int kind);
/* SgdEngine over a DSHD shard file (shard.hpp:9-35), ingested straight into the engine's
 * resident X/y (ds_shard_load): shard_n and shard_classes come from the file header. */
int ds_engine_create_from_shard(ds_engine** out, int device, const ds_model_desc* model, const char* path,
                                const ds_hyper* hp, uint64_t sweep_seed, const float* init_host, int kind);
int ds_engine_destroy(ds_engine* e);
/* Attach a master: the policy's exchanges run on-device against it (async/LockFree or
 * Locked as the master was created; deterministic when tickets are given). */
int ds_engine_attach_master(ds_engine* e, ds_master* m);
/* Deterministic schedule: this worker's exchanges take the given global tickets in
 * order (count entries). Pass count 0 to return to ticket-less exchanges. */
int ds_engine_set_tickets(ds_engine* e, const uint64_t* tickets, uint64_t count);

/* Run `steps` iterations of run_training_loop's body (engine.cpp:96-111): step,
 * policy, exchange-if-fired (against the attached master; with no master the
 * exchange is skipped, as with a null ExchangeFn). Asynchronous on the engine's
 * stream. If stop_at_exchange is nonzero the run ends after the first iteration whose
 * policy fires WITHOUT performing that exchange (for host ExchangeFn callbacks);
 * *ran_out (host, optional, synchronous when given) reports the iterations done. */
int ds_engine_run(ds_engine* e, uint64_t steps, int stop_at_exchange, uint64_t* ran_out);
/* Run `steps` iterations of several tensor-core engines (DS_ENGINE_TC; same device, model
 * and batch size; <= 8) in ONE cooperative launch, one thread-block cluster per engine, all
 * resident at once: the workers train concurrently and exchange with their masters
 * in-kernel, so deterministic tickets across them are honoured on a single GPU (the
 * reference's n-worker run_training_loop / simulate_async schedule, simulator.cpp:70-154).
 * Equivalent to ds_engine_run(e, steps, 0, NULL) on each engine; enqueued on engine 0's
 * stream, ordered after and before every engine's own stream work. */
int ds_engine_run_group(ds_engine** engines, uint32_t n, uint64_t steps);
/* Pre-size the engine's batch-plan and TrainLog buffers for the next `steps`
 * iterations so a following ds_engine_run(steps) allocates nothing (no implicit
 * device synchronisation inside a timed or latency-sensitive region). */
int ds_engine_reserve(ds_engine* e, uint64_t steps);
/* Momentum option (ds_sgd_momentum_update; layered engine only — the fused step keeps
 * mu = 0): every following iteration uses the momentum update with this mu. */
int ds_engine_set_momentum(ds_engine* e, float mu);
/* Synchronous data-parallel mode (layered engine, no EASGD master): every iteration
 * writes its gradient into the group's slot and applies ds_sync_reduce_update — the
 * simulate_sync round (simulator.cpp:156-223) across the group's GPUs. NULL detaches. */
int ds_engine_attach_sync(ds_engine* e, ds_sync* s);
/* Host-fed iteration (a data pipeline that owns the rows, like the reference worker's
 * ShardSweeper + gather_batch, engine.cpp:25-33 / model.cpp:12-21): copies `rows`
 * gathered rows (X_host row-major, y_host) from host memory — pinned for full speed —
 * into the engine's staging area, runs one iteration of run_training_loop on exactly
 * that batch (policy and exchange included), and, when loss_host is given, reads the
 * batch loss back (synchronous). The engine's own sweep position is not advanced. */
int ds_engine_step_host(ds_engine* e, const float* X_host, const uint32_t* y_host, uint32_t rows,
                        double* loss_host);
/* Pipelined form of ds_engine_step_host: the same iteration, enqueued without waiting.
 * Staging is double-buffered: X_host/y_host may be refilled two calls later, and
 * *loss_host (pinned for an asynchronous copy) is valid after ds_engine_sync or two
 * calls later. The host blocks only when it runs two iterations ahead of the device. */
int ds_engine_step_host_async(ds_engine* e, const float* X_host, const uint32_t* y_host, uint32_t rows,
                              double* loss_host);
/* Depth of the stream-mode ring: the host may run this many pushes ahead of the device. */
#define DS_STREAM_RING 8

/* Stream mode: ONE persistent launch trains `steps` iterations on batches the host pushes
 * while it runs (a DS_STREAM_RING-slot device ring; the copy engine lands each batch and then its
 * sequence word, the kernel waits for the word, frees the slot after its grid barrier).
 * Every batch crosses PCIe as an H2D copy; each step's loss is written by the kernel to
 * *loss_host[step] (pinned, mapped: zero-copy D2H), valid after ds_engine_stream_end.
 * push blocks only while the ring is full. X_host/y_host of push s may be rewritten once
 * push s+DS_STREAM_RING has returned (tensor-core engines copy them before push returns).
 * Fused one-hidden-layer engine; a Fixed or Adaptive policy (Adaptive needs the
 * in-kernel exchange: no master, a LockFree/sharded one, or a TC engine). A host that stops pushing for
 * 20 s makes the kernel finish with DS_FLAG_STREAM_TIMEOUT rather than hang. */
int ds_engine_stream_begin(ds_engine* e, uint64_t steps, double* loss_host);
int ds_engine_stream_push(ds_engine* e, const float* X_host, const uint32_t* y_host, uint32_t rows);
/* As ds_engine_stream_push, but gathers the batch itself: rows idx[0..rows) of the host
 * shard (X_host f32 [n x F], y_host u32 [n], any host memory) are copied into an
 * engine-owned pinned staging slot (gather_batch, model.cpp:12-21) and pushed. */
int ds_engine_stream_push_rows(ds_engine* e, const float* X_host, const uint32_t* y_host, const uint32_t* idx,
                               uint32_t rows);
/* As ds_engine_stream_push_rows for nsteps consecutive steps in one call: step s takes
 * rows[s] row indices from idx[s * batch_size ...] (the ShardSweeper layout). Blocks while
 * the ring is full. Tensor-core engines gather the rows as bf16 into a pinned staging ring
 * (labels in each slot's extra row) with helper threads and move groups of 4 steps per H2D
 * DMA (two CUDA calls per group). */
int ds_engine_stream_push_rows_n(ds_engine* e, const float* X_host, const uint32_t* y_host, const uint32_t* idx,
                                 const uint32_t* rows, uint64_t nsteps);
/* Tensor-core engines: keep a bf16 copy of the host shard X_host [n_rows x n_features]
 * (the same cast as the per-step gather), so later pushes that pass this X_host gather rows
 * by row copies — half the host memory traffic and no cast per step. X_host NULL drops the
 * copy. Not while a stream is open (DS_E_STATE); the caller keeps X_host unchanged while it
 * is cached. */
int ds_engine_stream_cache_host_shard(ds_engine* e, const float* X_host, uint64_t n_rows);
int ds_engine_stream_end(ds_engine* e);
/* Host-side gather + bf16 cast the tensor-core stream ring uses (no GPU involved): rows x F
 * floats, row r from X + idx[r] * F (idx NULL: X + r * F), into dst rows of `pitch` bf16
 * (padding untouched); round to nearest even, NaN -> 0x7FFF, denormals kept — the device's
 * __float2bfloat16_rn bits. DS_E_CONTRACT on null pointers or pitch < F. */
int ds_host_rows_to_bf16(const float* X, uint32_t F, const uint32_t* idx, uint32_t rows, uint16_t* dst,
                         uint64_t pitch);
/* Stream mode for several tensor-core engines trained in ONE launch (ds_engine_run_group):
 * each engine gets its own ring, pushes and ds_engine_stream_end as above; loss_host[i]
 * (pinned, or a NULL array) receives engine i's per-step losses. */
int ds_engine_stream_begin_group(ds_engine** engines, uint32_t n, uint64_t steps, double** loss_host);
/* Block until the engine's queued work finished; returns DS_E_NUMERIC/DS_E_CONTRACT
 * if any step hit the reference's error conditions (message names the iteration). */
int ds_engine_sync(ds_engine* e);
/* Engine stream (cudaStream_t) for event timing / interop. */
int ds_engine_stream(ds_engine* e, void** stream);
/* TrainLog rows [first, first+count) (metrics.hpp:11-24), synchronous copy to host.
 * Any output pointer may be NULL. */
int ds_engine_log(ds_engine* e, uint64_t first, uint64_t count, double* batch_loss,
                  double* cumulated, uint8_t* exchanged, uint32_t* period_len);
int ds_engine_iterations(ds_engine* e, uint64_t* iters);
/* SgdEngine::params / set_params (engine.hpp:76-78), host copies (synchronous). */
int ds_engine_get_params(ds_engine* e, float* host_out);
int ds_engine_set_params(ds_engine* e, const float* host_in);
/* Device pointer of the live parameter vector (valid until the next run call). */
int ds_engine_params_device(ds_engine* e, float** dev_ptr);
/* Resolved policy state (ExchangePolicy, engine.hpp:40-59). */
int ds_engine_policy(ds_engine* e, double* cumulated, uint32_t* since_exchange, double* loss_cut);
/* Loop-launch count since creation (kernels this engine launched). */
int ds_engine_launches(ds_engine* e, uint64_t* launches);

#ifdef __cplusplus
}
#endif

#endif /* DS_CUDA_H */
