// model.cuh — device model description and the layer-wise f64 forward/backward path.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "ds_cuda.h"

namespace dsb {

// Model::layers (model.cpp:103-121): per layer W[out x in] row-major, then b[out].
struct LayerInfo {
  uint64_t w_off, b_off;
  uint32_t in_dim, out_dim;
};

struct ModelInfo {
  int32_t kind = 0;  // 0 softmax, 1 mlp, 2 cifar10_quick, 3 alexnet (2, 3 NOT IN REFERENCE)
  uint32_t n_features = 0, n_classes = 0;
  std::vector<uint32_t> hidden;
  std::vector<LayerInfo> layers;
  uint64_t P = 0;
  uint32_t max_out = 0;
  uint64_t sum_out = 0;
  uint32_t alex_side = 0;  // kind 3: input side S
};

// Model::validate (model.cpp:44-57) + layer layout; DS_E_CONTRACT on invalid models.
int model_from_desc(const ds_model_desc* d, ModelInfo& out);

// Doubles of workspace the layered path needs for R rows.
uint64_t layered_workspace_doubles(const ModelInfo& m, uint32_t R);

// loss_and_grad / loss_only (model.cpp:242-275), reference summation order.
//  X: row-major f32 rows; if idx != nullptr row r is X[idx[r]] (a device-side gather).
//  y: labels indexed the same way. grad == nullptr selects loss_only's loss formula.
//  flags: device word the DS_FLAG_* conditions are OR-ed into (may be null).
//  gate: optional device word; if nonzero when a kernel starts it returns at once
//  (a failed earlier step freezes the engine, as the reference's throw would).
int launch_loss_and_grad(const ModelInfo& m, const float* params, const float* X,
                         const uint32_t* idx, const uint32_t* y, uint32_t R, float* grad,
                         double* loss_out, double* ws, uint32_t* flags, const uint32_t* gate,
                         cudaStream_t s);

// cifar10_quick (kind DS_MODEL_CIFAR10_QUICK, convnet.cu; NOT IN REFERENCE).
uint64_t cnn_workspace_bytes(const ModelInfo& m, uint32_t R);
int launch_cnn_loss_and_grad(const ModelInfo& m, const float* P, const float* X, const uint32_t* idx, const uint32_t* y,
                             uint32_t R, float* grad, double* loss_out, void* ws, uint32_t* flags,
                             const uint32_t* gate, cudaStream_t s);
int launch_cnn_count_hits(const ModelInfo& m, const float* P, const float* X, const uint32_t* y, uint32_t R, void* ws,
                          unsigned long long* hits, uint32_t* pred, cudaStream_t s);

// AlexNet-shaped (kind DS_MODEL_ALEXNET, alexnet.cu; NOT IN REFERENCE).
uint64_t alex_workspace_bytes(const ModelInfo& m, uint32_t R);
uint32_t alex_last_launches();  // kernels issued by this thread's last launch_alex_loss_and_grad
int launch_alex_loss_and_grad(const ModelInfo& m, const float* P, const float* X, const uint32_t* idx,
                              const uint32_t* y, uint32_t R, float* grad, double* loss_out, void* ws,
                              uint32_t* flags, const uint32_t* gate, cudaStream_t s);
int launch_alex_count_hits(const ModelInfo& m, const float* P, const float* X, const uint32_t* y, uint32_t R,
                           void* ws, unsigned long long* hits, uint32_t* pred, cudaStream_t s);

// Hits of predict() (model.cpp:303-318) against labels over rows [0,R).
int launch_count_hits(const ModelInfo& m, const float* params, const float* X, const uint32_t* y,
                      uint32_t R, double* ws, unsigned long long* hits, uint32_t* pred,
                      cudaStream_t s);

}  // namespace dsb
