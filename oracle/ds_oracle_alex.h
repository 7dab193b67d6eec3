/* ds_oracle_alex.h — TEST INFRASTRUCTURE ONLY (see ds_oracle.c). f64 CPU restatement of
 * an AlexNet-shaped convnet for model kind 3 (BASELINE config 4; NOT IN
 * THE REFERENCE — no reference to pin against; checked by central differences in
 * tests/test_oracle.py and against an independent PyTorch float64 autograd implementation
 * of the same layers in tests/test_oracle_cnn_torch.py: loss to 1e-12, grads to 1 ulp).
 *
 * Conventions follow the reference's models (model.cpp:103-159): flat parameters, per
 * layer W[out x fan_in] row-major then b[out] (conv W in Caffe order [Cout][Cin/g][kh][kw]);
 * init U(+-1/sqrt(fan_in)) for weights and biases; mean softmax cross-entropy with a
 * max-shifted log-sum-exp; the gradient is the f64 batch sum times 1/b, rounded to f32.
 *
 * Network (Caffe models/bvlc_alexnet/train_val.prototxt), input CHW 3 x S x S with
 * S = sqrt(n_features / 3) (S = 224 for config 4; any S >= 55 works):
 *   conv1 11x11/4 3->96          -> relu -> LRN(5, 1e-4, 0.75, k 1) -> MAX 3x3/2
 *   conv2 5x5 pad 2 96->256 g2   -> relu -> LRN                     -> MAX 3x3/2
 *   conv3 3x3 pad 1 256->384     -> relu
 *   conv4 3x3 pad 1 384->384 g2  -> relu
 *   conv5 3x3 pad 1 384->256 g2  -> relu -> MAX 3x3/2
 *   fc6 (256*P5*P5)->4096 -> relu ; fc7 4096->4096 -> relu ; fc8 4096->C -> softmax loss
 * Dropout is omitted (no reference semantics; keeps every run deterministic). Pooling
 * uses Caffe's ceil-mode output size, pad 0, first maximum in scan order; LRN is Caffe's
 * ACROSS_CHANNELS: scale = k + alpha/n * sum of squares over the clipped 5-channel
 * window, y = x * scale^-beta. fc6 reads the pooled map flattened in CHW order. */
#pragma once
#include <stdint.h>

#define DSO_ALEX_KIND 3
#define DSO_ALEX_LAYERS 8

typedef struct {
  uint64_t w_off, b_off;
  uint32_t in_dim, out_dim; /* fan_in ((Cin/g)*k*k for convs), outputs */
} dso_alex_layer;

/* Side S of the square input for n_features (0 if n_features is not 3*S*S with S >= 55). */
uint32_t dso_alex_side(uint32_t n_features);
/* The eight parameterised layers for input side S and C classes. */
void dso_alex_layers(uint32_t side, uint32_t n_classes, dso_alex_layer out[DSO_ALEX_LAYERS]);
uint64_t dso_alex_ws_doubles(uint32_t side, uint32_t n_classes);
/* Per-sample f64 pass; g (P doubles) accumulates the gradient when non-NULL. Returns the
 * sample loss; *pred receives the argmax class (first maximum). */
double dso_alex_sample(const float* P, uint32_t side, uint32_t n_classes, const float* x, uint32_t label, double* g,
                       double* ws, uint32_t* pred);
