/* ds_oracle_cnn.h — TEST INFRASTRUCTURE ONLY (see ds_oracle.c). f64 CPU restatement of
 * the Caffe cifar10_quick network for model kind 2 (NOT IN THE
 * REFERENCE — no reference to pin against; this restatement is checked by central
 * differences in tests/test_oracle.py and against an independent PyTorch float64 autograd
 * implementation in tests/test_oracle_cnn_torch.py: loss to 1e-12, grads bit-exact).
 *
 * Conventions follow the reference's models (model.cpp:103-159): flat parameters, per
 * layer W[out x fan_in] row-major then b[out]; init U(+-1/sqrt(fan_in)) for weights and
 * biases; mean softmax cross-entropy with a max-shifted log-sum-exp; the gradient is the
 * f64 batch sum times 1/b, rounded to f32 once.
 *
 * Network (Caffe examples/cifar10/cifar10_quick_train_test.prototxt), input CHW 3x32x32:
 *   conv1 5x5 3->32 pad 2 -> pool1 MAX 3x3/2 -> relu1
 *   conv2 5x5 32->32 pad 2 -> relu2 -> pool2 AVE 3x3/2
 *   conv3 5x5 32->64 pad 2 -> relu3 -> pool3 AVE 3x3/2
 *   ip1 1024->64 -> ip2 64->C -> softmax loss
 * Pooling uses Caffe's ceil-mode output size and, for AVE, the window clipped to the
 * image as the divisor (pad 0). */
#pragma once
#include <stdint.h>

#define DSO_CNN_KIND 2
#define DSO_CNN_FEATURES 3072u

typedef struct {
  uint64_t w_off, b_off;
  uint32_t in_dim, out_dim; /* fan_in (Cin*25 for convs), outputs */
} dso_cnn_layer;

/* The five parameterised layers of cifar10_quick for C classes. */
void dso_cnn_layers(uint32_t n_classes, dso_cnn_layer out[5]);

/* Per-sample f64 pass; g (P doubles) accumulates the gradient when non-NULL. Returns the
 * sample loss; *pred receives the argmax class (first maximum). ws: dso_cnn_ws_doubles(). */
uint64_t dso_cnn_ws_doubles(uint32_t n_classes);
double dso_cnn_sample(const float* P, uint32_t n_classes, const float* x, uint32_t label, double* g, double* ws,
                      uint32_t* pred);
