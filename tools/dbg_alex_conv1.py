"""conv1 gradient error pattern (debug tool)."""
import sys
import numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from oracle.oracle import ModelSpec, Oracle
import test_gpu_alexnet as t
import torch
from paper_1602_08191_b200 import _lib as L
orc = Oracle("dso")
side, c = 55, 5
m = ModelSpec.alexnet(side, c)
w = orc.init_params(m, 3)
X, y = orc.gen_synthetic(1, 3 * side * side, c, 1.0, 1.0, 21)
X = np.ascontiguousarray(X * 5.0, dtype=np.float32)
lr, gr = orc.loss_and_grad(m, w, X, y)
lg, gg, _ = t.gpu_lag(torch, L, t.desc(L, side, c), w, X, y)
W = (gg[:34848] - gr[:34848]).reshape(96, 3, 11, 11)
R = gr[:34848].reshape(96, 3, 11, 11)
print("bias relerr", np.linalg.norm(gg[34848:34944] - gr[34848:34944]) / np.linalg.norm(gr[34848:34944]))
e = np.abs(W).max(axis=(0, 1))
print("max |err| by (ky, kx) / max|ref|:")
print(np.array2string(e / np.abs(R).max(), precision=3, max_line_width=200))
print("max |err| by channel:", np.abs(W).max(axis=(0, 2, 3)) / np.abs(R).max())
