"""One AlexNet-shaped loss_and_grad at a small side (debug tool); DS_* env as given."""
import sys
import numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from oracle.oracle import ModelSpec, Oracle
import test_gpu_alexnet as t
import torch
from paper_1602_08191_b200 import _lib as L
orc = Oracle("dso")
side, c = int(sys.argv[1]) if len(sys.argv) > 1 else 55, 5
m = ModelSpec.alexnet(side, c)
w = orc.init_params(m, 3)
X, y = orc.gen_synthetic(2, 3 * side * side, c, 1.0, 1.0, 21)
try:
    print(t.gpu_lag(torch, L, t.desc(L, side, c), w, X, y)[0])
except Exception as e:
    print("ERR", e)
