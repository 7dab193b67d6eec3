"""Per-layer GPU-vs-oracle gradient statistics for the AlexNet-shaped model (debug tool)."""
import sys
import numpy as np
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from oracle.oracle import ModelSpec, Oracle
import test_gpu_alexnet as t
import torch
from paper_1602_08191_b200 import _lib as L
orc = Oracle("dso")
import os
cases = [(224, 1000, 2, 1.0)] if os.environ.get('DBG_FULL') else [(55, 5, 1, 5.0), (55, 5, 13, 5.0), (55, 5, 13, 1.0), (67, 10, 8, 1.0)]
for side, c, batch, scale in cases:
    m = ModelSpec.alexnet(side, c)
    w = orc.init_params(m, 4 if side == 224 else 3)
    X, y = orc.gen_synthetic(batch, 3 * side * side, c, 1.0, 1.0, 5 if side == 224 else 21)
    X = np.ascontiguousarray(X * scale, dtype=np.float32)
    lr, gr = orc.loss_and_grad(m, w, X, y)
    lg, gg, flags = t.gpu_lag(torch, L, t.desc(L, side, c), w, X, y)
    print(f"side {side} batch {batch} xscale {scale}: loss gpu {lg:.8f} ref {lr:.8f} flags {flags}")
    for li, (a, b) in enumerate(t.layer_bounds(orc, side, c)):
        ref, got = gr[a:b].astype(np.float64), gg[a:b].astype(np.float64)
        cos = float(ref @ got / (np.linalg.norm(ref) * np.linalg.norm(got) + 1e-300))
        err = np.abs(got - ref).max() / (np.abs(ref).max() + 1e-300)
        rn = np.linalg.norm(got - ref) / (np.linalg.norm(ref) + 1e-300)
        print(f"  layer {li}: cos {cos:.6f} maxerr/max {err:.3e} relnorm {rn:.3e} |ref| {np.abs(ref).max():.3e}")
