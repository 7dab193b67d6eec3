import os, sys, numpy as np
sys.path.insert(0, '/root/repo'); sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests")); import test_gpu_convnet as t
import torch
from oracle.oracle import Oracle
from paper_1602_08191_b200 import _lib as L
orc = Oracle("dso")
X, y = t.data(orc, 8)
w = orc.init_params(t.M, 2)
res = {}
for mode in ("1", "0"):
    os.environ["DS_CNN_FFMA"] = mode
    res[mode] = t.gpu_lag(torch, L, w, X, y)[1]
a, b = res["1"], res["0"]
segs = [("c1W",0,2400),("c1b",2400,2432),("c2W",2432,28032),("c2b",28032,28064),("c3W",28064,79264),("c3b",79264,79328),("ip1",79328,144928),("ip2",144928,145578)]
for n,lo,hi in segs:
    d = np.abs(a[lo:hi]-b[lo:hi]).max(); m = np.abs(a[lo:hi]).max()
    print(n, f"maxdiff {d:.3e} max {m:.3e} rel {d/m:.3e}", "ffma[:4]", a[lo:lo+4], "tc[:4]", b[lo:lo+4])
