"""Measure the AlexNet production tf32 path's per-layer gradient deviation from (a) the f64
oracle and (b) the GPU's own f32-accurate 3xTF32 products, and the prediction agreement
against the oracle as a function of the top-2 logit margin. Sets the bars stated in
tests/test_gpu_alexnet.py. Tool only: python tools/alex_tol.py"""
import ctypes as C
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))


def main():
    import torch
    from oracle.oracle import ModelSpec, Oracle
    from paper_1602_08191_b200 import _lib as L
    from test_gpu_alexnet import desc, gpu_lag, layer_bounds

    orc = Oracle("dso")
    out = []

    def rel(a, b):
        a, b = a.astype(np.float64), b.astype(np.float64)
        return float(np.linalg.norm(a - b) / np.linalg.norm(b))

    for side, c, batch, seed, scale, with_f64 in [(55, 5, 13, 21, 5.0, True), (224, 1000, 2, 5, 1.0, True),
                                                   (224, 1000, 32, 6, 1.0, False), (67, 10, 64, 7, 5.0, False)]:
        m = ModelSpec.alexnet(side, c)
        w = orc.init_params(m, 4)
        X, y = orc.gen_synthetic(batch, 3 * side * side, c, 1.0, 1.0, seed)
        X = np.ascontiguousarray(X * scale, dtype=np.float32)
        d = desc(L, side, c)
        os.environ.pop("DS_GEMM_3XTF32", None)
        lt, gt, _ = gpu_lag(torch, L, d, w, X, y)
        os.environ["DS_GEMM_3XTF32"] = "1"
        lx, gx, _ = gpu_lag(torch, L, d, w, X, y)
        os.environ.pop("DS_GEMM_3XTF32", None)
        rec = {"side": side, "batch": batch, "loss_tf32_vs_3x": abs(lt - lx) / abs(lx)}
        rec["layers_tf32_vs_3x"] = [rel(gt[a:b], gx[a:b]) for a, b in layer_bounds(orc, side, c)]
        if with_f64:
            lr, gr = orc.loss_and_grad(m, w, X, y)
            rec["layers_tf32_vs_f64"] = [rel(gt[a:b], gr[a:b]) for a, b in layer_bounds(orc, side, c)]
            rec["layers_3x_vs_f64"] = [rel(gx[a:b], gr[a:b]) for a, b in layer_bounds(orc, side, c)]
        out.append(rec)
        print(json.dumps(rec), flush=True)
    # predictions vs margins
    side, c = 55, 7
    m = ModelSpec.alexnet(side, c)
    w = orc.init_params(m, 6)
    X, y = orc.gen_synthetic(200, 3 * side * side, c, 1.0, 1.0, 9)
    X = np.ascontiguousarray(X * 5.0, dtype=np.float32)
    ref = orc.predict(m, w, X)
    d = desc(L, side, c)
    pd = torch.from_numpy(w).cuda()
    Xd = torch.from_numpy(X).cuda()
    pred = torch.zeros(len(y), dtype=torch.int32, device="cuda")
    L.check(L.lib.ds_predict(C.byref(d), C.c_void_p(pd.data_ptr()), C.c_void_p(Xd.data_ptr()), len(y),
                             C.c_void_p(pred.data_ptr()), None))
    torch.cuda.synchronize()
    got = pred.cpu().numpy()
    print(json.dumps({"predict_agree": float((got == ref).mean()), "n": len(y)}), flush=True)


if __name__ == "__main__":
    main()
