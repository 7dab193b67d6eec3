"""Standalone elastic-exchange kernel run for profiling (config 5 shape): w and the center
of P f32 parameters, updated in place a few times through ds_elastic_update."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1602_08191_b200 import _lib as L  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 256 * 1024 * 1024
w = torch.rand(P, device="cuda")
m = torch.rand(P, device="cuda")
s = torch.cuda.current_stream()
for _ in range(5):
    L.check(L.lib.ds_elastic_update(C.c_void_p(w.data_ptr()), C.c_void_p(m.data_ptr()), P, C.c_float(0.1),
                                    C.c_void_p(s.cuda_stream)))
torch.cuda.synchronize()
print("ok", P)
