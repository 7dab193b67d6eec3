"""paper_1602_08191_b200 — B200-native DeepSpark EASGD hot path (sm_100a).

The product is the C-ABI library ``lib/libds_cuda.so`` (include/ds_cuda.h) and the
reference-compatible C++ API ``lib/libdeepspark_b200.so`` (include/deepspark/*.hpp).
This package only binds them for Python callers (tests, bench). Importing a submodule
that needs the CUDA library fails loudly when it is missing; there is no CPU fallback.
"""

__all__ = ["_lib"]
