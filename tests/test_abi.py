"""CPU-side checks of the drop-in boundary: the C-ABI library loads and exports every
symbol include/ds_cuda.h declares (no device work is launched here)."""
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    src = open(os.path.join(ROOT, "include", header)).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(ds_\w+)\s*\(", src, re.M)))


def exported(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True, check=True).stdout
    return {l.split()[-1] for l in out.splitlines() if l.strip()}


def test_c_abi_exports_every_declared_symbol():
    from paper_1602_08191_b200 import _lib
    names = declared("ds_cuda.h")
    assert len(names) >= 30
    syms = exported(_lib.LIB_PATH)
    missing = [n for n in names if n not in syms]
    assert not missing, missing
    assert sorted(names) == sorted(_lib.EXPORTED)
    for n in names:
        getattr(_lib.lib, n)  # resolvable through ctypes


def test_library_targets_sm100a_only():
    from paper_1602_08191_b200 import _lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_version_and_no_device_is_an_error_not_a_fallback():
    from paper_1602_08191_b200 import _lib
    assert "sm_100a" in _lib.version()
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if not has_gpu:
        import ctypes as C
        import numpy as np
        m = C.c_void_p()
        init = np.zeros(4, np.float32)
        rc = _lib.lib.ds_master_create(C.byref(m), 0, 4, C.c_float(0.1), 0, init.ctypes.data)
        assert rc == _lib.DS_E_CUDA
