#!/bin/bash
# Engine parity tests, bench (no extras), per-phase stamps and one ncu capture of the fused step kernel.
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
TAG=${1:-p}
timeout 600 python -m pytest tests/test_gpu_engine.py tests/test_cpp_api_parity.py tests/test_reference_suites.py -q -m gpu -p no:cacheprovider > gpurun_out/${TAG}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_tests.log
timeout 300 python bench.py --no-extras --cifar-steps 0 --alexnet-steps 0 > gpurun_out/${TAG}_bench.log 2>&1
DS_FUSED_PROFILE=gpurun_out/${TAG}_phases.txt timeout 300 python bench.py --no-extras --cifar-steps 0 --alexnet-steps 0 --steps 1000 --warmup 5 > gpurun_out/${TAG}_bphase.log 2>&1
if [ "${NO_NCU:-0}" != "1" ]; then
timeout 300 python bench.py --no-extras --cifar-steps 0 --alexnet-steps 0 --steps 400 --warmup 5 > gpurun_out/${TAG}_bsmall.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"mlp_kernel|fused_kernel" -s 1 -c 1 \
    -o gpurun_out/${TAG}_prof_fused python bench.py --no-extras --cifar-steps 0 --alexnet-steps 0 --steps 400 --warmup 5 > gpurun_out/${TAG}_ncu.log 2>&1
fi
echo done
