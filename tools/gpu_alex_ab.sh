#!/bin/bash
# AlexNet change check: GPU tests of the convnets, bench alexnet leg, launch list with metrics
cd "$(dirname "$0")/.." || exit 1
O=gpurun_out/${1:-alexab}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_alexnet.py -q -x -p no:cacheprovider > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
timeout 600 python bench.py --no-extras --steps 100 --cifar-steps 0 --alexnet-steps 40 > $O/bench.json 2> $O/bench.err
[ "${NO_PROF:-0}" = 1 ] || bash tools/gpu_alex_prof.sh ${1:-alexab}
