#!/bin/bash
# cifar10_quick change check: convnet GPU tests, bench cifar legs, launch list
cd "$(dirname "$0")/.." || exit 1
O=gpurun_out/${1:-cifarab}; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_convnet.py tests/test_gpu_sync.py -q -x -p no:cacheprovider > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
timeout 600 python bench.py --no-extras --steps 100 --alexnet-steps 0 > $O/bench.json 2> $O/bench.err
timeout 300 python tools/prof_cnn.py --steps 20 > $O/cnn.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv python tools/prof_cnn.py --steps 20 > $O/ncu.log 2>&1
echo done
