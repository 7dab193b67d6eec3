#!/bin/bash
# One gpurun call: GPU tests, smoke, bench, launch list and ncu captures (outputs in gpurun_out/).
cd "$(dirname "$0")/.." || exit 1
mkdir -p gpurun_out
TAG=${1:-r}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.used --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 1200 python -m pytest tests -q -m gpu -p no:cacheprovider -rs > gpurun_out/${TAG}_tests.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_smoke.log
timeout 600 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; echo "rc=$?" >> gpurun_out/${TAG}_bench.log
if [ "${NO_NCU:-0}" != "1" ]; then
  timeout 300 python bench.py --steps 200 --warmup 5 --no-extras --cifar-steps 0 --alexnet-steps 0 > gpurun_out/${TAG}_bsmall.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
      python bench.py --steps 200 --warmup 5 --no-extras --cifar-steps 0 --alexnet-steps 0 > gpurun_out/${TAG}_ncu1.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"mlp_kernel|fused_kernel" -s 1 -c 1 \
      -o gpurun_out/${TAG}_prof_fused python bench.py --steps 200 --warmup 5 --no-extras --cifar-steps 0 --alexnet-steps 0 > gpurun_out/${TAG}_ncu2.log 2>&1
  timeout 120 python tools/prof_exchange.py > gpurun_out/${TAG}_pexch.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:elastic -s 2 -c 1 \
      -o gpurun_out/${TAG}_prof_elastic python tools/prof_exchange.py > gpurun_out/${TAG}_ncu3.log 2>&1
fi

if [ "${NO_NCU:-0}" != "1" ]; then
  timeout 300 python tools/prof_cnn.py --steps 20 > gpurun_out/${TAG}_cnn.log 2>&1 && \
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_cnn_launches.csv \
      python tools/prof_cnn.py --steps 20 > gpurun_out/${TAG}_ncu4.log 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:conv5_tc_kernel -s 1 -c 1 \
      -o gpurun_out/${TAG}_prof_conv_tc python tools/prof_cnn.py --steps 5 > gpurun_out/${TAG}_ncu5.log 2>&1
fi
echo done
