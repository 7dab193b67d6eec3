#!/bin/bash
# ncu --set full of the cifar10_quick weight-gradient convolution (conv2: <32, 32, 16, 4>)
cd "$(dirname "$0")/.." || exit 1
O=gpurun_out/${1:-cnnncu}; mkdir -p $O
DS_ENGINE_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv5_wgrad_tc_kernel \
  --launch-skip 3 --launch-count 3 -o $O/wgrad python tools/prof_cnn.py --steps 3 > $O/ncu.log 2>&1
echo done
