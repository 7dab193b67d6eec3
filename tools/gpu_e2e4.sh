#!/bin/bash
# e2e (host-fed stream mode) at 1 and 4 GPUs + the TC stream tests
cd "$(dirname "$0")/.." || exit 1
O=gpurun_out/${1:-e2e4}; mkdir -p $O
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_tc.py -q -x -p no:cacheprovider > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --cifar-steps 0 --alexnet-steps 0 > $O/b1.json 2> $O/b1.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29571 bench.py --gpus 4 --cifar-steps 0 --alexnet-steps 0 > $O/b4.json 2> $O/b4.err
echo done
