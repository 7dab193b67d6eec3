#!/bin/bash
# final bench lines at N = 2 and 4 (all legs), one box
cd "$(dirname "$0")/.." || exit 1
O=gpurun_out/${1:-finscale}; mkdir -p $O
CUDA_VISIBLE_DEVICES=0,1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29581 bench.py --gpus 2 > $O/bench_n2.json 2> $O/bench_n2.err
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29582 bench.py --gpus 4 > $O/bench_n4.json 2> $O/bench_n4.err
echo done
