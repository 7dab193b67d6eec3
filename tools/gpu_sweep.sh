#!/bin/bash
# Config 5 exchange sweep at 1 / 2 / 4 GPUs (tools/exchange_sweep.py)
cd "$(dirname "$0")/.." || exit 1
O=gpurun_out/${1:-sweep}; mkdir -p $O
CUDA_VISIBLE_DEVICES=0 timeout 600 python tools/exchange_sweep.py > $O/sweep_n1.jsonl 2> $O/sweep_n1.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29561 tools/exchange_sweep.py > $O/sweep_n2.jsonl 2> $O/sweep_n2.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29562 tools/exchange_sweep.py > $O/sweep_n4.jsonl 2> $O/sweep_n4.err
echo done
