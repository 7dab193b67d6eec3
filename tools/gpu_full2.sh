#!/bin/bash
# Two-GPU verification: the whole GPU suite (multi-GPU tests included), smoke, bench at N=1 and N=2
cd "$(dirname "$0")/.." || exit 1
O=gpurun_out/${1:-full2}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/smi.txt 2>&1
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider -rs > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py > $O/bench_n1.json 2> $O/bench_n1.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 > $O/bench_n2.json 2> $O/bench_n2.err
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/ref_n1.json 2> $O/ref_n1.err
echo done
