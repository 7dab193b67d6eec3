#!/bin/bash
# Four-GPU verification: the GPU suite (multi-GPU tests at world 2-4), bench at N=4
cd "$(dirname "$0")/.." || exit 1
O=gpurun_out/${1:-full4}; mkdir -p $O
nvidia-smi topo -m > $O/topo.txt 2>&1
[ "${NO_TESTS:-0}" = 1 ] || timeout 1800 python -m pytest tests/test_mgpu.py -q -p no:cacheprovider -rs > $O/mgpu_tests.log 2>&1; echo "rc=$?" >> $O/mgpu_tests.log
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29544 bench.py --gpus 4 > $O/bench_n4.json 2> $O/bench_n4.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29545 bench.py --impl reference --gpus 4 --steps 3 --warmup 3 > $O/ref_n4.json 2> $O/ref_n4.err
echo done
