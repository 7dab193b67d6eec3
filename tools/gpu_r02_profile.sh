#!/bin/bash
# One gpurun call: bench line, launch list, one ncu --set full capture of mlp_tc_kernel (as
# the bench launches it: two workers in one group launch).
cd "$(dirname "$0")/.." || exit 1
O=gpurun_out/r02
mkdir -p $O
timeout 900 python bench.py > $O/bench_n1.json 2> $O/bench_n1.err; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $O/launches.csv \
  python bench.py --steps 300 --warmup 3 --no-extras --min-window-ms 0 --cifar-steps 0 --alexnet-steps 0 \
  > $O/launches.log 2>&1; echo "launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:mlp_tc_kernel -s 2 -c 1 -o $O/mlp_tc \
  python bench.py --steps 300 --warmup 3 --no-extras --min-window-ms 0 --cifar-steps 0 --alexnet-steps 0 \
  > $O/ncu_full.log 2>&1; echo "ncu full rc=$?"
# compute-sanitizer is closed on the GPU pool (it left GPUs needing a reset); the device
# asserts build (DS_DEVICE_ASSERTS=1 make) plus the sanitize_targets runs replace it.
