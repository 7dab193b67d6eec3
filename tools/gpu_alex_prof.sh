#!/bin/bash
# AlexNet step launch list with per-launch grid, tensor-pipe activity and DRAM bytes (second step)
cd "$(dirname "$0")/.." || exit 1
O=gpurun_out/${1:-alex}; mkdir -p $O
timeout 300 python tools/prof_alex.py 2 > $O/plain.log 2>&1
DS_ENGINE_NO_GRAPH=1 timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file $O/launches.csv python tools/prof_alex.py 2 > $O/ncu.log 2>&1
echo done
