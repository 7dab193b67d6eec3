#!/bin/bash
# ncu --set full of every tf32 GEMM launch of the second AlexNet step (no graph, one stream)
cd "$(dirname "$0")/.." || exit 1
O=gpurun_out/${1:-alexncu}; mkdir -p $O
DS_ENGINE_NO_GRAPH=1 timeout 1500 ncu --set full --clock-control none --import-source on -k regex:gemm_tf32_kernel \
  --launch-skip 32 --launch-count 32 -o $O/alex_gemm python tools/prof_alex.py 2 > $O/ncu.log 2>&1
ncu -i $O/alex_gemm.ncu-rep --page raw --csv --metrics gpu__time_duration.sum,launch__grid_size,launch__block_size,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed > $O/alex_gemm_raw.csv 2>&1
echo done
