#!/bin/bash
# exchange-path A/B: committed build (tools/_var/libds_cuda_HEAD.so) vs the working tree
cd "$(dirname "$0")/.." || exit 1
O=gpurun_out/${1:-xab}; mkdir -p $O
for v in HEAD default HEAD default; do
  if [ $v = default ]; then LIB=""; else LIB="tools/_var/libds_cuda_$v.so"; fi
  DS_LIB_PATH=$LIB timeout 300 python tools/prof_tc_det.py 6000 >> $O/det_$v.log 2>&1
  DS_LIB_PATH=$LIB timeout 300 python bench.py --no-extras --cifar-steps 0 --alexnet-steps 0 >> $O/bench_$v.jsonl 2>> $O/bench_$v.err
done
DS_LIB_PATH=tools/_var/libds_cuda_profx.so DS_TC_PROF_X=1 DS_FUSED_PROFILE=$O/prof_x.txt timeout 300 python tools/prof_tc_det.py 3000 > $O/x.log 2>&1
timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_master.py -q -x -p no:cacheprovider > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
