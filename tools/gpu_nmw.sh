#!/bin/bash
# A/B of tensor-core step builds (tools/_var) on one box + the TC parity tests of the default build
cd "$(dirname "$0")/.." || exit 1
O=gpurun_out/${1:-nmw}; mkdir -p $O
for v in ${VARIANTS:-HEAD DS_TC_NMW=1 DS_TC_NMW=2 default DS_TC_NMW=4}; do
  if [ $v = default ]; then LIB=""; else LIB="tools/_var/libds_cuda_$v.so"; fi
  DS_LIB_PATH=$LIB DS_FUSED_PROFILE=$O/prof_$v.txt timeout 120 python tools/prof_tc.py 3000 > $O/prof_$v.log 2>&1
  DS_LIB_PATH=$LIB timeout 300 python bench.py --no-extras --cifar-steps 0 --alexnet-steps 0 > $O/bench_$v.json 2> $O/bench_$v.err
done
DS_LIB_PATH=${TEST_LIB:-} timeout 900 python -m pytest tests/test_gpu_tc.py tests/test_gpu_engine.py -q -x -p no:cacheprovider > $O/tc_tests.log 2>&1; echo "rc=$?" >> $O/tc_tests.log
