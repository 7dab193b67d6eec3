#!/bin/bash
cd "$(dirname "$0")/.." || exit 1
O=gpurun_out/${1:-lastrel}; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_tc.py tests/test_gpu_master.py tests/test_mgpu.py -q -x -p no:cacheprovider > $O/tests.log 2>&1; echo "rc=$?" >> $O/tests.log
for v in gather default gather default; do
  if [ $v = default ]; then LIB=""; else LIB="tools/_var/libds_cuda_$v.so"; fi
  CUDA_VISIBLE_DEVICES=0 DS_LIB_PATH=$LIB timeout 300 python tools/prof_tc_det.py 6000 >> $O/det_$v.log 2>&1
done
echo done
