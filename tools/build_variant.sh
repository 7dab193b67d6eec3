#!/bin/bash
# Instrumented variant of libds_cuda.so with one extra define on mlp_tc.cu (tools/ experiments):
#   tools/build_variant.sh DS_TC_PROF_X   -> tools/_var/libds_cuda_DS_TC_PROF_X.so
# Load it with DS_LIB_PATH=tools/_var/libds_cuda_<DEF>.so.
set -e
cd "$(dirname "$0")/.."
DEF=$1
mkdir -p tools/_var build/var
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -ccbin /usr/bin/g++ -Xcompiler -fPIC -Iinclude -Ipaper_1602_08191_b200/csrc --expt-relaxed-constexpr"
$NV -D$DEF -c paper_1602_08191_b200/csrc/mlp_tc.cu -o build/var/mlp_tc_$DEF.o
OBJS=$(ls build/csrc/*.o | grep -v "/cpp_" | grep -v "/mlp_tc.o")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -ccbin /usr/bin/g++ -shared -cudart static \
  -o tools/_var/libds_cuda_$DEF.so $OBJS build/var/mlp_tc_$DEF.o -lpthread -ldl -lrt
echo tools/_var/libds_cuda_$DEF.so
