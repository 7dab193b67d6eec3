#!/bin/bash
# Instrumented / A-B variant of libds_cuda.so with extra defines on mlp_tc.cu (tools/ experiments):
#   tools/build_variant.sh NAME DEF1 [DEF2 ...]  -> tools/_var/libds_cuda_NAME.so
#   (tools/build_variant.sh DS_TC_PROF_X DS_TC_PROF_X)
# Load it with DS_LIB_PATH=tools/_var/libds_cuda_NAME.so.
set -e
cd "$(dirname "$0")/.."
NAME=$1; shift
DEFS=""; for d in "$@"; do DEFS="$DEFS -D$d"; done
mkdir -p tools/_var build/var
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -ccbin /usr/bin/g++ -Xcompiler -fPIC -Iinclude -Ipaper_1602_08191_b200/csrc --expt-relaxed-constexpr -diag-suppress 177"
$NV $DEFS -c paper_1602_08191_b200/csrc/mlp_tc.cu -o build/var/mlp_tc_$NAME.o
OBJS=$(ls build/csrc/*.o | grep -v "/cpp_" | grep -v "/mlp_tc.o")
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -ccbin /usr/bin/g++ -shared -cudart static \
  -o tools/_var/libds_cuda_$NAME.so $OBJS build/var/mlp_tc_$NAME.o -lpthread -ldl -lrt
echo tools/_var/libds_cuda_$NAME.so
