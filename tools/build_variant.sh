#!/bin/bash
# tools/build_variant.sh NAME "NVCC FLAGS" -- libcnmf_b200.so with xstream_tc.cu
# recompiled under extra -D flags, in paper_1712_02248_b200/build_var/NAME
# (kernel experiments; select with CNMF_LIB=.../libcnmf_b200.so).
set -e
R=/root/repo/paper_1712_02248_b200
mkdir -p $R/build_var/$1
/usr/local/cuda/bin/nvcc -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC \
  --expt-relaxed-constexpr $2 -c $R/csrc/xstream_tc.cu -o $R/build_var/$1/xstream_tc.o 2>&1 | grep -E " error" || true
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static \
  -o $R/build_var/$1/libcnmf_b200.so $R/build_var/$1/xstream_tc.o $(ls $R/build/*.o | grep -v xstream_tc.o)
echo "built $1"
