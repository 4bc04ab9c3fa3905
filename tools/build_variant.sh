#!/bin/bash
# tools/build_variant.sh NAME "NVCC FLAGS" -- libcnmf_b200.so with every CUDA
# source recompiled under extra -D flags, in paper_1712_02248_b200/build_var/NAME
# (kernel experiments; select with CNMF_LIB=.../libcnmf_b200.so).
set -e
R=/root/repo/paper_1712_02248_b200
O=$R/build_var/$1
mkdir -p $O
for f in rng xstream xstream_tc xstream_i8 recon_tc qr hals hals_resident metrics synth dense sparse; do
  /usr/local/cuda/bin/nvcc -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC \
    --expt-relaxed-constexpr $2 -c $R/csrc/$f.cu -o $O/$f.o 2>&1 | grep -E " error" || true &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static \
  -o $O/libcnmf_b200.so $O/*.o $R/build/engine.o $R/build/mt_jump.o $R/build/data_io.o -ldl
echo "built $1"
