#!/bin/bash
# Build a tuning variant of the step kernel: scripts/build_variant.sh NAME "-DFLAG=..."
# -> paper_1909_05098_b200/libfedheat_b200_NAME.so (use with FH_LIB=...); other units shared.
set -e
cd "$(dirname "$0")/../paper_1909_05098_b200/csrc"
test -f build/fh_exact.o || make -s  # shared units only; the main library is left as it is
mkdir -p build_$1
NV=/usr/local/cuda/bin/nvcc
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I../../include --expt-relaxed-constexpr"
$NV $FL $2 -Xptxas -v -c fh_tiled.cu -o build_$1/fh_tiled.o 2> build_$1/ptxas.txt
$NV $FL $2 -c fh_api.cu -o build_$1/fh_api.o
$NV -gencode arch=compute_100a,code=sm_100a -shared -o ../libfedheat_b200_$1.so build_$1/fh_api.o build_$1/fh_tiled.o \
  build/fh_exact.o build/fh_precompute.o build/fh_partition.o build/fh_dist.o build/fh_meshio.o -lcudart_static -lrt -ldl -lpthread
echo built libfedheat_b200_$1.so
