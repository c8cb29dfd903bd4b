#!/bin/bash
# Build a variant library: scripts/build_variant.sh NAME "-DFLAG=..."
# -> paper_1909_05098_b200/libfedheat_b200_NAME.so (use with FH_LIB=...).  The
# step kernels (fh_tiled.cu, fh_resident.cu, fh_atomic.cu) and fh_api.cu are
# rebuilt with the flags; the other units are shared with the main build.
#   scripts/build_variant.sh checked "-DFH_CHECKS"   device bounds checks (trap on failure)
set -e
cd "$(dirname "$0")/../paper_1909_05098_b200/csrc"
make -s  # shared units (the main library is left as it is)
mkdir -p build_$1
NV=/usr/local/cuda/bin/nvcc
FL="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I../../include --expt-relaxed-constexpr"
$NV $FL $2 -Xptxas -v -c fh_tiled.cu -o build_$1/fh_tiled.o 2> build_$1/ptxas.txt
$NV $FL $2 -fmad=false -c fh_resident.cu -o build_$1/fh_resident.o
$NV $FL $2 -c fh_atomic.cu -o build_$1/fh_atomic.o
$NV $FL $2 -c fh_api.cu -o build_$1/fh_api.o
$NV -gencode arch=compute_100a,code=sm_100a -shared -o ../libfedheat_b200_$1.so build_$1/fh_api.o build_$1/fh_tiled.o \
  build_$1/fh_resident.o build_$1/fh_atomic.o build/fh_exact.o build/fh_precompute.o build/fh_partition.o \
  build/fh_dist.o build/fh_meshio.o -lcudart_static -lrt -ldl -lpthread
echo built libfedheat_b200_$1.so
