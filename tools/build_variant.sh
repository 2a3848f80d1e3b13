#!/bin/bash
# build a variant library with extra nvcc flags: tools/build_variant.sh NAME "-DFOO=1 ..."
# -> paper_2508_19140_b200/libinpc_raster_NAME.so (A/B on the GPU box by copying it over libinpc_raster.so)
cd "$(dirname "$0")/.."
P=paper_2508_19140_b200
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -shared -Xcompiler -fPIC \
  -Xcompiler -fvisibility=hidden --expt-relaxed-constexpr -Xptxas -v $2 -I include -I $P/csrc $P/csrc/inpc_raster.cu \
  -o $P/libinpc_raster_$1.so > /tmp/ptxas_$1.txt 2>&1 || { tail -20 /tmp/ptxas_$1.txt; exit 1; }
echo built $P/libinpc_raster_$1.so
