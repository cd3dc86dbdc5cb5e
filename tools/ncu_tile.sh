#!/bin/bash
# Full ncu capture of one band_tile_kernel launch (SKIP = launches to skip; Λ order: level 4, 3, 2, 1).
TAG=${1:-x}; SKIP=${2:-3}; KERN=${3:-band_tile_kernel}
mkdir -p gpurun_out
timeout 300 python tools/one_decompose.py c5 1 > gpurun_out/pre_$TAG.log 2>&1 || exit 1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$KERN" --launch-skip $SKIP -c 1 \
  -o gpurun_out/full_$TAG -f python tools/one_decompose.py c5 1 > gpurun_out/ncufull_$TAG.log 2>&1
echo done
