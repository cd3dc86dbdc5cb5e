#!/bin/bash
# Round evidence: bench line, launch list (ncu, one decompose), full ncu capture of the dominant launch.
# Usage: tools/round_profile.sh TAG   (outputs under gpurun_out/)
TAG=${1:-r}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > gpurun_out/smi_$TAG.txt 2>&1
./tools/ffma_peak > gpurun_out/ffma_$TAG.json 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_$TAG.log
timeout 300 python tools/one_decompose.py c5 2 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
  --log-file gpurun_out/launches_$TAG.csv python tools/one_decompose.py c5 1 > gpurun_out/ncu_launch_$TAG.log 2>&1
python tools/launches.py gpurun_out/launches_$TAG.csv > gpurun_out/launches_$TAG.txt 2>&1
# the dominant launch: fine kernel, level 1 (the first fine launch: the largest level runs first)
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:fine_kernel --launch-skip 0 -c 1 \
  -o gpurun_out/full_$TAG -f python tools/one_decompose.py c5 1 > gpurun_out/ncufull_$TAG.log 2>&1
timeout 600 python tools/shard_times.py c5 1 2 4 8 > gpurun_out/shards_$TAG.log 2>&1
echo done
timeout 600 python tools/fista_bench.py 38 > gpurun_out/fista_$TAG.log 2>&1
ncu -i gpurun_out/full_$TAG.ncu-rep --page details --csv > gpurun_out/ncu_details_$TAG.csv 2>&1
ncu -i gpurun_out/full_$TAG.ncu-rep --page raw --csv > gpurun_out/ncu_raw_$TAG.csv 2>&1
