#!/bin/bash
TAG=r2q
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > gpurun_out/smi_$TAG.txt 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?"
timeout 300 python tools/launch_profile.py c5 > gpurun_out/launch_profile_c5_$TAG.json 2>/dev/null
timeout 300 python tools/one_decompose.py c5 2 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
  --log-file gpurun_out/launches_$TAG.csv python tools/one_decompose.py c5 1 > gpurun_out/ncu_launch_$TAG.log 2>&1
python tools/launches.py gpurun_out/launches_$TAG.csv > gpurun_out/launches_$TAG.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fine_kernel --launch-skip 0 -c 1 \
  -o gpurun_out/full_$TAG -f python tools/one_decompose.py c5 1 > gpurun_out/ncufull_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fine_kernel --launch-skip 2 -c 1 \
  -o gpurun_out/full_l3_$TAG -f python tools/one_decompose.py c5 1 > gpurun_out/ncufull_l3_$TAG.log 2>&1
ncu -i gpurun_out/full_$TAG.ncu-rep --page details --csv > gpurun_out/ncu_details_$TAG.csv 2>&1
ncu -i gpurun_out/full_$TAG.ncu-rep --page raw --csv > gpurun_out/ncu_raw_$TAG.csv 2>&1
ncu -i gpurun_out/full_l3_$TAG.ncu-rep --page details --csv > gpurun_out/ncu_details_l3_$TAG.csv 2>&1
ncu -i gpurun_out/full_l3_$TAG.ncu-rep --page raw --csv > gpurun_out/ncu_raw_l3_$TAG.csv 2>&1
ncu -i gpurun_out/full_$TAG.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/ncu_source_$TAG.csv 2>&1
mkdir -p /tmp/reps; mv gpurun_out/*.ncu-rep /tmp/reps/ 2>/dev/null; du -sh gpurun_out
echo done
