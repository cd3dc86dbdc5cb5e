#!/bin/bash
# End-of-round evidence on HEAD: full GPU suite, smoke, bench, launch list, full ncu of fine level 1.
TAG=r2z
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu,power.draw --format=csv > gpurun_out/smi_$TAG.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q --tb=short -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
cp gpurun_out/parity_errors.jsonl gpurun_out/parity_errors_$TAG.jsonl 2>/dev/null
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_$TAG.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?"
timeout 300 python tools/one_decompose.py c5 2 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
  --log-file gpurun_out/launches_c5_$TAG.csv python tools/one_decompose.py c5 1 > gpurun_out/ncu_launch_$TAG.log 2>&1
python tools/launches.py gpurun_out/launches_c5_$TAG.csv > gpurun_out/launches_c5_$TAG.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fine_kernel --launch-skip 0 -c 1 \
  -o gpurun_out/full_$TAG -f python tools/one_decompose.py c5 1 > gpurun_out/ncufull_$TAG.log 2>&1
ncu -i gpurun_out/full_$TAG.ncu-rep --page details --csv > gpurun_out/ncu_full_fine_level1_$TAG.csv 2>&1
ncu -i gpurun_out/full_$TAG.ncu-rep --page raw --csv > gpurun_out/ncu_raw_fine_level1_$TAG.csv 2>&1
timeout 600 python tools/configs_bench.py > gpurun_out/configs_$TAG.jsonl 2> gpurun_out/configs_$TAG.err
rm -f gpurun_out/*.ncu-rep
echo done
