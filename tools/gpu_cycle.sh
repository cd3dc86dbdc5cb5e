#!/bin/bash
# One GPU iteration: parity tests, bench, launch list, one full ncu capture of the top kernel.
# Usage: tools/gpu_cycle.sh TAG [pytest-args]
TAG=${1:-x}
shift
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > gpurun_out/smi_$TAG.txt 2>&1
./tools/ffma_peak > gpurun_out/ffma_$TAG.json 2>&1
timeout 1500 python -m pytest tests -m gpu -q --tb=short -p no:cacheprovider "$@" > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_$TAG.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench_$TAG.log
timeout 300 python tools/one_decompose.py c5 2 > gpurun_out/one_$TAG.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_$TAG.csv python tools/one_decompose.py c5 1 > gpurun_out/ncu_$TAG.log 2>&1
python tools/launches.py gpurun_out/launches_$TAG.csv > gpurun_out/launches_$TAG.txt 2>&1
if [ -n "$NCU_FULL" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$NCU_FULL" -c ${NCU_COUNT:-1} \
    -o gpurun_out/full_$TAG -f python tools/one_decompose.py c5 1 > gpurun_out/ncufull_$TAG.log 2>&1
fi
echo done
