#!/bin/bash
# One GPU iteration: parity tests, bench, launch list.  Usage: tools/gpu_cycle.sh TAG [pytest-args]
TAG=${1:-x}
shift
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q --tb=short -p no:cacheprovider "$@" > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench_$TAG.log 2>&1
python tools/one_decompose.py c5 2 > gpurun_out/one_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_$TAG.csv python tools/one_decompose.py c5 1 > gpurun_out/ncu_$TAG.log 2>&1
echo done
