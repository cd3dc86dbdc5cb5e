#!/bin/bash
# Final evidence on HEAD (after the d = 3 path): full GPU suite, smoke, bench, ncu of the d = 3 kernel.
TAG=r2zz
mkdir -p gpurun_out; rm -f gpurun_out/parity_errors.jsonl
timeout 1500 python -m pytest tests -m gpu -q --tb=short -p no:cacheprovider > gpurun_out/pytest_gpu_$TAG.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
cp gpurun_out/parity_errors.jsonl gpurun_out/parity_errors_$TAG.jsonl 2>/dev/null
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_$TAG.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
echo "bench rc=$?"
timeout 300 python tools/volume_bench.py > /dev/null 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:rows3d_kernel --launch-skip 7 -c 1 \
  -o gpurun_out/full_vol_$TAG -f python tools/volume_bench.py > gpurun_out/ncufull_vol_$TAG.log 2>&1
ncu -i gpurun_out/full_vol_$TAG.ncu-rep --page details --csv > gpurun_out/ncu_full_rows3d_64_$TAG.csv 2>&1
ncu -i gpurun_out/full_vol_$TAG.ncu-rep --page raw --csv > gpurun_out/ncu_raw_rows3d_64_$TAG.csv 2>&1
rm -f gpurun_out/*.ncu-rep
tail -3 gpurun_out/pytest_gpu_$TAG.log
echo done
