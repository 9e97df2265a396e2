#!/bin/bash
# First GPU pass of a session: parity tests, a bench line, the ncu launch list.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
lscpu > gpurun_out/lscpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 50 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e \
  > gpurun_out/bench_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/bench_ncu.log
