#!/bin/bash
# Round profile: launch list of the bench command + one full capture of the solver kernel.
mkdir -p gpurun_out
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e \
  > gpurun_out/bench_under_ncu.log 2>&1
echo "launch list rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:solver_kernel -s 1 -c 1 \
  -o gpurun_out/bench_full python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e \
  > gpurun_out/ncu_full.log 2>&1
echo "full capture rc=$?"
