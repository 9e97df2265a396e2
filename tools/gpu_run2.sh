#!/bin/bash
# Per-phase breakdown + one full ncu capture of the bench kernel.
set -x
mkdir -p gpurun_out
timeout 300 python tools/probe_one.py C2 296 > gpurun_out/probe_one_c2.log 2>&1
timeout 300 python tools/probe_pass.py C2 200 > gpurun_out/probe_pass_c2.log 2>&1
timeout 300 python tools/probe_pass.py C1 500 > gpurun_out/probe_pass_c1.log 2>&1
timeout 300 python tools/probe_pass.py C3 20 > gpurun_out/probe_pass_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -c 1 \
  -o gpurun_out/bench_full python bench.py --steps 1 --warmup 0 --no-cpu --no-e2e \
  > gpurun_out/ncu_full.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full.log
