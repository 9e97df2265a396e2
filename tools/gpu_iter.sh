#!/bin/bash
# Iteration loop on the box: parity tests, diagnostics probe, optional bench line.
mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -4 gpurun_out/pytest_gpu.log
timeout 120 python tools/probe_one.py C2 296 > gpurun_out/probe_one_c2.log 2>&1
cat gpurun_out/probe_one_c2.log
if [ "$1" == "bench" ]; then
  timeout 300 python bench.py --no-cpu > gpurun_out/bench.log 2>&1
  tail -c 1500 gpurun_out/bench.log
fi
