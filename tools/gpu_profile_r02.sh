#!/bin/bash
# Round-2 evidence run (on the B200 box): sanitizers on a small C3 sweep, the bench launch
# list and DRAM traffic of the C3 bench kernel, one `--set full` capture of the C3 kernel.
set -x
mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool synccheck python tools/probe_one.py C3 4 trunc 3000 > gpurun_out/san_synccheck.txt 2>&1
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard python tools/probe_one.py C3 2 trunc 2000 > gpurun_out/san_racecheck.txt 2>&1
timeout 900 compute-sanitizer --tool memcheck python tools/probe_one.py C5 2 trunc 3000 > gpurun_out/san_memcheck.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02_launches_c3.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_bench.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:solver_kernel -c 1 -o gpurun_out/r02_c3_full python tools/probe_one.py C3 296 > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
