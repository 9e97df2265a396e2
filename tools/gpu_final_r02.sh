#!/bin/bash
# Final round-2 evidence on the committed tree: sanitizers on small sweeps, the bench launch
# list with DRAM traffic, and the sections capture of a 296-setup C3 launch.
mkdir -p gpurun_out
timeout 900 compute-sanitizer --tool synccheck python tools/probe_one.py C3 4 trunc 3000 > gpurun_out/san_synccheck_f.txt 2>&1
timeout 900 compute-sanitizer --tool memcheck python tools/probe_one.py C5 2 trunc 3000 > gpurun_out/san_memcheck_f.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02f_launches_c3.csv python bench.py --steps 1 --warmup 1 --no-cpu --no-e2e > gpurun_out/ncu_bench_f.log 2>&1
timeout 1500 ncu --section SpeedOfLight --section WarpStateStats --section SchedulerStats \
  --section MemoryWorkloadAnalysis --section Occupancy --section SourceCounters \
  --section LaunchStats --clock-control none --import-source on -k regex:solver_kernel -c 1 \
  -o gpurun_out/r02f_c3_sections python tools/probe_one.py C3 296 > gpurun_out/ncu_sections_f.log 2>&1
tail -2 gpurun_out/san_synccheck_f.txt gpurun_out/san_memcheck_f.txt gpurun_out/ncu_bench_f.log gpurun_out/ncu_sections_f.log
ls -la gpurun_out | tail -8
