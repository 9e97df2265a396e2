#!/bin/bash
# ncu capture of the C3 solver kernel (one 296-setup launch) with the sections that explain
# it (throughput, warp states, scheduler, memory, source counters) — `--set full` timed out
# on this 2 s persistent kernel.
mkdir -p gpurun_out
timeout 1500 ncu --section SpeedOfLight --section WarpStateStats --section SchedulerStats \
  --section MemoryWorkloadAnalysis --section Occupancy --section SourceCounters \
  --section LaunchStats --clock-control none --import-source on -k regex:solver_kernel -c 1 \
  -o gpurun_out/r02_c3_sections python tools/probe_one.py C3 296 > gpurun_out/ncu_sections.log 2>&1
tail -3 gpurun_out/ncu_sections.log
