#!/bin/bash
# Timing experiments on the box: build variants of the library out of tree (/tmp) with
# -D flags and run the C2 probe on each.  usage: exp_variants.sh "-DFOO" "-DBAR" ...
mkdir -p gpurun_out
for v in "$@"; do
  d=/tmp/exp_$(echo "$v" | tr -c 'A-Za-z0-9' '_')
  rm -rf $d; mkdir -p $d
  cp -r paper_2604_10907_b200 tools include $d/
  (cd $d/paper_2604_10907_b200 && make clean >/dev/null && make -j8 EXTRA="$v" >/dev/null 2>&1) || echo "build $v failed"
  echo "=== variant $v" | tee -a gpurun_out/exp.txt
  (cd $d && timeout 120 python tools/probe_one.py C2 296 2>&1) | tee -a gpurun_out/exp.txt | grep -E "kernel|load|empty|walk|pass |stage|slowcyc"
done
