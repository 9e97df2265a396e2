#!/bin/bash
# Build each variant tree given as an argument, then bench them round-robin twice.
for B in "$@"; do (cd $B/paper_2604_10907_b200 && make -j8 >/dev/null 2>&1) || echo "build $B failed"; done
for r in 1 2; do
  for d in . "$@"; do
    (cd $d && timeout 300 python bench.py --no-cpu --no-e2e --steps 3 --warmup 3 2>/dev/null) | python -c "import json,sys; l=json.loads(sys.stdin.read()); print('$d', round(l['kernel_ms_per_step'],1), '%.4g' % l['value'])"
  done
done
