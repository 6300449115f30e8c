#!/bin/bash
# A/B of libsad builds on configs 4 and 5 (GPU box): tools/ab_configs.sh lib1 lib2 ... -> gpurun_out/ab5.txt
out=gpurun_out/ab5.txt; : > $out
for r in 1 2; do for lib in "$@"; do
 for cfg in 4 5; do
  res=$(SAD_LIB_PATH=$lib timeout 180 python bench.py --config $cfg --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4f %.4f %.4f' % (d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac']))")
  echo "$lib cfg$cfg: $res" >> $out
 done; done; done
