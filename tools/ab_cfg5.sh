#!/bin/bash
# A/B of libsad builds on config 5 only (GPU box) -> gpurun_out/ab_c5.txt
out=gpurun_out/ab_c5.txt; : > $out
for r in 1 2; do for lib in "$@"; do
  res=$(SAD_LIB_PATH=$lib timeout 180 python bench.py --config 5 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4f %.4f %.4f' % (d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['frac']))")
  echo "$lib cfg5: $res" >> $out
done; done
