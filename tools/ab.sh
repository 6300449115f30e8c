#!/bin/bash
# A/B of libsad builds on the GPU box: tools/ab.sh ROUNDS lib1[:ENV=VAL] lib2 ... -> gpurun_out/ab.txt
out=gpurun_out/ab.txt; : > $out
rounds=$1; shift
for r in $(seq $rounds); do
  for spec in "$@"; do
    lib=${spec%%:*}; envs=""; [[ "$spec" == *:* ]] && envs=${spec#*:}
    res=$(env SAD_LIB_PATH=$lib $envs timeout 180 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('%.4f %.4f %.4f %.4f' % (d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['operand_build_ms']))")
    echo "$spec: $res" >> $out
  done
done
