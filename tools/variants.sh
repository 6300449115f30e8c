#!/bin/bash
# build + bench several compile-time variants of the all-pairs kernel (experiments; GPU box)
out=gpurun_out/variants.txt; : > $out
for v in "$@"; do
  SAD_NVCC_EXTRA="$v" python -m paper_0901_2742_b200.build --force > /dev/null 2>&1 || { echo "$v: build failed" >> $out; continue; }
  r=$(timeout 180 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['kernel_ms'], d['roofline']['operand_build_ms'])")
  echo "$v: $r" >> $out
done
python -m paper_0901_2742_b200.build --force > /dev/null 2>&1
