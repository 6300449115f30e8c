#!/bin/bash
# build compile-time variants and time each with the G = 8 virtual rank and the G = 1 bench step (GPU box)
out=gpurun_out/variants_share.txt; : > $out
for v in "$@"; do
  SAD_NVCC_EXTRA="$v" python -m paper_0901_2742_b200.build --force > /dev/null 2>&1 || { echo "$v: build failed" >> $out; continue; }
  g8=$(timeout 300 python tools/rank_share.py 8 2>/dev/null | grep -o "graph-replayed step [0-9.]* ms" | head -1)
  g1=$(timeout 180 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'])")
  echo "$v: G=8 $g8; G=1 bench step $g1 ms" >> $out
done
python -m paper_0901_2742_b200.build --force > /dev/null 2>&1
