#!/bin/bash
# e2e step time against the number of H2D/k-mer-count pipeline chunks of sad_load (GPU box)
out=gpurun_out/e2e_chunks.txt; : > $out
for c in "$@"; do
  r=$(SAD_LOAD_CHUNKS=$c timeout 180 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['e2e']['ms_per_step'])")
  echo "chunks=$c: $r" >> $out
done
