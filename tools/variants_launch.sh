#!/bin/bash
# per-variant kernel time of one kernel (ncu launch list); experiments only
out=gpurun_out/variants_launch.txt; : > $out
pat="$1"; shift
for v in "$@"; do
  SAD_NVCC_EXTRA="$v" python -m paper_0901_2742_b200.build --force > /dev/null 2>&1 || { echo "$v: build failed" >> $out; continue; }
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:$pat" -c 3 --csv --log-file /tmp/l.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline > /dev/null 2>&1
  echo "$v: $(grep -o '"gpu__time_duration.sum","[a-z]*","[0-9.,]*"' /tmp/l.csv | tail -2 | tr '\n' ' ')" >> $out
done
python -m paper_0901_2742_b200.build --force > /dev/null 2>&1
