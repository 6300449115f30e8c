#!/bin/bash
out=gpurun_out/variants_clk.txt; : > $out
for v in "$@"; do
  SAD_NVCC_EXTRA="$v" python -m paper_0901_2742_b200.build --force > /dev/null 2>&1 || { echo "$v: build failed" >> $out; continue; }
  echo "$v: $(python tools/clock_probe.py 2>&1 | tail -1)" >> $out
done
python -m paper_0901_2742_b200.build --force > /dev/null 2>&1
