#!/bin/bash
# K5 wait-time profile (SAD_TC_DBG_PROF printf build, extra flags in $PROF_FLAGS) + timing variants (GPU box)
: > gpurun_out/tcprof.txt
for pf in "" $PROF_FLAGS; do
  SAD_NVCC_EXTRA="-DSAD_TC_DBG_PROF ${pf//,/ }" python -m paper_0901_2742_b200.build --force > /dev/null 2>&1 || { echo "prof build failed"; continue; }
  echo "== prof $pf" >> gpurun_out/tcprof.txt
  timeout 180 python bench.py --steps 1 --warmup 3 --no-cpu-baseline 2>/dev/null | grep tcprof | grep "blk 0 " | tail -6 >> gpurun_out/tcprof.txt
done
bash tools/variants.sh "$@"
