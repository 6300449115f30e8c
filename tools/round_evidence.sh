#!/bin/bash
# bench line + launch list + one ncu --set full capture of the all-pairs kernel (GPU box).
# usage: tools/round_evidence.sh TAG [bench args...]
tag=$1; shift
python bench.py "$@" > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo "bench rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline "$@" > /dev/null 2>&1; echo "ncu launches rc=$?"
python tools/launches.py gpurun_out/launches_$tag.csv 0 > gpurun_out/launches_${tag}_summary.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_syrk -s 3 -c 1 -f -o gpurun_out/prof_$tag \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline "$@" > gpurun_out/ncu_$tag.log 2>&1; echo "ncu full rc=$?"
