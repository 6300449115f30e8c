#!/bin/bash
# Round-2 results table: one bench line per config / layout on this B200, the CPU
# oracle beside it (all host threads; 1 thread for configs 1-2), plus the f1 / f2 modes of config 4.
# usage: tools/r02_results.sh   (GPU box) -> gpurun_out/res_*.json
mkdir -p gpurun_out
run() { tag=$1; shift; python bench.py --cpu-seconds 8 "$@" > gpurun_out/res_$tag.json 2> gpurun_out/res_$tag.err; echo "$tag rc=$?"; }
run cfg1_p2 --config 1
run cfg1_p2_t1 --config 1 --oracle-threads 1
run cfg2_p8 --config 2
run cfg2_p8_t1 --config 2 --oracle-threads 1
run cfg3_p2 --config 3 --p 2
run cfg3_p4 --config 3 --p 4
run cfg3_p8 --config 3 --p 8
run cfg4_p8 --config 4
run cfg5_p1 --config 5 --p 1
run cfg5_p8 --config 5 --p 8
run cfg4_p8_f1 --config 4 --rank-mode samples --no-cpu-baseline
run cfg4_p1_f2 --config 4 --p 1 --no-cpu-baseline --steps 5
