#!/bin/bash
# Round-2 profiling evidence on the GPU box: launch list of the bench step (ncu, serialized,
# cold-cache; only the kernels' SHARE of the step is comparable with the bench) and one
# `ncu --set full` capture of every kernel of the step (one launch each), summarised per kernel.
# usage: tools/r02_profile.sh TAG [bench args...]
tag=$1; shift
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-graph "$@" > gpurun_out/ncu_launch_$tag.log 2>&1
echo "ncu launches rc=$?"
python tools/launches.py gpurun_out/launches_$tag.csv 0 > gpurun_out/launches_${tag}_summary.txt 2>&1
ncu --set full --clock-control none --import-source on \
    -k "regex:k_profile<|k_xrows_g|k_xfill|k_indicator|k_rank_vs_ga|k_seg_sort|k_merge_runs|k_syrk_tc|k_shard_plan|k_plan|k_rank_merge|k_gather_res|k_local_anc|k_lenscatter|k_f1_" \
    -s 40 -c 16 -f -o gpurun_out/prof_$tag \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph "$@" > gpurun_out/ncu_full_$tag.log 2>&1
echo "ncu full rc=$?"
