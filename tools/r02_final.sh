#!/bin/bash
# GPU box, end of round 2: bench line (with the CPU oracle beside it), launch list, per-kernel ncu
# summaries of the step's main kernels, and the virtual-rank projections for configs 3, 4 and 5.
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_final.log 2>&1 || { echo build failed; exit 1; }
python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo "bench rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu launches rc=$?"
python tools/launches.py gpurun_out/launches_final.csv 0 > gpurun_out/launches_final_summary.txt 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_syrk|k_profile<|k_xrows_g|k_indicator|k_xfill|k_rank_vs_ga|k_shard_plan" \
    -s 40 -c 7 -f -o gpurun_out/prof_final python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_final.log 2>&1
echo "ncu full rc=$?"
for G in "--cfg 4 --p 8 1 2 4 8" "--cfg 5 --p 8 1 2 4 8" "--cfg 3 --p-eq-g 1 2 4 8"; do
  python tools/rank_share.py $G >> gpurun_out/share_final.txt 2>&1
done
cat gpurun_out/share_final.txt
