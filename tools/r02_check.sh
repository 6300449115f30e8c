#!/bin/bash
# GPU box: rebuild, GPU tests (optional -k filter), bench line, rank share at G = 1 and 8, and the
# per-kernel launch lists of the bench step and of the G = 8 virtual rank.
# usage: tools/r02_check.sh TAG [pytest -k expression | all | none]
tag=$1; sel=${2:-all}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$tag.log 2>&1 || { echo build failed; tail gpurun_out/build_$tag.log; exit 1; }
if [ "$sel" = all ]; then timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_$tag.log 2>&1
elif [ "$sel" != none ]; then timeout 900 python -m pytest tests -m gpu -x -q -k "$sel" > gpurun_out/gputest_$tag.log 2>&1; fi
echo "pytest rc=$?"; tail -2 gpurun_out/gputest_$tag.log 2>/dev/null
python bench.py --no-cpu-baseline > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo "bench rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/bench_$tag.json').readline()); r=d['roofline']; print('step', d['ms_per_step'], 'e2e', d['e2e']['ms_per_step'], 'k5', r['kernel_ms'], 'op', r['operand_build_ms'], d['clocks'])"
python tools/rank_share.py 1 8 > gpurun_out/share_$tag.txt 2>&1; cat gpurun_out/share_$tag.txt
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu rc=$?"
python tools/launches.py gpurun_out/launches_$tag.csv 0 > gpurun_out/launches_${tag}_summary.txt 2>&1
head -16 gpurun_out/launches_${tag}_summary.txt
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_g8_$tag.csv \
    python tools/rank_share.py 8 > /dev/null 2>&1; echo "ncu g8 rc=$?"
python tools/launches.py gpurun_out/launches_g8_$tag.csv 0 > gpurun_out/launches_g8_${tag}_summary.txt 2>&1
cat gpurun_out/launches_g8_${tag}_summary.txt
