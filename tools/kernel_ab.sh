#!/bin/bash
# per-kernel A/B of prebuilt libraries (GPU box): tools/kernel_ab.sh REGEX lib1 lib2 ...
# -> gpurun_out/kernel_ab.txt: median duration (us) of the whole-step launches matching REGEX (ncu
# launch list, serialized, config 4 G = 1) and the G = 8 virtual-rank step (tools/rank_share.py 8)
out=gpurun_out/kernel_ab.txt
re=$1; shift
for lib in "$@"; do
  SAD_LIB_PATH=$lib ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:$re" --csv --log-file gpurun_out/kab.csv \
      python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-graph > /dev/null 2>&1
  r=$(python - <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/kab.csv")))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]; vi, ui = h.index("Metric Value"), h.index("Metric Unit")
v = [float(r[vi].replace(",", "")) * {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}[r[ui]] for r in rows[hi + 1:] if len(r) > vi]
d = sorted(x for x in v if x > 0.6 * max(v)) if v else []
print(f"n={len(d)} median={d[len(d) // 2]:.2f} us min={d[0]:.2f} us" if d else "none")
PY
)
  g8=$(SAD_LIB_PATH=$lib timeout 300 python tools/rank_share.py 8 2>/dev/null | grep -o "graph-replayed step [0-9.]* ms" | head -1)
  echo "$lib: $re $r; G=8 $g8" >> $out
done
