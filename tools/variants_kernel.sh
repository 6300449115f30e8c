#!/bin/bash
# compile-time variants timed per kernel (ncu launch list, serialized): tools/variants_kernel.sh REGEX "flags1" "flags2" ...
# (GPU box) -> gpurun_out/variants_kernel.txt: mean duration (us) of the kernels matching REGEX per variant
out=gpurun_out/variants_kernel.txt; : > $out
re=$1; shift
for v in "$@"; do
  SAD_NVCC_EXTRA="$v" python -m paper_0901_2742_b200.build --force > /dev/null 2>&1 || { echo "$v: build failed" >> $out; continue; }
  ncu --metrics gpu__time_duration.sum --clock-control none -k "regex:$re" --csv --log-file gpurun_out/vk.csv \
      python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-graph > /dev/null 2>&1
  r=$(python - <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/vk.csv")))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hi]; vi, ui = h.index("Metric Value"), h.index("Metric Unit")
v = [float(r[vi].replace(",", "")) * {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3}[r[ui]] for r in rows[hi + 1:] if len(r) > vi]
# whole-step launches only (the chunked host loads of the e2e part launch K1/K2 per chunk)
d = sorted(x for x in v if x > 0.6 * max(v)) if v else []
print(f"device-step launches n={len(d)} median={d[len(d) // 2]:.2f} us min={d[0]:.2f} us" if d else "none")
PY
)
  echo "$v: $r" >> $out
done
python -m paper_0901_2742_b200.build --force > /dev/null 2>&1
