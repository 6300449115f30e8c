"""Summarise an ncu --metrics gpu__time_duration.sum launch list: per-kernel totals per step."""
import collections
import csv
import sys


def main(path, steps):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0}.get(r[ui], 1e-6)
        name = r[ki].split("(")[0][:60]
        tot[name] += v
        cnt[name] += 1
    allms = sum(tot.values())
    if steps <= 0:   # auto: one all-pairs launch per step
        steps = float(max(c for k, c in cnt.items() if "syrk" in k or "allpairs" in k))
    print(f"{len(rows) - hi - 1} launches, {allms / steps:.3f} ms of kernel time per step ({steps} steps)")
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{v / steps:9.4f} ms/step {cnt[k] / steps:5.1f} launches/step {100 * v / allms:5.1f}%  {k}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 0.0)
