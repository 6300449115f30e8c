"""Hot SASS instructions of one kernel in an ncu report: stall samples and executed counts.

    python tools/ncu_sass_hot.py gpurun_out/prof.ncu-rep k_profile [top]
"""
import collections
import csv
import io
import subprocess
import sys


def main(rep, kern, top=40):
    out = subprocess.run(["ncu", "-i", rep, "-k", f"regex:{kern}", "--page", "source", "--csv"],
                         capture_output=True, text=True).stdout
    lines = out.splitlines()
    hi = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
    rows = list(csv.reader(io.StringIO("\n".join(lines[hi:]))))
    h = rows[0]
    si, ei, src = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed"), h.index("Source")
    data = []
    for r in rows[1:]:
        if len(r) <= ei or not r[si].strip().isdigit():
            continue
        data.append((int(r[si]), int(r[ei] or 0), r[0], r[src].strip()))
    tot_s = sum(d[0] for d in data) or 1
    tot_e = sum(d[1] for d in data) or 1
    print(f"{len(data)} SASS lines, {tot_s} stall samples, {tot_e} warp instructions")
    byop = collections.Counter()
    byop_e = collections.Counter()
    for s, e, a, t in data:
        op = t.split()[0] if not t.startswith("@") else t.split()[1]
        byop[op.split(".")[0]] += s
        byop_e[op.split(".")[0]] += e
    print("by opcode (stall %, exec %):")
    for op, s in byop.most_common(15):
        print(f"  {op:10s} {100 * s / tot_s:5.1f}% {100 * byop_e[op] / tot_e:5.1f}%")
    print("hottest instructions:")
    for s, e, a, t in sorted(data, reverse=True)[:top]:
        print(f"  {100 * s / tot_s:5.1f}% exec {e:10d}  {a[-5:]}  {t[:90]}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 40)
