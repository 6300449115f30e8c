"""Run the all-pairs stage back to back for a few seconds while sampling SM clocks and power
(experiment: does the epilogue's ALU load pull the clock down under sustained tensor work?)."""
import os
import subprocess
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0901_2742_b200.runtime import Context  # noqa: E402
from synth import gen  # noqa: E402


def main(seconds=3.0, cfg=4):
    spec = gen.SPECS[cfg]
    a, o = gen.generate(spec)
    n = len(o) - 1
    dev = torch.device("cuda", 0)
    ctx = Context(spec.alphabet, spec.k, spec.p, kernel="tc")
    d_a, d_o = torch.from_numpy(a).to(dev), torch.from_numpy(o).to(dev)
    ctx.load(d_a, d_o, n, 0, residues=int(o[-1]))
    ctx.build_profiles()
    anc = ctx.rank_local()
    torch.cuda.synchronize()
    ctx.reset_stats()
    log = open("/tmp/clk.csv", "w")
    p = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.active",
                          "--format=csv,noheader,nounits", "-lms", "50"], stdout=log)
    t0 = time.time()
    calls = 0
    while time.time() - t0 < seconds:
        for _ in range(20):
            ctx.load(d_a, d_o, n, 0, residues=int(o[-1]))
            ctx.build_profiles()
            ctx.rank_local()
            calls += 1
        torch.cuda.synchronize()
    p.terminate()
    p.wait()
    log.close()
    st = ctx.stats()
    rows = [l.strip().split(",") for l in open("/tmp/clk.csv") if l.count(",") == 2]
    sm = sorted(float(r[0]) for r in rows)
    pw = sorted(float(r[1]) for r in rows)
    reasons = sorted(set(r[2].strip() for r in rows))
    print(f"calls {calls} allpairs ms/call {st['allpairs_ms_total'] / max(st['calls'], 1):.3f} "
          f"sm_mhz median {sm[len(sm) // 2]:.0f} min {sm[0]:.0f} power median {pw[len(pw) // 2]:.0f} W reasons {reasons}")


if __name__ == "__main__":
    main()
