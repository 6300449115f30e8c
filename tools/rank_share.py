"""Device time of one rank's share of config 4 at G GPUs (p = 8 shards, p/G per rank), on one GPU:
every stage up to the partition plan, with the exchanged buffers emulated by repeating this
rank's own (the collectives themselves are not timed). A lower bound of the per-GPU step at G."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0901_2742_b200.runtime import Context  # noqa: E402
from synth import gen  # noqa: E402


def main(G=8, steps=10):
    spec = gen.SPECS[4]
    a, o = gen.generate(spec)
    n, p = len(o) - 1, 8
    pl = p // G
    sb = gen.shard_bounds(n, p)
    lo, hi = sb[0], sb[pl]
    dev = torch.device("cuda", 0)
    d_a = torch.from_numpy(np.ascontiguousarray(a[o[lo]: o[hi]])).to(dev)
    d_o = torch.from_numpy(np.ascontiguousarray(o[lo: hi + 1] - o[lo])).to(dev)
    ctx = Context(spec.alphabet, spec.k, p, world=G, rank=0, kernel="tc")
    st = torch.cuda.current_stream(dev)
    R = int(o[hi] - o[lo])

    names = ["load", "build_profiles", "rank_local", "rank_global", "plan"]
    evs = []

    def step():
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
        ev[0].record(st)
        ctx.load(d_a, d_o, n, lo, residues=R)
        ev[1].record(st)
        ctx.build_profiles()
        ev[2].record(st)
        anc = ctx.rank_local()
        ev[3].record(st)
        smp = ctx.rank_global(anc.repeat(G, 1))
        ev[4].record(st)
        ctx.partition_plan(smp.repeat(G))
        ev[5].record(st)
        evs.append(ev)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    ms = []
    for _ in range(steps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(st)
        step()
        e.record(st)
        torch.cuda.synchronize()
        ms.append(s.elapsed_time(e))
    parts = np.median([[e[i].elapsed_time(e[i + 1]) for i in range(5)] for e in evs[3:]], axis=0)
    print(f"G={G}: one rank's share ({hi - lo} sequences, {pl} shard(s)) {np.median(ms):.3f} ms/step up to the plan | " +
          " ".join(f"{nm}={x:.3f}" for nm, x in zip(names, parts)))


if __name__ == "__main__":
    for g in ([int(x) for x in sys.argv[1:]] or (1, 2, 4, 8)):
        main(g)
