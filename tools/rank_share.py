"""One rank's device share of the config-4 step at G GPUs (p = 8 shards, p/G per rank), measured
on ONE GPU: the G ranks of the split API run in one process (tests/test_gpu_multirank.py style,
real per-rank data, the exchanges done by host copies), and every call of rank 0 is bracketed by
CUDA events: load, build_profiles, rank_local (operand + all-pairs + ancestors), rank_global (GA,
rank vs GA, local sort, samples), plan, pack, finish (the receive-side merge of G runs). The sum is
the device time rank 0 spends per step at G, exchanges excluded; the projection adds a stated
estimate of the four NCCL steps and the one host round trip of sad_partition.

    python tools/rank_share.py [G ...]     (GPU box) -> one line per G
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0901_2742_b200.runtime import Context  # noqa: E402
from synth import gen  # noqa: E402

# Estimated cost of the exchange steps per step at G > 1 (not measurable on one GPU): three small
# ncclAllGathers (ancestor records 8 x 16 KB, samples 448 B, counts + status 8 x 160 B) at ~10 us
# each (NVLink/NVSwitch small-message latency), the count read-back + host decision ~20 us, and the
# all-to-all of ~3.5 MB per rank at an effective ~300 GB/s (~12 us) plus ~10 us of launch latency.
EXCHANGE_EST_MS = 0.072

NAMES = ["load", "build_profiles", "rank_local", "rank_global", "plan", "pack", "finish"]


def one(G: int, steps: int = 10, warmup: int = 3):
    spec = gen.SPECS[4]
    a, o = gen.generate(spec)
    n, p = len(o) - 1, 8
    pl = p // G
    sb = gen.shard_bounds(n, p)
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream(dev)
    ctxs, dat = [], []
    for r in range(G):
        lo, hi = sb[r * pl], sb[(r + 1) * pl]
        d_a = torch.from_numpy(np.ascontiguousarray(a[o[lo]: o[hi]])).to(dev)
        d_o = torch.from_numpy(np.ascontiguousarray(o[lo: hi + 1] - o[lo])).to(dev)
        ctxs.append(Context(spec.alphabet, spec.k, p, world=G, rank=r, kernel="tc", stream=st))
        dat.append((d_a, d_o, lo, int(o[hi] - o[lo])))
    rows = []
    for it in range(warmup + steps):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(14)]
        for r, c in enumerate(ctxs):
            d_a, d_o, lo, R = dat[r]
            if r == 0:
                ev[0].record(st)
            c.load(d_a, d_o, n, lo, residues=R)
            if r == 0:
                ev[1].record(st)
            c.build_profiles()
            if r == 0:
                ev[2].record(st)
        ancs = []
        for r, c in enumerate(ctxs):
            if r == 0:
                ev[3].record(st)
            ancs.append(c.rank_local())
            if r == 0:
                ev[4].record(st)
        anc_all = torch.cat(ancs)
        smps = []
        for r, c in enumerate(ctxs):
            if r == 0:
                ev[5].record(st)
            smps.append(c.rank_global(anc_all))
            if r == 0:
                ev[6].record(st)
        smp_all = torch.cat(smps)
        cnts = []
        for r, c in enumerate(ctxs):
            if r == 0:
                ev[7].record(st)
            cnts.append(c.partition_plan(smp_all))
            if r == 0:
                ev[8].record(st)
        counts_all = torch.cat(cnts).cpu().numpy().reshape(p, p, 2)
        sends = []
        for r, c in enumerate(ctxs):
            if r == 0:
                ev[9].record(st)
            sends.append(c.pack(counts_all) if G > 1 else None)
            if r == 0:
                ev[10].record(st)
        for r, c in enumerate(ctxs):
            if G > 1:
                rm = torch.cat([torch.split(s[0], [int(x) for x in s[2]])[r] for s in sends])
                rr = torch.cat([torch.split(s[1], [int(x) for x in s[3]])[r] for s in sends])
            if r == 0:
                ev[11].record(st)
            if G > 1:
                c.finish(counts_all, rm, rr, sync=False)
            else:
                c.finish(None, sync=False)
            if r == 0:
                ev[12].record(st)
        torch.cuda.synchronize()
        if it >= warmup:
            pairs = [(0, 1), (1, 2), (3, 4), (5, 6), (7, 8), (9, 10), (11, 12)]
            rows.append([ev[i].elapsed_time(ev[j]) for i, j in pairs])
    med = np.median(np.array(rows), axis=0)
    dev_ms = float(med.sum())
    proj = dev_ms + (EXCHANGE_EST_MS if G > 1 else 0.0)
    for c in ctxs:
        c.close()
    return dev_ms, proj, med, sb[pl] - sb[0]


def main():
    Gs = [int(x) for x in sys.argv[1:]] or [1, 2, 4, 8]
    base = None
    for G in Gs:
        dev_ms, proj, med, w = one(G)
        if G == 1:
            base = dev_ms
        eff = f" projected E({G}) = {base / (G * proj):.2f}" if base and G > 1 else ""
        print(f"G={G}: rank 0 ({w} sequences, {8 // G} shard(s)) device {dev_ms:.3f} ms/step"
              f" (+{EXCHANGE_EST_MS if G > 1 else 0:.3f} ms exchange estimate = {proj:.3f}){eff} | " +
              " ".join(f"{nm}={x:.3f}" for nm, x in zip(NAMES, med)), flush=True)


if __name__ == "__main__":
    main()
