"""One rank's device share of the config-4 step at G GPUs (p = 8 shards, p/G per rank), measured
on ONE GPU as a "virtual rank": a world-1 context over exactly rank 0's slice (the same p/G shards
of w = 12 500 sequences each), its whole step (load .. partition) captured in one CUDA graph and
replayed, so the number is device time without host gaps. Relative to the real rank 0 of a
G-GPU job this runs the same profile, operand and all-pairs work; its partition has p/G buckets
instead of p (a smaller plan, a merge of p/G local runs instead of p received runs). The exchange
steps the real rank adds (not measurable with one GPU) are added as a stated estimate.

    python tools/rank_share.py [G ...]     (GPU box) -> one line per G
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0901_2742_b200.runtime import Context  # noqa: E402
from synth import gen  # noqa: E402

# Estimated cost of the exchange steps per step at G > 1: three small ncclAllGathers (ancestor
# records 8 x 16 KB, samples 448 B, counts + status 8 x 160 B) at ~10 us each (NVLink/NVSwitch
# small-message latency), the count read-back + host decision ~20 us, and the all-to-all of
# ~3.5 MB per rank at an effective ~300 GB/s (~12 us) plus ~10 us of launch latency.
EXCHANGE_EST_MS = 0.072


def one(G: int, steps: int = 20, warmup: int = 3):
    spec = gen.SPECS[4]
    a, o = gen.generate(spec)
    n, p = len(o) - 1, 8
    pl = p // G
    sb = gen.shard_bounds(n, p)
    lo, hi = sb[0], sb[pl]
    dev = torch.device("cuda", 0)
    st = torch.cuda.Stream(dev)
    d_a = torch.from_numpy(np.ascontiguousarray(a[o[lo]: o[hi]])).to(dev)
    d_o = torch.from_numpy(np.ascontiguousarray(o[lo: hi + 1] - o[lo])).to(dev)
    R = int(o[hi] - o[lo])
    ctx = Context(spec.alphabet, spec.k, pl, stream=st)
    for _ in range(warmup):
        ctx.load(d_a, d_o, hi - lo, 0, residues=R)
        ctx.run(sync=False)
    torch.cuda.synchronize()
    g = ctx.capture_step(d_a, d_o, R)
    ms = []
    for _ in range(steps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            s.record(st)
            g.replay()
            e.record(st)
        torch.cuda.synchronize()
        ctx.graph_account()
        ms.append(s.elapsed_time(e))
    stt = ctx.stats()
    ap = stt["allpairs_ms_total"] / max(stt["calls"], 1)
    op = stt["operand_ms_total"] / max(stt["calls"], 1)
    ctx.close()
    return float(np.median(ms)), ap, op, hi - lo


def main():
    Gs = [int(x) for x in sys.argv[1:]] or [1, 2, 4, 8]
    base = None
    for G in Gs:
        dev_ms, ap, op, w = one(G)
        if G == 1:
            base = dev_ms
        proj = dev_ms + (EXCHANGE_EST_MS if G > 1 else 0.0)
        eff = f" projected E({G}) = {base / (G * proj):.2f}" if base and G > 1 else ""
        print(f"G={G}: virtual rank 0 ({w} sequences, {8 // G} shard(s)) graph-replayed step {dev_ms:.3f} ms"
              f" (all-pairs kernel {ap:.3f}, operand stage {op:.3f}; rest {dev_ms - ap - op:.3f})"
              f" + {EXCHANGE_EST_MS if G > 1 else 0:.3f} ms exchange estimate = {proj:.3f} ms{eff}", flush=True)


if __name__ == "__main__":
    main()
