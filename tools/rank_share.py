"""One rank's device share of the config-4 step at G GPUs (p = 8 shards, p/G per rank), measured
on ONE GPU as a "virtual rank": a world-1 context over exactly rank 0's slice (the same p/G shards
of w = 12 500 sequences each), its whole step (load .. partition) captured in one CUDA graph and
replayed, so the number is device time without host gaps. Relative to the real rank 0 of a
G-GPU job this runs the same profile, operand and all-pairs work; its partition has p/G buckets
instead of p (a smaller plan, a merge of p/G local runs instead of p received runs). The exchange
steps the real rank adds (not measurable with one GPU) are added as a stated estimate.

    python tools/rank_share.py [G ...]     (GPU box) -> one line per G (config 4, p = 8)
    python tools/rank_share.py --cfg C [--p P | --p-eq-g] [G ...]
        another config; --p-eq-g: p = G buckets at every G (config 3's layout: one shard per GPU),
        projected throughput = the whole job's within-shard pairs / rank 0's step
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


_DATA = {}


def one(G: int, steps: int = 20, warmup: int = 3, cfg: int = 4, p: int = 8):
    spec = gen.SPECS[cfg]
    if cfg not in _DATA:
        _DATA[cfg] = gen.generate(spec)
    a, o = _DATA[cfg]
    n = len(o) - 1
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
    pairs = sum((sb[s + 1] - sb[s]) * (sb[s + 1] - sb[s] - 1) // 2 for s in range(p))   # the whole job's
    return float(np.median(ms)), ap, op, hi - lo, pairs


def main():
    args = sys.argv[1:]
    cfg, p, p_eq_g = 4, 8, False
    if "--cfg" in args:
        i = args.index("--cfg")
        cfg = int(args[i + 1])
        del args[i: i + 2]
    if "--p" in args:
        i = args.index("--p")
        p = int(args[i + 1])
        del args[i: i + 2]
    if "--p-eq-g" in args:
        args.remove("--p-eq-g")
        p_eq_g = True
    Gs = [int(x) for x in args] or [1, 2, 4, 8]
    base = None
    for G in Gs:
        pG = G if p_eq_g else p
        dev_ms, ap, op, w, pairs = one(G, cfg=cfg, p=pG)
        if G == 1:
            base = dev_ms
        proj = dev_ms + (EXCHANGE_EST_MS if G > 1 else 0.0)
        eff = f" projected E({G}) = {base / (G * proj):.2f}" if base and G > 1 and not p_eq_g else ""
        print(f"cfg{cfg} G={G} p={pG}: virtual rank 0 ({w} sequences, {pG // G} shard(s)) graph-replayed step"
              f" {dev_ms:.3f} ms (all-pairs kernel {ap:.3f}, operand stage {op:.3f}; rest {dev_ms - ap - op:.3f})"
              f" + {EXCHANGE_EST_MS if G > 1 else 0:.3f} ms exchange estimate = {proj:.3f} ms;"
              f" projected {pairs / (proj * 1e-3):.3e} pairs/s{eff}", flush=True)


if __name__ == "__main__":
    main()
