"""f2 across GPUs (SAD_F_TILE_SPLIT): one rank's device share of the centralized rank of config 4
(p = 1: the N x N all-pairs of all 100 000 sequences) at G ranks, measured on ONE GPU as rank 0 of
G (the whole input, rank 0's row blocks of the all-pairs tiles, its K6 rows), the step captured in
one CUDA graph and replayed; plus a stated estimate of the one collective the real rank adds (an
ncclAllReduce of T: N x 8 bytes).

    python tools/f2_share.py [G ...]     (GPU box) -> one line per G
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0901_2742_b200.runtime import Context  # noqa: E402
from synth import gen  # noqa: E402

ALLREDUCE_EST_MS = 0.03     # 800 KB all-reduce over NVLink 5 / NVSwitch (latency + ~2 x 800 KB / 400 GB/s)


def one(G, steps=10, warmup=3, p=1):
    spec = gen.SPECS[4]
    a, o = gen.generate(spec)
    n = len(o) - 1
    dev = torch.device("cuda", 0)
    st = torch.cuda.Stream(dev)
    d_a = torch.from_numpy(a).to(dev)
    d_o = torch.from_numpy(o).to(dev)
    R = int(o[-1])
    ctx = Context(spec.alphabet, spec.k, p, world=G, rank=0, stream=st, tile_split=True)
    for _ in range(warmup):
        ctx.load(d_a, d_o, n, 0, residues=R)
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
    ctx.close()
    return float(np.median(ms)), ap


def main():
    Gs = [int(x) for x in sys.argv[1:]] or [1, 2, 4, 8]
    base = None
    for G in Gs:
        dev_ms, ap = one(G)
        if G == 1:
            base = dev_ms
        proj = dev_ms + (ALLREDUCE_EST_MS if G > 1 else 0.0)
        eff = f" projected E({G}) = {base / (G * proj):.2f}" if base and G > 1 else ""
        print(f"G={G}: rank 0 of the centralized config-4 step (N = 100000, p = 1) graph-replayed {dev_ms:.3f} ms "
              f"(all-pairs kernel {ap:.3f}) + {ALLREDUCE_EST_MS if G > 1 else 0:.3f} ms all-reduce estimate = "
              f"{proj:.3f} ms{eff}", flush=True)


if __name__ == "__main__":
    main()
