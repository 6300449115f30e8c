"""Measured issue rate of tcgen05.mma.cta_group::2.kind::mxf4.block_scale on this B200 (GPU box).

No library fp4 GEMM is reachable from torch here, so the fp4 tensor peak is measured with the
all-pairs kernel itself built MMA-only (-DSAD_TC_DBG_NOTMA -DSAD_TC_DBG_NOEPI: no operand loads,
no epilogue; results are meaningless, only the MMA stream remains): dense ops actually issued
(256 x summed tile N x K padded to 256 x 2) / kernel time, on config 4 (p = 8; ~1.3 ms of MMAs
per launch). Prints one JSON object.

    SAD_LIB_PATH=ab/libsad_mma.so python tools/mma_peak.py
"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0901_2742_b200.runtime import Context  # noqa: E402
from synth import gen  # noqa: E402

BM, BN = 256, 240


def tile_cols(w):
    """Summed MMA N over a shard's tiles (the last column block runs with N = its real columns
    rounded up to 16)."""
    nI, nJ = (w + BM - 1) // BM, (w + BN - 1) // BN
    nlast = (w - (nJ - 1) * BN + 15) // 16 * 16
    t = 0
    for I in range(nI):
        need = BM * I - (BN - 1)
        jmin = 0 if need <= 0 else (need + BN - 1) // BN
        if jmin < nJ:
            t += (nJ - 1 - jmin) * BN + nlast
    return t


def run(a, o, p, steps=5):
    n = len(o) - 1
    dev = torch.device("cuda", 0)
    d_a, d_o = torch.from_numpy(a).to(dev), torch.from_numpy(o).to(dev)
    ctx = Context("protein", 3, p, kernel="tc")
    for _ in range(2):
        ctx.load(d_a, d_o, n, 0, residues=int(o[-1]))
        ctx.run(sync=True)
    ctx.reset_stats()
    for _ in range(steps):
        ctx.load(d_a, d_o, n, 0, residues=int(o[-1]))
        ctx.run(sync=True)
    st = ctx.stats()
    ms = st["allpairs_ms_total"] / max(st["calls"], 1)
    _, _, kcols = ctx.profile_info()
    sb = gen.shard_bounds(n, p)
    hw = sum(tile_cols(int(sb[s + 1] - sb[s])) * BM * ((int(kcols[s]) + 255) // 256 * 256) * 2 for s in range(p))
    return ms, hw / (ms / 1e3) / 1e12


def main():
    a, o = gen.generate(gen.SPECS[4])
    ms8, tops8 = run(a, o, 8)
    print(json.dumps({"fp4_mma_tops": tops8, "p8_kernel_ms": ms8, "lib": os.environ.get("SAD_LIB_PATH", ""),
                      "how": "all-pairs kernel built MMA-only (no TMA, no epilogue): issued dense ops of "
                             "tcgen05.mma.cta_group::2.kind::mxf4 (256x240 tiles, K padded to 256) / kernel time"}))


if __name__ == "__main__":
    main()
