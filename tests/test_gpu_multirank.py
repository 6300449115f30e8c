"""G ranks emulated in ONE process on one GPU: the device path of world > 1 (per-rank
shards, sad_pack, the receive-side rank-merge of sad_finish) with the collectives done
by host-driven copies between the ranks' torch buffers (no kernel waits on another rank).
The output must be byte-identical to world = 1 and to the oracle (SURVEY T4 G-invariance)."""
import numpy as np
import pytest
import torch

import oracle
from synth import gen

pytestmark = pytest.mark.gpu


def run_emulated(a, o, alpha, k, p, G, kernel, rank_mode="ga"):
    from paper_0901_2742_b200.runtime import Context
    n = len(o) - 1
    sb = gen.shard_bounds(n, p)
    pl = p // G
    ctxs = [Context(alpha, k, p, world=G, rank=r, kernel=kernel, rank_mode=rank_mode) for r in range(G)]
    for r, c in enumerate(ctxs):
        lo, hi = sb[r * pl], sb[(r + 1) * pl]
        c.load(a[o[lo]: o[hi]], o[lo: hi + 1] - o[lo], n, lo)
        c.build_profiles()
    anc_all = torch.cat([c.rank_local() for c in ctxs])              # all-gather, rank order
    smp_all = torch.cat([c.rank_global(anc_all) for c in ctxs])
    counts_all = torch.cat([c.partition_plan(smp_all) for c in ctxs]).cpu().numpy().reshape(p, p, 2)
    sends = [c.pack(counts_all) for c in ctxs]
    out = []
    for r, c in enumerate(ctxs):                                      # all_to_all_v
        rm = torch.cat([torch.split(s[0], [int(x) for x in s[2]])[r] for s in sends])
        rr = torch.cat([torch.split(s[1], [int(x) for x in s[3]])[r] for s in sends])
        sizes = c.finish(counts_all, rm, rr)
        out.append(c)
    return ctxs, sizes


@pytest.mark.parametrize("kernel", ["tc", "tc1", "alu"])
@pytest.mark.parametrize("G", [2, 4, 8])
def test_g_invariance(kernel, G):
    spec = gen.SPECS[3]
    a, o = gen.generate(spec, n=1600)
    p = 8
    r = oracle.run(a, o, spec.alphabet, spec.k, p)
    ctxs, sizes = run_emulated(a, o, spec.alphabet, spec.k, p, G, kernel)
    assert sizes.tolist() == r.bsize.tolist()
    seqs = gen.to_strings(a, o)
    pl = p // G
    for rank, c in enumerate(ctxs):
        loc, ga = c.ancestors()
        assert loc.tolist() == r.anc.tolist() and ga == r.ga
        assert [int(x) & 0x7FFFFFFF for x in c.pivots()] == r.pivots.tolist()
        for b in range(rank * pl, (rank + 1) * pl):
            idx, key, res, off = c.bucket(b)
            assert idx.tolist() == r.buckets()[b]
            assert [bytes(res[off[i]: off[i + 1]]).decode() for i in range(len(idx))] == [seqs[i] for i in idx]


@pytest.mark.parametrize("G", [2, 4])
def test_g_invariance_samples_mode(G):
    """SURVEY §8(f) f1 across emulated ranks: the rank-sample records are all-gathered like the
    ancestor records; buckets identical to the oracle's mode "samples"."""
    spec = gen.SPECS[2]
    a, o = gen.generate(spec)
    p = spec.p
    ctxs, _ = run_emulated(a, o, spec.alphabet, spec.k, p, G, "tc", rank_mode="samples")
    r = oracle.run(a, o, spec.alphabet, spec.k, p, mode="samples")
    pl = p // G
    for rk, c in enumerate(ctxs):
        for b in range(rk * pl, (rk + 1) * pl):
            assert c.bucket(b)[0].tolist() == r.buckets()[b]

