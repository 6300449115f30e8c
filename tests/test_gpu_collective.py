"""The collective API (include/sad.h: sad_rank / sad_partition) on the GPU: the step without host
synchronization, its CUDA-graph capture, the library's own NCCL communicator (a single-rank
communicator: the exchange steps, pack, grouped ncclSend/ncclRecv and the receive-side merge all
run through NCCL), the operand-capacity replan, sad_abort, and device-detected input errors
reported at the step's first synchronizing call. Every result is compared with the oracle.
"""
import numpy as np
import pytest
import torch

import oracle
from synth import gen

pytestmark = pytest.mark.gpu


def _full_compare(ctx, a, o, p, r):
    n = len(o) - 1
    sb = gen.shard_bounds(n, p)
    T = np.concatenate([ctx.local_rank(s) for s in range(p)])
    assert np.array_equal(T, r.T)
    loc, ga = ctx.ancestors()
    assert loc.tolist() == r.anc.tolist() and ga == r.ga
    assert np.array_equal(np.concatenate([ctx.sorted(s) for s in range(p)]), r.sorted)
    assert [int(x) & 0x7FFFFFFF for x in ctx.pivots()] == r.pivots.tolist()
    seqs = gen.to_strings(a, o)
    for b, want in enumerate(r.buckets()):
        idx, key, res, off = ctx.bucket(b)
        assert idx.tolist() == want
        assert [bytes(res[off[i]: off[i + 1]]).decode() for i in range(len(idx))] == [seqs[i] for i in want]
    assert sb[-1] == n


@pytest.mark.parametrize("kernel", ["tc", "tc8", "alu"])
@pytest.mark.parametrize("cfg", [1, 2])
def test_single_rank_nccl_communicator(cfg, kernel):
    """sad_create with an NCCL id at world == 1: the all-gathers, the count exchange (status tail,
    one wait) and the all-to-all (pack, ncclSend/ncclRecv to itself, merge of received runs)."""
    from paper_0901_2742_b200.runtime import Context
    spec = gen.SPECS[cfg]
    a, o = gen.generate(cfg)
    n = len(o) - 1
    ctx = Context(spec.alphabet, spec.k, spec.p, kernel=kernel, comm=True)
    ctx.load(a, o, n, 0)
    sizes = ctx.run()
    r = oracle.run(a, o, spec.alphabet, spec.k, spec.p)
    assert sizes.tolist() == r.bsize.tolist()
    _full_compare(ctx, a, o, spec.p, r)
    # a second step on the same context (buffers, capacity and communicator reused)
    ctx.load(a, o, n, 0)
    assert ctx.run().tolist() == r.bsize.tolist()
    _full_compare(ctx, a, o, spec.p, r)
    ctx.close()


@pytest.mark.parametrize("kernel", ["tc", "alu"])
@pytest.mark.parametrize("cfg", [2, 4])
def test_graph_captured_step(cfg, kernel):
    """load (device inputs) .. sad_partition captured into ONE CUDA graph and replayed: identical
    buckets; the captured stage events give the all-pairs kernel time per replay."""
    from paper_0901_2742_b200.runtime import Context
    spec = gen.SPECS[cfg]
    p = 8 if cfg == 4 else spec.p
    a, o = gen.generate(cfg)
    n = len(o) - 1
    stream = torch.cuda.Stream()
    ctx = Context(spec.alphabet, spec.k, p, kernel=kernel, stream=stream)
    d_a, d_o = torch.from_numpy(a).cuda(), torch.from_numpy(o).cuda()
    R = int(o[-1])
    for _ in range(2):                      # eager steps: buffers and the operand capacity settle
        ctx.load(d_a, d_o, n, 0, residues=R)
        ctx.run(sync=False)
    torch.cuda.synchronize()
    g = ctx.capture_step(d_a, d_o, R)
    ctx.reset_stats()
    for _ in range(3):
        with torch.cuda.stream(stream):
            g.replay()
        torch.cuda.synchronize()
        ctx.graph_account()
    st = ctx.stats()
    assert st["calls"] == 3 and st["allpairs_ms_total"] > 0
    keys = ctx.out_keys().cpu().numpy().view(np.uint64)
    if cfg == 2:
        r = oracle.run(a, o, spec.alphabet, spec.k, p)
        assert ctx.bucket_sizes_now().tolist() == r.bsize.tolist()
        _full_compare(ctx, a, o, p, r)
    else:
        import hashlib
        import json
        import os
        path = os.path.join(os.path.dirname(__file__), "golden", "full", "cfg4_p8.json")
        if not os.path.exists(path):
            pytest.skip("config 4 golden not written yet (tests/make_goldens.py)")
        g4 = json.load(open(path))
        assert ctx.bucket_sizes_now().tolist() == g4["bsize"]
        for b in range(p):
            idx = ctx.bucket(b)[0]
            assert hashlib.sha256(np.ascontiguousarray(idx, "<i8").tobytes()).hexdigest() == g4["buckets"][b]["order"]
    assert np.all(keys[1:] > keys[:-1])
    ctx.close()


@pytest.mark.parametrize("kernel", ["tc", "tcfull", "tc8"])
def test_operand_capacity_replan(kernel):
    """DNA k = 2 (A^k = 16): poly-A runs push K = sum_tau M(tau) far above the initial capacity of
    8 A^k columns (no layer cap fits: the excess beyond T = 8 exceeds a byte), so the first step
    overflows, the collective call returns SAD_E_REPLAN and the runtime reruns it; the split API
    returns it from sad_rank_local. Results stay bit-identical to the oracle."""
    from paper_0901_2742_b200 import SadError
    from paper_0901_2742_b200.runtime import Context
    rng = np.random.default_rng(3)
    seqs = ["A" * 900, "A" * 400 + "C" * 300, "ACGT" * 50] + [
        "".join(rng.choice(list("ACGT"), int(rng.integers(20, 300)))) for _ in range(61)]
    a, o = gen.from_strings(seqs)
    n = len(o) - 1
    for p in (1, 2):
        r = oracle.run(a, o, "dna", 2, p)
        ctx = Context("dna", 2, p, kernel=kernel)
        ctx.load(a, o, n, 0)
        sizes = ctx.run()                     # replans internally
        assert sizes.tolist() == r.bsize.tolist()
        _full_compare(ctx, a, o, p, r)
        ctx.close()
        # split API: the overflow surfaces at sad_rank_local of a fresh context
        ctx = Context("dna", 2, p, kernel=kernel)
        ctx.load(a, o, n, 0)
        ctx.build_profiles()
        with pytest.raises(SadError) as e:
            ctx.rank_local()
        assert e.value.name == "SAD_E_REPLAN"
        ctx.build_profiles()
        anc = ctx.rank_local()                # the grown capacity fits
        smp = ctx.rank_global(anc)
        ctx.partition_plan(smp[: p * (p - 1)] if p > 1 else smp)
        assert ctx.finish(None).tolist() == r.bsize.tolist()
        ctx.close()


def test_abort_and_errors():
    from paper_0901_2742_b200 import SadError
    from paper_0901_2742_b200.runtime import Context
    spec = gen.SPECS[1]
    a, o = gen.generate(1)
    ctx = Context(spec.alphabet, spec.k, spec.p, comm=True)
    ctx.load(a, o, len(o) - 1, 0)
    ctx._call("sad_abort")
    with pytest.raises(SadError) as e:
        ctx.run()
    assert e.value.name == "SAD_E_STATE"
    # an illegal symbol is found by K1 and reported at the step's first synchronizing call
    bad = gen.to_strings(a, o)
    bad[37] = bad[37][:10] + "B" + bad[37][11:]
    a2, o2 = gen.from_strings(bad)
    ctx = Context(spec.alphabet, spec.k, spec.p, comm=True)
    ctx.load(a2, o2, len(o2) - 1, 0)
    with pytest.raises(SadError) as e:
        ctx.run()
    assert e.value.name == "SAD_E_SYMBOL" and e.value.location == (37, 10)


@pytest.mark.parametrize("kernel", ["tc", "tc1", "tc8"])
@pytest.mark.parametrize("case", [("cfg2", 1, 3), ("cfg2", 8, 4), ("cfg3s", 1, 8), ("excess", 2, 3)])
def test_tile_split_emulated(kernel, case):
    """SAD_F_TILE_SPLIT (SURVEY §8(f) f2 across GPUs): G contexts, each with the whole input, every
    one computing only its row blocks' tiles (and their K6 excess rows), no communicator: their
    partial T summed on the host equals the oracle's T element by element (every tile exactly once,
    the excess of every computed pair present)."""
    from paper_0901_2742_b200.runtime import Context
    name, p, G = case
    if name == "cfg2":
        spec = gen.SPECS[2]
        a, o = gen.generate(spec)
        alpha, k = spec.alphabet, spec.k
    elif name == "cfg3s":
        spec = gen.SPECS[3]
        a, o = gen.generate(spec, n=3000, seed=41)
        alpha, k = spec.alphabet, spec.k
    else:                                   # repeats: shards with layer caps and K6 excess rows
        rng = np.random.default_rng(43)
        al = list("ACDEFGHIKLMNPQRSTVWY")
        seqs = ["".join(rng.choice(al, int(rng.integers(40, 400)))) + "".join(rng.choice(al, 4)) * int(rng.integers(1, 9))
                for _ in range(1500)]
        a, o = gen.from_strings(seqs)
        alpha, k = "protein", 3
    n = len(o) - 1
    r = oracle.run(a, o, alpha, k, p)
    T = np.zeros(n, np.uint64)
    for rank in range(G):
        ctx = Context(alpha, k, p, world=G, rank=rank, kernel=kernel, tile_split=True)
        ctx.load(a, o, n, 0)
        ctx.run()
        T += np.concatenate([ctx.local_rank(s) for s in range(p)])
        ctx.close()
    assert np.array_equal(T, r.T)


@pytest.mark.parametrize("p", [1, 8])
def test_tile_split_single_rank_reduce(p):
    """Tile split with a (single-rank) NCCL communicator: the ncclAllReduce of T runs inside
    sad_rank right after the all-pairs kernel; the whole step then matches the oracle."""
    from paper_0901_2742_b200.runtime import Context
    spec = gen.SPECS[2]
    a, o = gen.generate(spec)
    n = len(o) - 1
    ctx = Context(spec.alphabet, spec.k, p, world=1, rank=0, tile_split=True, comm=True)
    ctx.load(a, o, n, 0)
    sizes = ctx.run()
    r = oracle.run(a, o, spec.alphabet, spec.k, p)
    assert sizes.tolist() == r.bsize.tolist()
    _full_compare(ctx, a, o, p, r)
    ctx.close()
