"""GPU path (libsad.so through the C ABI) vs the CPU oracle, bit for bit.

All arithmetic on the path is integer, so every comparison is
exact: T_i, local ancestors, GA, S_i/den_i, keys, local sort order, samples,
pivots, bucket membership and order, and the redistributed residues.
"""
import numpy as np
import pytest

import oracle
from synth import gen

pytestmark = pytest.mark.gpu

def _kernels():
    # the tensor-core kernel is mandatory once built (tc_supported() in k_allpairs_tc.cu)
    import os
    return ["tc", "tc1", "tc8", "tc81", "tcfull", "tc8full", "alu"] if os.environ.get("SAD_TEST_TC", "1") == "1" else ["alu"]


KERNELS = _kernels()


def _ctx(alpha, k, p, kernel, keep_sim=False):
    from paper_0901_2742_b200.runtime import Context
    return Context(alpha, k, p, kernel=kernel, keep_sim=keep_sim)


def _run_gpu(a, o, alpha, k, p, kernel, keep_sim=False):
    ctx = _ctx(alpha, k, p, kernel, keep_sim)
    n = len(o) - 1
    ctx.load(a, o, n, 0)
    sizes = ctx.run()
    return ctx, sizes


def _compare_full(ctx, sizes, r, a, o, p):
    n = len(o) - 1
    sb = gen.shard_bounds(n, p)
    # T per shard (O4)
    T = np.concatenate([ctx.local_rank(s) for s in range(p)])
    assert np.array_equal(T, r.T), "T_i differs"
    # ancestors and GA (O5, O6)
    loc, ga = ctx.ancestors()
    assert loc.tolist() == r.anc.tolist()
    assert ga == r.ga
    # ranks vs GA (O7) and keys
    S = np.concatenate([ctx.ranks(s)[0] for s in range(p)]).astype(np.int64)
    D = np.concatenate([ctx.ranks(s)[1] for s in range(p)]).astype(np.int64)
    K = np.concatenate([ctx.ranks(s)[2] for s in range(p)])
    assert np.array_equal(S, r.S) and np.array_equal(D, r.den)
    q = np.array([oracle.q(int(s), int(d)) for s, d in zip(r.S, r.den)], dtype=object)
    assert [int(x) for x in K] == [(int(qq) << 31) + i for i, qq in enumerate(q)]
    # local sort (O8)
    srt = np.concatenate([ctx.sorted(s) for s in range(p)])
    assert np.array_equal(srt, r.sorted)
    # pivots (O9): keys of the oracle's pivot sequences
    piv = ctx.pivots()
    assert [int(x) & 0x7FFFFFFF for x in piv] == r.pivots.tolist()
    # buckets (O10, O11)
    assert sizes.tolist() == r.bsize.tolist()
    seqs = gen.to_strings(a, o)
    for b, ref in enumerate(r.buckets()):
        idx, key, res, off = ctx.bucket(b)
        assert idx.tolist() == ref
        got = [bytes(res[off[i]: off[i + 1]]).decode() for i in range(len(idx))]
        assert got == [seqs[i] for i in ref]
    assert sb[-1] == n


@pytest.mark.parametrize("kernel", KERNELS)
def test_fixed_point_selftest(kernel):
    if kernel != "alu":
        pytest.skip("self-test is kernel independent")
    ctx = _ctx("protein", 3, 1, kernel)
    assert ctx.selftest_fixed_point(65535) == 0


@pytest.mark.parametrize("kernel", KERNELS)
def test_worked_example(kernel):
    seqs = ["ACGTAC", "ACGTTT", "CGTAAA", "TTTTGG", "ACGG", "TTTGGA"]
    a, o = gen.from_strings(seqs)
    ctx, sizes = _run_gpu(a, o, "dna", 2, 2, kernel)
    r = oracle.run(a, o, "dna", 2, 2)
    _compare_full(ctx, sizes, r, a, o, 2)
    assert [ctx.bucket(b)[0].tolist() for b in range(2)] == [[3], [5, 1, 2, 4, 0]]


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("cfg", [1, 2])
def test_configs_1_2_full(kernel, cfg):
    spec = gen.SPECS[cfg]
    a, o = gen.generate(cfg)
    ctx, sizes = _run_gpu(a, o, spec.alphabet, spec.k, spec.p, kernel, keep_sim=(cfg == 1))
    r = oracle.run(a, o, spec.alphabet, spec.k, spec.p)
    _compare_full(ctx, sizes, r, a, o, spec.p)
    if cfg == 1:      # full similarity matrices of config 1
        n = len(o) - 1
        sb = gen.shard_bounds(n, spec.p)
        for s in range(spec.p):
            Sm = ctx.similarity(s)
            ii, jj = np.meshgrid(np.arange(sb[s], sb[s + 1]), np.arange(sb[s], sb[s + 1]), indexing="ij")
            Sref, _ = oracle.pairs_S(a, o, spec.k, ii.ravel(), jj.ravel())
            assert np.array_equal(Sm.ravel().astype(np.int64), Sref)


@pytest.mark.parametrize("kernel", KERNELS)
@pytest.mark.parametrize("case", ["cfg3_small", "cfg4_small", "cfg5_small_p1", "cfg5_small_p4", "ragged_p3"])
def test_scaled_configs(kernel, case):
    """Oracle-sized versions of configs 3-5 (same recipe, fewer sequences) that still span
    several 128-row tiles, ragged shard tails and p not dividing N."""
    if case == "cfg3_small":
        spec, n, p = gen.SPECS[3], 1500, 8
    elif case == "cfg4_small":
        spec, n, p = gen.SPECS[4], 2100, 8
    elif case == "cfg5_small_p1":
        spec, n, p = gen.SPECS[5], 700, 1
    elif case == "cfg5_small_p4":
        spec, n, p = gen.SPECS[5], 903, 4
    else:
        spec, n, p = gen.SPECS[2], 1001, 3
    a, o = gen.generate(spec, n=n)
    ctx, sizes = _run_gpu(a, o, spec.alphabet, spec.k, p, kernel)
    r = oracle.run(a, o, spec.alphabet, spec.k, p)
    _compare_full(ctx, sizes, r, a, o, p)


@pytest.mark.parametrize("kernel", KERNELS)
def test_adversarial(kernel):
    """poly-A (counts far above any cap, K columns grow), L == k, identical sequences (all
    rank ties -> index order), containment (F = 1 without identity), w = p."""
    rng = np.random.default_rng(5)
    seqs = ["A" * 3000, "A" * 3, "ACD", "W" * 700, "AAAAAAAAAC", "AAC", "MMMMMMMMMMMMMM"]
    seqs += ["ACDEFGHIK" * 10] * 9
    seqs += ["".join(rng.choice(list("ACDEFGHIKLMNPQRSTVWY"), int(rng.integers(3, 400)))) for _ in range(200)]
    a, o = gen.from_strings(seqs)
    for p in (1, 4):
        ctx, sizes = _run_gpu(a, o, "protein", 3, p, kernel)
        r = oracle.run(a, o, "protein", 3, p)
        _compare_full(ctx, sizes, r, a, o, p)
    same = ["ACDEFGHIKL"] * 16                                    # w == p == 4
    a, o = gen.from_strings(same)
    ctx, sizes = _run_gpu(a, o, "protein", 3, 4, kernel)
    r = oracle.run(a, o, "protein", 3, 4)
    _compare_full(ctx, sizes, r, a, o, 4)


@pytest.mark.parametrize("kernel", KERNELS)
def test_excess_path(kernel):
    """The capped layers + sparse excess: rows whose per-row excess
    sum_tau (n - T)+ sits just below / above the 255 byte bound of each cap T in {1,2,4,8}
    (periodic sequences), pairs whose excess is ~200, shards with and without excess, list
    lengths above a warp, and a ragged tail across several 256 x 240 tiles."""
    rng = np.random.default_rng(11)
    alpha = list("ACDEFGHIKLMNPQRSTVWY")
    seqs = []
    for _ in range(40):                                         # ~10 3-mers x 21 repeats: excess 200 at T=1
        seqs.append("ACDEFGHIKL" * 21 + "".join(rng.choice(alpha, int(rng.integers(0, 30)))))
    seqs += ["ACDEFG" * 50, "MNPQRS" * 43, "ACDEFGHIKLMN" * 23]  # excess > 255 at T=1 (T=2, 4, 8 or none)
    for _ in range(560):                                        # families with shared repeats
        base = "".join(rng.choice(alpha, int(rng.integers(40, 500))))
        rep = "".join(rng.choice(alpha, 4)) * int(rng.integers(1, 12))
        cut = int(rng.integers(0, len(base)))
        seqs.append(base[:cut] + rep + base[cut:])
    order = rng.permutation(len(seqs))
    seqs = [seqs[i] for i in order]
    a, o = gen.from_strings(seqs)
    for p in (1, 3):
        ctx, sizes = _run_gpu(a, o, "protein", 3, p, kernel)
        r = oracle.run(a, o, "protein", 3, p)
        _compare_full(ctx, sizes, r, a, o, p)
    # one shard with a row far above every cap next to shards with none
    seqs2 = ["A" * 5000] + ["".join(rng.choice(alpha, int(rng.integers(50, 300)))) for _ in range(299)]
    a, o = gen.from_strings(seqs2)
    ctx, sizes = _run_gpu(a, o, "protein", 3, 3, kernel)
    r = oracle.run(a, o, "protein", 3, 3)
    _compare_full(ctx, sizes, r, a, o, 3)


def test_errors():
    from paper_0901_2742_b200 import SadError
    a, o = gen.from_strings(["ACDE", "ACDX", "ACDE", "ACDE"])
    ctx = _ctx("protein", 3, 1, "alu")
    ctx.load(a, o, 4, 0)
    with pytest.raises(SadError) as e:
        ctx.run()
    assert e.value.name == "SAD_E_SYMBOL" and e.value.location == (1, 3)
    a, o = gen.from_strings(["ACDE", "AC", "ACDE", "ACDE"])
    ctx = _ctx("protein", 3, 1, "alu")
    ctx.load(a, o, 4, 0)
    with pytest.raises(SadError) as e:
        ctx.run()
    assert e.value.name == "SAD_E_TOO_SHORT" and e.value.location[0] == 1
    a, o = gen.from_strings(["ACDE"] * 5)
    ctx = _ctx("protein", 3, 3, "alu")
    with pytest.raises(SadError) as e:
        ctx.load(a, o, 5, 0)
    assert e.value.name == "SAD_E_INSUFFICIENT"


def test_errors_long_sequences():
    """The same locations through the block-per-sequence K1/K2 (average L >= 1024): the first bad
    symbol (smallest index, then smallest position, also in a later staged segment), a too-short
    sequence among long ones, and L - k + 1 > 65 535."""
    from paper_0901_2742_b200 import SadError
    rng = np.random.default_rng(5)
    seqs = ["".join(rng.choice(list("ACGT"), int(rng.integers(3000, 12000)))) for _ in range(12)]
    bad = list(seqs)
    x = list(bad[7]); x[9000 % len(x)] = "N"; x[100] = "A"; bad[7] = "".join(x)
    y = list(bad[3]); pos = len(y) - 2; y[pos] = "J"; bad[3] = "".join(y)       # smaller index wins
    a, o = gen.from_strings(bad)
    ctx = _ctx("dna", 6, 2, "tc")
    ctx.load(a, o, len(bad), 0)
    with pytest.raises(SadError) as e:
        ctx.run()
    assert e.value.name == "SAD_E_SYMBOL" and e.value.location == (3, pos)
    short = list(seqs); short[5] = "ACG"
    a, o = gen.from_strings(short)
    ctx = _ctx("dna", 6, 2, "tc")
    ctx.load(a, o, len(short), 0)
    with pytest.raises(SadError) as e:
        ctx.run()
    assert e.value.name == "SAD_E_TOO_SHORT" and e.value.location[0] == 5
    longs = list(seqs); longs[9] = "".join(rng.choice(list("ACGT"), 65535 + 6))  # Tw = 65 536
    a, o = gen.from_strings(longs)
    ctx = _ctx("dna", 6, 2, "tc")
    ctx.load(a, o, len(longs), 0)
    with pytest.raises(SadError) as e:
        ctx.run()
    assert e.value.name == "SAD_E_TOO_LONG" and e.value.location[0] == 9
    # and the largest legal length (Tw = 65 535: eight staged segments) against the oracle
    ok = list(seqs); ok[9] = longs[9][:-1]
    a, o = gen.from_strings(ok)
    ctx, sizes = _run_gpu(a, o, "dna", 6, 2, "tc")
    _compare_full(ctx, sizes, oracle.run(a, o, "dna", 6, 2), a, o, 2)


@pytest.mark.parametrize("kernel", KERNELS[:1])
@pytest.mark.parametrize("cfg", [4, 5])
def test_full_size_sampled(kernel, cfg):
    """BASELINE sizes in the bench's launch configuration (config 4: N = 100k, p = 8 on one
    GPU; config 5: N = 10k DNA, p = 1): sampled T rows and GA ranks against the oracle one
    by one, and the properties that hold at any size."""
    spec = gen.SPECS[cfg]
    p = spec.p
    a, o = gen.generate(cfg)
    n = len(o) - 1
    ctx, sizes = _run_gpu(a, o, spec.alphabet, spec.k, p, kernel)
    sb = gen.shard_bounds(n, p)
    rng = np.random.default_rng(cfg)
    T = np.concatenate([ctx.local_rank(s) for s in range(p)])
    rows = np.concatenate([rng.choice(np.arange(sb[s], sb[s + 1]), 6, replace=False) for s in range(p)])
    assert np.array_equal(oracle.rows_T(a, o, spec.k, p, rows), T[rows])
    loc, ga = ctx.ancestors()
    for s in range(p):                                           # a_s = argmax T (ties -> smaller index)
        seg = T[sb[s]: sb[s + 1]]
        assert loc[s] == sb[s] + int(np.flatnonzero(seg == seg.max())[0])
    assert ga in loc.tolist()
    S = np.concatenate([ctx.ranks(s)[0] for s in range(p)]).astype(np.int64)
    D = np.concatenate([ctx.ranks(s)[1] for s in range(p)]).astype(np.int64)
    K = np.concatenate([ctx.ranks(s)[2] for s in range(p)])
    samp = rng.choice(n, 400, replace=False)
    Sref, Dref = oracle.pairs_S(a, o, spec.k, samp, np.full(len(samp), ga))
    assert np.array_equal(S[samp], Sref) and np.array_equal(D[samp], Dref)
    assert all(int(K[i]) == (oracle.q(int(S[i]), int(D[i])) << 31) + int(i) for i in samp)
    # buckets: a permutation, each in key order, bucket ranges increasing, <= 2w + p
    assert int(sizes.sum()) == n and int(sizes.max()) <= 2 * (n // p) + p
    keys = ctx.out_keys().cpu().numpy().view(np.uint64)
    assert np.all(keys[1:] > keys[:-1])
    assert np.array_equal(np.sort((keys & np.uint64(0x7FFFFFFF)).astype(np.int64)), np.arange(n))
    assert np.array_equal(np.sort(K), keys)
    piv = ctx.pivots()
    first = np.concatenate([[0], np.cumsum(sizes)])
    for b in range(p - 1):
        if sizes[b]:
            assert keys[first[b + 1] - 1] <= piv[b]
        if first[b + 1] < n:
            assert keys[first[b + 1]] > piv[b]


@pytest.mark.parametrize("kernel", ["tc", "alu"])
@pytest.mark.parametrize("cfg", [1, 2])
def test_bucket_distance_matrices(kernel, cfg):
    """SURVEY §8(f) f3 (SPEC S:347 build_distance_matrix): after the redistribution, every bucket's
    distance matrix d = 1 - S/den on the GPU equals the oracle: S exact (integers), d bit-exact to
    the same IEEE float32 arithmetic (fdiv then fsub) and within 2^-23 of the fp64 value."""
    spec = gen.SPECS[cfg]
    a, o = gen.generate(cfg)
    ctx, sizes = _run_gpu(a, o, spec.alphabet, spec.k, spec.p, kernel)
    for b in range(spec.p):
        idx = ctx.bucket(b)[0]
        if len(idx) == 0:
            continue
        D, S = ctx.bucket_distances(b)
        ii, jj = np.meshgrid(idx, idx, indexing="ij")
        Sref, dref = oracle.pairs_S(a, o, spec.k, ii.ravel(), jj.ravel())
        assert np.array_equal(S.ravel().astype(np.int64), Sref)
        Dg = D.cpu().numpy().ravel()
        d32 = np.float32(1) - np.float32(Sref) / np.float32(dref)
        d32[np.flatnonzero(ii.ravel() == jj.ravel())] = 0
        assert np.array_equal(Dg, d32)
        d64 = 1.0 - Sref / dref
        d64[ii.ravel() == jj.ravel()] = 0
        assert np.max(np.abs(Dg - d64)) <= 2.0 ** -23
        assert np.array_equal(D.cpu().numpy(), D.cpu().numpy().T)


def _compare_f1(ctx, sizes, r, a, o, p):
    """rank against the k*p samples: keys, local order, PSRS pivots, buckets."""
    n = len(o) - 1
    T = np.concatenate([ctx.local_rank(s) for s in range(p)])
    assert np.array_equal(T, r.T)
    loc, ga = ctx.ancestors()
    assert ga == -1 and loc.tolist() == r.anc.tolist()
    # reading A27: key = (T' << index bits) + index, T' the exact sum of q over the samples
    ib = ctx.key_index_bits
    assert ib == max(1, int(n - 1).bit_length())
    K = np.concatenate([ctx.ranks(s)[2] for s in range(p)])
    assert [int(x) for x in K] == [(int(t) << ib) + i for i, t in enumerate(r.S)]
    S_lo = np.concatenate([ctx.ranks(s)[0] for s in range(p)]).astype(np.int64)
    S_hi = np.concatenate([ctx.ranks(s)[1] for s in range(p)]).astype(np.int64)
    assert ((S_hi << 32) + S_lo).tolist() == [int(t) for t in r.S]
    assert np.array_equal(np.concatenate([ctx.sorted(s) for s in range(p)]), r.sorted)
    assert ctx.key_index(ctx.pivots()).tolist() == r.pivots.tolist()
    assert sizes.tolist() == r.bsize.tolist()
    for b, ref in enumerate(r.buckets()):
        assert ctx.bucket(b)[0].tolist() == ref
    assert int(sizes.sum()) == n


@pytest.mark.parametrize("kernel", ["tc", "tc1", "tc+cc", "tc8", "alu"])
@pytest.mark.parametrize("case", ["cfg1", "cfg2", "cfg3_small_p4", "dna_p3", "adv", "p12"])
def test_samples_mode(kernel, case):
    """the GPU path in rank-against-samples mode is bit-identical
    to the oracle's mode "samples" -- the fp4 kernels with the rank on the tensor cores (tc, tc1),
    or on the CUDA cores (tc+cc, and the int8 / ALU kernels). p = 12: 132 samples (the f1 tile's
    N = 144), shards with and without layer caps."""
    from paper_0901_2742_b200.runtime import Context
    if case in ("cfg1", "cfg2"):
        spec = gen.SPECS[int(case[3])]
        a, o = gen.generate(spec)
        alpha, k, p = spec.alphabet, spec.k, spec.p
    elif case == "cfg3_small_p4":
        spec = gen.SPECS[3]
        a, o = gen.generate(spec, n=3000, seed=17)
        alpha, k, p = spec.alphabet, spec.k, 4
    elif case == "dna_p3":
        spec = gen.SPECS[5]
        a, o = gen.generate(spec, n=600, seed=5)
        alpha, k, p = spec.alphabet, spec.k, 3
    else:   # k-mer counts above 255 on both sides of a (sequence, sample) pair: the exact fix-up
        rng = np.random.default_rng(23)
        seqs = ["A" * int(rng.integers(300, 3000)) for _ in range(12)] + ["A" * 40 + "C" * 400] * 3
        seqs += ["".join(rng.choice(list("ACDEFGHIKLMNPQRSTVWY"), int(rng.integers(20, 300)))) for _ in range(45)]
        seqs = [seqs[i] for i in rng.permutation(len(seqs))]
        a, o = gen.from_strings(seqs)
        alpha, k, p = "protein", 3, 3
    if case == "p12":
        spec = gen.SPECS[3]
        a, o = gen.generate(spec, n=2000, seed=29)
        alpha, k, p = spec.alphabet, spec.k, 12
    n = len(o) - 1
    cc = kernel == "tc+cc"
    ctx = Context(alpha, k, p, kernel="tc" if cc else kernel, rank_mode="samples", f1_cuda_cores=cc)
    ctx.load(a, o, n, 0)
    sizes = ctx.run()
    r = oracle.run(a, o, alpha, k, p, mode="samples")
    _compare_f1(ctx, sizes, r, a, o, p)


def test_centralized_full_size_sampled():
    """the centralized rank (one shard of all N = 100 000 sequences of config 4,
    the 5 x 10^9-pair all-pairs on the tensor cores): sampled T_i against the oracle row by row,
    and the properties that hold at any size."""
    spec = gen.SPECS[4]
    a, o = gen.generate(spec)
    n = len(o) - 1
    ctx, sizes = _run_gpu(a, o, spec.alphabet, spec.k, 1, "tc")
    T = ctx.local_rank(0)
    rows = np.random.default_rng(44).choice(n, 12, replace=False)
    assert np.array_equal(oracle.rows_T(a, o, spec.k, 1, rows), T[rows])
    assert sizes.tolist() == [n]
    keys = ctx.out_keys().cpu().numpy().view(np.uint64)
    assert np.all(keys[1:] > keys[:-1])
    assert np.array_equal(np.sort((keys & np.uint64(0x7FFFFFFF)).astype(np.int64)), np.arange(n))


def test_upgma_random_and_tied_matrices():
    """f4 kernel vs the oracle UPGMA on synthetic distance matrices: continuous (no ties), heavily
    tied (values on a grid of 8 levels) and all-equal, n from 2 to 700: identical merges, heights
    bit-equal (the same IEEE float64 operation sequence)."""
    import torch
    from oracle import upgma as U
    from paper_0901_2742_b200.runtime import upgma
    rng = np.random.default_rng(9)
    for n, kind in [(2, "c"), (3, "c"), (17, "t"), (64, "c"), (200, "t"), (333, "e"), (700, "t")]:
        if kind == "e":
            D = np.ones((n, n)) - np.eye(n)
        else:
            A = rng.random((n, n))
            if kind == "t":
                A = np.floor(A * 8) / 8
            D = np.triu(A, 1)
            D = D + D.T
        ref = U.upgma(D)
        got = upgma(torch.from_numpy(D).cuda())
        assert np.array_equal(got[0], ref[0]), (n, kind)
        assert np.array_equal(got[1], ref[1]) and np.array_equal(got[2], ref[2])


@pytest.mark.parametrize("cfg", [1, 2])
def test_bucket_guide_trees(cfg):
    """f4 on the path's output: every bucket's UPGMA tree on the GPU (from its float64 k-mer
    distances) equals the oracle's tree on the oracle's distances."""
    from oracle import upgma as U
    spec = gen.SPECS[cfg]
    a, o = gen.generate(cfg)
    ctx, sizes = _run_gpu(a, o, spec.alphabet, spec.k, spec.p, "tc")
    for b in range(spec.p):
        idx = ctx.bucket(b)[0]
        if len(idx) < 2:
            continue
        ii, jj = np.meshgrid(idx, idx, indexing="ij")
        Sref, dref = oracle.pairs_S(a, o, spec.k, ii.ravel(), jj.ravel())
        ref = U.upgma(U.distance_f64(Sref.reshape(len(idx), -1), dref.reshape(len(idx), -1)))
        got = ctx.bucket_guide_tree(b)
        assert np.array_equal(got[0], ref[0]) and np.array_equal(got[1], ref[1]) and np.array_equal(got[2], ref[2])



@pytest.mark.gpu
def test_host_load_pipelined():
    """Host inputs of 4 MB or more are copied in chunks with each chunk's k-mer counts started
    as it lands (sad_load): the results equal those of a device-resident load, a bad symbol in the
    last chunk is still reported with its position, and a reused context reloads correctly."""
    import torch
    from paper_0901_2742_b200 import SadError
    spec = gen.SPECS[3]
    a, o = gen.generate(3, n=16000)
    n = len(o) - 1
    assert int(o[-1]) >= 4 << 20
    ctx_h = _ctx(spec.alphabet, spec.k, 8, KERNELS[0])
    ctx_h.load(a, o, n, 0)
    sizes_h = ctx_h.run()
    ctx_d = _ctx(spec.alphabet, spec.k, 8, KERNELS[0])
    ctx_d.load(torch.from_numpy(a).cuda(), torch.from_numpy(o).cuda(), n, 0, residues=int(o[-1]))
    sizes_d = ctx_d.run()
    assert np.array_equal(sizes_h, sizes_d)
    for s in range(8):
        assert np.array_equal(ctx_h.local_rank(s), ctx_d.local_rank(s))
    assert np.array_equal(ctx_h.out_keys().cpu().numpy(), ctx_d.out_keys().cpu().numpy())
    # the same context again (chunk events and the profile flag reset per load)
    ctx_h.load(a, o, n, 0)
    assert np.array_equal(ctx_h.run(), sizes_d)
    assert np.array_equal(ctx_h.out_keys().cpu().numpy(), ctx_d.out_keys().cpu().numpy())
    bad = a.copy()
    pos = int(o[n - 1]) + 5
    bad[pos] = ord("X")
    ctx_e = _ctx(spec.alphabet, spec.k, 8, KERNELS[0])
    ctx_e.load(bad, o, n, 0)
    with pytest.raises(SadError) as e:
        ctx_e.run()
    assert e.value.name == "SAD_E_SYMBOL" and e.value.location == (n - 1, 5)


@pytest.mark.parametrize("kernel", [k for k in KERNELS if k in ("tc", "tc8", "tc1")])
def test_tile_edges(kernel):
    """Shard widths around the 256 x 240 tile grid of the tensor-core path: a last column block
    with 1, 16, 17, 239 or 240 real columns (the edge tiles run with N = the real columns rounded
    up to 16), a single row block, and shards of unequal width (N mod p != 0)."""
    rng = np.random.default_rng(23)
    fam = gen.random_set(rng, 40, "protein", 60, 200)
    for n, p in ((481, 1), (496, 1), (497, 1), (719, 1), (720, 1), (255, 1), (1443, 3)):
        a, o = gen.random_set(rng, n, "protein", 30, 260)
        if n > 600:                                    # shared families: S spans the fixed-point range
            s_f = gen.to_strings(*fam)
            s = gen.to_strings(a, o)
            s = [s_f[i % len(s_f)] if i % 3 == 0 else x for i, x in enumerate(s)]
            a, o = gen.from_strings(s)
        ctx, sizes = _run_gpu(a, o, "protein", 3, p, kernel)
        r = oracle.run(a, o, "protein", 3, p)
        _compare_full(ctx, sizes, r, a, o, p)


@pytest.mark.parametrize("kernel", [k for k in KERNELS if k != "alu"])
def test_long_k_deep_ring(kernel):
    """Operand rows of 64+ K blocks (16 384+ fp4 columns) in a shard: the all-pairs launch of the
    CTA-pair fp4 kernel then takes the 5-stage / 1-excess-buffer ring (k_allpairs_tc.cu,
    SAD_TC_DEEP_KB), chosen from the K of the previous step of the same context. DNA k = 7
    (V = 16 384, every k-mer present), random and family sequences of ~1.5-3.5 kb, p = 1 and 2.
    Two steps per context, each compared element-wise with the oracle."""
    rng = np.random.default_rng(77)
    seqs = ["".join(rng.choice(list("ACGT"), int(rng.integers(1500, 3500)))) for _ in range(420)]
    for _ in range(30):                                          # families: near-identical pairs
        base = seqs[int(rng.integers(0, len(seqs)))]
        x = list(base)
        for j in rng.integers(0, len(x), len(x) // 20):
            x[j] = "ACGT"[int(rng.integers(0, 4))]
        seqs.append("".join(x))
    seqs = [seqs[i] for i in rng.permutation(len(seqs))]
    a, o = gen.from_strings(seqs)
    for p in (1, 2):
        r = oracle.run(a, o, "dna", 7, p)
        ctx = _ctx("dna", 7, p, kernel)
        ctx.load(a, o, len(o) - 1, 0)
        for step in range(2):
            sizes = ctx.run()
            _compare_full(ctx, sizes, r, a, o, p)
        K = ctx.profile_info()[2]
        assert int(K.max()) >= 64 * 256, K
        ctx.close()


@pytest.mark.parametrize("kernel", [k for k in KERNELS if k != "alu"])
def test_wide_rows_several_slices(kernel):
    """Long rows through the block-per-row K4 (k_indicator_blk: average L - k + 1 >= 1024) with
    operand rows wider than one 16 KB shared-memory slice: DNA k = 8 (V = 65 536), random and
    near-duplicate sequences of 2.5-5 kb, so a shard has > 32 768 fp4 columns (two or more slices
    per row, the row's entries re-read per slice). p = 1 and 2, two steps per context, every
    output compared element-wise with the oracle."""
    rng = np.random.default_rng(91)
    seqs = ["".join(rng.choice(list("ACGT"), int(rng.integers(2500, 5000)))) for _ in range(150)]
    for _ in range(14):
        x = list(seqs[int(rng.integers(0, len(seqs)))])
        for j in rng.integers(0, len(x), len(x) // 25):
            x[j] = "ACGT"[int(rng.integers(0, 4))]
        seqs.append("".join(x))
    seqs = [seqs[i] for i in rng.permutation(len(seqs))]
    a, o = gen.from_strings(seqs)
    for p in (1, 2):
        r = oracle.run(a, o, "dna", 8, p)
        ctx = _ctx("dna", 8, p, kernel)
        ctx.load(a, o, len(o) - 1, 0)
        for step in range(2):
            sizes = ctx.run()
            _compare_full(ctx, sizes, r, a, o, p)
        K = ctx.profile_info()[2]
        assert int(K.max()) > 32768, K
        ctx.close()


@pytest.mark.parametrize("kernel", KERNELS)
def test_similarity_near_the_fp32_bound(kernel):
    """S up to 65 535 = the ABI's L - k + 1 bound (SAD_E_TOO_LONG), where the fp32 accumulators
    of the fp4 kernel must still be exact (S < 2^24) and the u16 lanes of the ALU kernel do not
    wrap: all-'A' sequences (one k-mer of count L - k + 1, no layer cap possible, K grows past the
    initial operand capacity -> SAD_E_REPLAN and a rerun), random DNA of 65 537 residues and
    mutated copies of it (S ~ 6e4 over 64 k-mers), next to short sequences."""
    rng = np.random.default_rng(65535)
    big = "".join(rng.choice(list("ACGT"), 65537))
    seqs = ["A" * 65537, "A" * 65537, "A" * 65000, big, big]
    for rate in (0.01, 0.05, 0.2):
        x = list(big)
        for j in rng.integers(0, len(x), int(rate * len(x))):
            x[j] = "ACGT"[int(rng.integers(0, 4))]
        seqs.append("".join(x))
    seqs += ["".join(rng.choice(list("ACGT"), int(rng.integers(3, 3000)))) for _ in range(40)]
    seqs = [seqs[i] for i in rng.permutation(len(seqs))]
    a, o = gen.from_strings(seqs)
    for p in (1, 2):
        ctx, sizes = _run_gpu(a, o, "dna", 3, p, kernel, keep_sim=True)
        r = oracle.run(a, o, "dna", 3, p)
        _compare_full(ctx, sizes, r, a, o, p)
        n = len(o) - 1
        sb = gen.shard_bounds(n, p)
        smax = 0
        for s in range(p):
            Sm = ctx.similarity(s)
            ii, jj = np.meshgrid(np.arange(sb[s], sb[s + 1]), np.arange(sb[s], sb[s + 1]), indexing="ij")
            Sref, _ = oracle.pairs_S(a, o, 3, ii.ravel(), jj.ravel())
            assert np.array_equal(Sm.ravel().astype(np.int64), Sref)
            smax = max(smax, int(Sref.max()))
        assert smax == 65535
        ctx.close()


def test_pipeline_double_buffered():
    """runtime.Pipeline (the e2e path of bench.py): steps over different host inputs taken in turn by
    two contexts on two streams, each step's keys and bucket sizes equal to the oracle's."""
    from paper_0901_2742_b200.runtime import Pipeline
    spec = gen.SPECS[2]
    sets = [gen.generate(spec, n=1200 + 97 * j, seed=300 + j) for j in range(5)]
    pipe = Pipeline(spec.alphabet, spec.k, spec.p, depth=2)
    got = []
    for j, (a, o) in enumerate(sets):
        pipe.submit(a, o)
        if j >= 1:
            h, sz = pipe.collect()
            got.append((h.clone().numpy(), sz))
    h, sz = pipe.collect()
    got.append((h.clone().numpy(), sz))
    pipe.close()
    for (a, o), (keys, sizes) in zip(sets, got):
        r = oracle.run(a, o, spec.alphabet, spec.k, spec.p)
        assert sizes.tolist() == r.bsize.tolist()
        idx = np.concatenate([np.asarray(b, np.int64) for b in r.buckets()])
        q = np.array([oracle.q(int(r.S[i]), int(r.den[i])) for i in idx], dtype=object)
        want = [(int(qq) << 31) + int(i) for qq, i in zip(q, idx)]     # GA mode: key = (q << 31) + index
        assert [int(x) & ((1 << 64) - 1) for x in keys.tolist()] == want
