"""Pins of the CPU oracle to things other than itself (no GPU).

Each pin cites the passage that fixes the value: SPEC.md hand values (relabelled
to the 20-letter alphabet where SPEC used B/X), the SURVEY worked example
(tests/golden), closed forms of sum-min, invariants of the method, and a Python
brute force (tests/bruteforce.py: Counter + Fraction) on small random inputs.
"""
import math
import os

import numpy as np
import pytest
from fractions import Fraction

import oracle
from synth import gen
from tests import bruteforce as bf

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------- counts (O2)

def test_counts_hand_values():
    # SPEC.md:153 "AAAA", k=2 -> {AA: 3}
    assert oracle.count("AAAA", 2) == {"AA": 3}
    # SPEC.md:154 "ACGT", k=4 -> {ACGT: 1}
    assert oracle.count("ACGT", 4) == {"ACGT": 1}
    # SPEC.md:155 "ABCAB", k=2 -> {AB:2, BC:1, CA:1}; relabelled B->D (SURVEY §8(c) pins)
    assert oracle.count("ADCAD", 2) == {"AD": 2, "DC": 1, "CA": 1}


@pytest.mark.parametrize("k", [1, 2, 3, 6])
def test_counts_vs_bruteforce_and_total(k):
    rng = np.random.default_rng(10 + k)
    for _ in range(40):
        L = int(rng.integers(k, 60))
        x = "".join(rng.choice(list("ACDEFGHIKLMNPQRSTVWY"), L))
        c = oracle.count(x, k)
        assert c == dict(bf.kmers(x, k))
        assert sum(c.values()) == L - k + 1          # SPEC.md:136 invariant: sum of counts == L-k+1


# ---------------------------------------------------------------- similarity (O4)

def test_similarity_hand_values():
    # SPEC.md:162 x == y == "ACGTACGT", k=3 -> 1.0
    S, d = oracle.pair("ACGTACGT", "ACGTACGT", 3)
    assert S == d == 6
    # SPEC.md:163 "AAAA" vs "CCCC", k=2 -> 0
    assert oracle.pair("AAAA", "CCCC", 2) == (0, 3)
    # SPEC.md:164 "ABCAB" vs "BCABX" -> 3/4 (relabelled B->D, X->W)
    assert oracle.pair("ADCAD", "DCADW", 2) == (3, 4)
    # SURVEY §8(c) brute-forced values: repeated k-mers, F = 1 without identity, DNA k=6
    assert oracle.pair("ACACAC", "CACACA", 2) == (4, 5)
    assert oracle.pair("AAAAC", "AAC", 2) == (2, 2)
    assert oracle.pair("ACGTACGTAC", "TTACGTACGG", 6) == (3, 5)


def test_fixed_point_values():
    # q = floor(2^32 S / den) (reading A5); closed forms: 3/4 = 3*2^30, etc.
    assert oracle.q(3, 4) == 3 * 2 ** 30 == 3221225472
    assert oracle.q(4, 5) == 3435973836
    assert oracle.q(3, 5) == 2576980377
    assert oracle.q(2, 5) == 1717986918
    assert oracle.q(1, 3) == 1431655765
    assert oracle.q(3, 5) + oracle.q(2, 5) == 2 ** 32 - 1      # floors truncate each term
    assert oracle.q(7, 7) == 2 ** 32 and oracle.q(0, 9) == 0
    # exact over a grid: q*den <= S*2^32 < (q+1)*den
    for den in (1, 2, 3, 7, 255, 256, 4097, 7995, 65535):
        for S in sorted({0, 1, den // 3, den // 2, den - 1, den}):
            qq = oracle.q(S, den)
            assert qq * den <= S << 32 < (qq + 1) * den


def test_rank_R_values():
    # ln(0.1+0.9) = 0, ln 0.1, ln 1.1 (natural log, reading A4)
    assert oracle.rank_R(0.9) == pytest.approx(0.0, abs=1e-15)
    assert oracle.rank_R(0.0) == pytest.approx(math.log(0.1))
    assert oracle.rank_R(1.0) == pytest.approx(0.0953101798, abs=1e-10)


def test_similarity_closed_forms_and_invariants():
    """sum_tau min(a,b) == sum_t [a>=t][b>=t] (A.1) == (sum a + sum b - sum|a-b|)/2 (A.2),
    computed from the oracle's COUNT output and compared with its PAIR output."""
    rng = np.random.default_rng(7)
    for alpha, letters in (("protein", "ACDEFGHIKLMNPQRSTVWY"), ("dna", "ACGT")):
        for k in (2, 3, 6):
            for _ in range(25):
                x = "".join(rng.choice(list(letters), int(rng.integers(k, 60))))
                y = "".join(rng.choice(list(letters), int(rng.integers(k, 60))))
                if rng.random() < 0.3:          # related pair
                    y = x[int(rng.integers(0, 5)):] + y[:5]
                    if len(y) < k:
                        y = x
                cx, cy = oracle.count(x, k), oracle.count(y, k)
                S, den = oracle.pair(x, y, k)
                keys = set(cx) | set(cy)
                a1 = sum(1 for t in keys for l in range(1, 70)
                         if cx.get(t, 0) >= l and cy.get(t, 0) >= l)
                a2 = (sum(cx.values()) + sum(cy.values()) - sum(abs(cx.get(t, 0) - cy.get(t, 0)) for t in keys))
                assert a2 % 2 == 0
                assert S == a1 == a2 // 2
                assert den == min(len(x), len(y)) - k + 1
                assert 0 <= S <= den                               # 0 <= F <= 1
                assert oracle.pair(y, x, k) == (S, den)           # symmetry
                assert oracle.pair(x, x, k) == (len(x) - k + 1,) * 2   # F(x,x) = 1
                assert S == bf.S(x, y, k)


# ---------------------------------------------------------------- the worked example

def _golden(name):
    seqs, kv, buckets = [], {}, []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            tok = line.split()
            if tok[0] == "seq":
                seqs.append(tok[2])
            elif tok[0] == "bucket":
                buckets.append([int(t) for t in tok[2:]])
            else:
                kv[tok[0]] = tok[1:]
    return seqs, kv, buckets


def test_worked_example():
    seqs, kv, buckets = _golden("worked_example_k2_dna.txt")
    k, p = int(kv["k"][0]), int(kv["p"][0])
    a, o = gen.from_strings(seqs)
    r = oracle.run(a, o, kv["alphabet"][0], k, p)
    assert [int(t) - 2 ** 32 for t in r.T] == [int(v) for v in kv["T_minus_2p32"]]
    assert r.anc.tolist() == [int(v) for v in kv["ancestors"]]
    assert r.ga == int(kv["ga"][0])
    assert r.S.tolist() == [int(v) for v in kv["rank_S"]]
    assert r.den.tolist() == [int(v) for v in kv["rank_den"]]
    assert r.sorted.tolist() == [int(v) for v in kv["sorted"]]
    assert r.samples.tolist() == [int(v) for v in kv["samples"]]
    assert r.pivots.tolist() == [int(v) for v in kv["pivots"]]
    assert r.buckets() == buckets
    # and the brute force agrees
    b = bf.pipeline(seqs, k, p)
    assert b["buckets"] == buckets and b["ga"] == r.ga


# ---------------------------------------------------------------- whole pipeline vs brute force

@pytest.mark.parametrize("alpha,k", [("protein", 2), ("protein", 3), ("dna", 2), ("dna", 6), ("dna", 3)])
@pytest.mark.parametrize("p", [1, 2, 4, 8])
def test_pipeline_vs_bruteforce(alpha, k, p):
    rng = np.random.default_rng(1000 * p + 10 * k + len(alpha))
    for trial in range(3):
        n = int(rng.integers(p * p, max(p * p + 1, 64) + 1))
        if trial == 0:
            a, o = gen.random_set(rng, n, alpha, k, 60)
        else:   # related families (more ties, more repeated k-mers)
            spec = gen.Spec("t", n, alpha, k, p, 2, "equal", 0.0, ("normal", 30, 10, max(k, 8), 60),
                            (0.05, 0.3), 0.05, int(rng.integers(1 << 30)))
            a, o = gen.generate(spec)
        seqs = gen.to_strings(a, o)
        r = oracle.run(a, o, alpha, k, p)
        b = bf.pipeline(seqs, k, p)
        assert [int(t) for t in r.T] == b["T"]
        assert r.anc.tolist() == b["anc"]
        assert r.ga == b["ga"]
        assert [oracle.q(int(s), int(d)) for s, d in zip(r.S, r.den)] == [bf.fixed(f) for f in b["f"]]
        assert all(int(s) * f.denominator == f.numerator * int(d) for s, d, f in zip(r.S, r.den, b["f"]))
        assert r.sorted.tolist() == b["sorted"]
        assert r.samples.tolist() == b["samples"]
        assert r.pivots.tolist() == b["pivots"]
        assert r.bucket.tolist() == b["bucket"]
        assert r.buckets() == b["buckets"]


@pytest.mark.parametrize("alpha,k", [("protein", 3), ("dna", 2), ("dna", 6)])
@pytest.mark.parametrize("p", [2, 3, 4])
def test_pipeline_samples_mode_vs_bruteforce(alpha, k, p):
    """SURVEY §8(f) f1 (the rank against the k*p gathered samples): the oracle's
    mode "samples" against the brute force (Counter + Fraction), every intermediate."""
    rng = np.random.default_rng(7000 + 100 * p + k)
    for trial in range(3):
        n = int(rng.integers(p * p, max(p * p + 1, 48) + 1))
        if trial == 0:
            a, o = gen.random_set(rng, n, alpha, k, 50)
        else:
            spec = gen.Spec("t", n, alpha, k, p, 2, "equal", 0.0, ("normal", 30, 10, max(k, 8), 60),
                            (0.05, 0.3), 0.05, int(rng.integers(1 << 30)))
            a, o = gen.generate(spec)
        seqs = gen.to_strings(a, o)
        r = oracle.run(a, o, alpha, k, p, mode="samples")
        b = bf.pipeline(seqs, k, p, mode="samples")
        assert [int(t) for t in r.T] == b["T"]
        assert r.rsamples.tolist() == b["rsamples"]
        assert r.ga == -1 and set(r.den.tolist()) == {1}
        assert [int(s) for s in r.S] == [int(f) for f in b["f"]]
        assert r.sorted.tolist() == b["sorted"]
        assert r.samples.tolist() == b["samples"]
        assert r.pivots.tolist() == b["pivots"]
        assert r.buckets() == b["buckets"]


def test_samples_mode_hand_case():
    """f1 by hand: p = 2, four DNA sequences, k = 2. Shards {0,1}, {2,3};
    T within each shard, one rank sample per shard at position floor(1*2/2) = 1 of its local order
    (the smaller T), rank T' = q(x, s0) + q(x, s1) (reading A27: the exact fixed-point sum; the
    mean's common factor 1/2 is dropped like A5's 1/N)."""
    seqs = ["ACGT", "ACGA", "TTTT", "TTTA"]
    a, o = gen.from_strings(seqs)
    r = oracle.run(a, o, "dna", 2, 2, mode="samples")
    # shard 0: F(0,1) = |{AC,CG}| / 3 = 2/3 -> T0 = T1 = 2^32 + floor(2^32 * 2/3)
    # shard 1: F(2,3) = |{TT, TT}| = min counts: TT 3 vs 2 -> 2/3 -> T2 = T3; ties -> smaller index
    assert r.rsamples.tolist() == [0, 2]
    q23 = (2 << 32) // 3
    assert [int(t) for t in r.T] == [(1 << 32) + q23] * 4
    # T'_0 = q(ACGT, ACGT) + q(ACGT, TTTT) = 2^32 + 0 (S(ACGT, TTTT) = 0)
    assert int(r.S[0]) == 1 << 32
    # T'_1: F(ACGA, ACGT) = 2/3, F(ACGA, TTTT) = 0
    assert int(r.S[1]) == q23
    # T'_2: F(TTTT, ACGT) = 0, self = 2^32
    assert int(r.S[2]) == 1 << 32
    # T'_3: F(TTTA, ACGT) = 0 (TT, TA vs AC, CG, GT), F(TTTA, TTTT) = 2/3
    assert int(r.S[3]) == q23
    # order (T', index): 1 < 3 < 0 < 2; the rank samples' own T' via the reference-set routine
    assert oracle.rank_vs_set(a, o, 2, [0, 2]).tolist() == [int(x) for x in r.S]


@pytest.mark.parametrize("alpha,k", [("protein", 3), ("dna", 2), ("dna", 6)])
def test_sample_degeneracy(alpha, k):
    """SPEC S:208 / acceptance #3: ranking against samples = the FULL set equals
    the centralized rank exactly. The reference-set sum (or_rank_vs_set, the f1 rank path) over all
    N sequences must equal T_i of the centralized run (p = 1, the O4 all-pairs loop, a different
    code path), and the reported R = ln(0.1 + D) with D = T'/(N 2^32) and
    D = T/(N 2^32) are the same doubles; pinned to the Counter + Fraction brute force too."""
    rng = np.random.default_rng(900 + k)
    for trial in range(4):
        n = int(rng.integers(8, 50))
        a, o = gen.random_set(rng, n, alpha, k, 60)
        if trial == 3:                                  # repeats, so ties exist
            seqs = gen.to_strings(a, o)
            seqs = seqs[: n // 2] + seqs[: n - n // 2]
            a, o = gen.from_strings(seqs)
        seqs = gen.to_strings(a, o)
        cen = oracle.run(a, o, alpha, k, 1)
        deg = oracle.rank_vs_set(a, o, k, np.arange(n))
        assert deg.tolist() == cen.T.tolist()
        assert deg.tolist() == bf.pipeline(seqs, k, 1)["T"]
        D = lambda t: float(t) / (n * 2.0 ** 32)
        assert [oracle.rank_R(D(x)) for x in deg] == [oracle.rank_R(D(x)) for x in cen.T]
        # and the f1 mode's own sums equal the reference-set routine on its rank samples
        if n >= 9:
            r = oracle.run(a, o, alpha, k, 3, mode="samples")
            assert oracle.rank_vs_set(a, o, k, r.rsamples).tolist() == [int(x) for x in r.S]


# ---------------------------------------------------------------- invariants (north star)

def _check_invariants(r, n, p):
    flat = [i for bk in r.buckets() for i in bk]
    assert sorted(flat) == list(range(n))                         # permutation of the input
    assert int(r.bsize.sum()) == n
    key = lambda i: (int(r.S[i]), int(r.den[i]), i)
    less = lambda a, b: (a[0] * b[1], a[2]) < (b[0] * a[1], b[2])
    for bk in r.buckets():
        for u, v in zip(bk, bk[1:]):
            assert less(key(u), key(v))                           # each bucket sorted
    nonempty = [bk for bk in r.buckets() if bk]
    for b1, b2 in zip(nonempty, nonempty[1:]):
        assert less(key(b1[-1]), key(b2[0]))                      # max(b) < min(b+1)


def test_invariants_configs_1_2():
    for c in (1, 2):
        spec = gen.SPECS[c]
        a, o = gen.generate(c)
        r = oracle.run(a, o, spec.alphabet, spec.k, spec.p)
        n = len(o) - 1
        _check_invariants(r, n, spec.p)
        w = n // spec.p
        assert r.bsize.max() <= 2 * w + spec.p


def test_p1_single_bucket_is_sorted_input():
    a, o = gen.generate(1)
    r = oracle.run(a, o, "protein", 3, 1)
    assert r.pivots.size == 0 and r.bsize.tolist() == [64]
    assert r.buckets()[0] == r.sorted.tolist()
    assert r.anc[0] == r.ga


def test_adversarial_inputs():
    # poly-A (counts far above any cap), L == k, identical sequences (all ties -> index order),
    # containment (F = 1 without identity)
    seqs = ["A" * 300, "A" * 3, "ACD", "ACDEFGHIK" * 10, "ACDEFGHIK" * 10, "ACDEFGHIK" * 10,
            "AAAAAAAAAC", "AAC", "W" * 40, "ACDEFGHIK" * 3, "KIHGFEDCA" * 4, "MMMMMMMMMMMMMM"]
    a, o = gen.from_strings(seqs)
    for p in (1, 2, 3):
        r = oracle.run(a, o, "protein", 3, p)
        b = bf.pipeline(seqs, 3, p)
        assert r.buckets() == b["buckets"] and [int(t) for t in r.T] == b["T"]
        _check_invariants(r, len(seqs), p)
    same = ["ACDEFGHIKL"] * 16
    a, o = gen.from_strings(same)
    r = oracle.run(a, o, "protein", 3, 4)
    assert r.ga == 0 and r.anc.tolist() == [0, 4, 8, 12]
    assert [i for bk in r.buckets() for i in bk] == list(range(16))


def test_errors():
    a, o = gen.from_strings(["ACDX", "ACDE"])                     # X rejected (reading A18)
    with pytest.raises(oracle.OracleError) as e:
        oracle.run(a, o, "protein", 3, 1)
    assert e.value.name == "SYMBOL" and (e.value.idx, e.value.pos) == (0, 3)
    a, o = gen.from_strings(["ACDE", "AC"])                       # L < k (reading A19)
    with pytest.raises(oracle.OracleError) as e:
        oracle.run(a, o, "protein", 3, 1)
    assert e.value.name == "TOO_SHORT" and e.value.idx == 1
    a, o = gen.from_strings(["ACDE"] * 5)                         # w < p (reading A16)
    with pytest.raises(oracle.OracleError) as e:
        oracle.run(a, o, "protein", 3, 3)
    assert e.value.name == "INSUFFICIENT"
    with pytest.raises(oracle.OracleError) as e:
        oracle.run(np.zeros(0, np.uint8), np.zeros(1, np.int64), "protein", 3, 1)
    assert e.value.name == "EMPTY"


# ---------------------------------------------------------------- PSRS load bound

@pytest.mark.parametrize("p", [2, 4, 8])
def test_psrs_load_bound_trials(p):
    """n = 4 p^3 short random DNA sequences (heavy rank ties), 70 seeded rounds per p
    (210 in total, SPEC.md:733 asks >= 200): every bucket <= 2w + p, and < 2w when
    p | w (the paper's "always less than 2w", PAPER.md:188,
    is read as reading A23)."""
    n = 4 * p ** 3
    w = n // p
    rng = np.random.default_rng(p)
    for _ in range(70):
        a, o = gen.random_set(rng, n, "dna", 2, 9)
        r = oracle.run(a, o, "dna", 2, p)
        assert r.bsize.sum() == n
        assert r.bsize.max() <= 2 * w + p
        assert r.bsize.max() < 2 * w                                # p | w here


# ---------------------------------------------------------------- f4: UPGMA guide tree (oracle)

def test_upgma_spec_examples():
    """n = 2 -> one join at d(0,1)/2; n = 3 with d(0,1) = 0.2 < d(0,2) = 0.8,
    d(1,2) = 0.9 -> {0,1} first, then with 2 at height (0.8 + 0.9)/4; n = 1 -> no join."""
    from oracle import upgma as U
    m, h, s = U.upgma(np.array([[0.0, 0.6], [0.6, 0.0]]))
    assert m.tolist() == [[0, 1]] and h.tolist() == [0.3] and s.tolist() == [2]
    D = np.array([[0.0, 0.2, 0.8], [0.2, 0.0, 0.9], [0.8, 0.9, 0.0]])
    m, h, s = U.upgma(D)
    assert m.tolist() == [[0, 1], [3, 2]]
    assert h[0] == 0.1 and h[1] == (0.8 + 0.9) / 4 and s.tolist() == [2, 3]
    m, h, s = U.upgma(np.zeros((1, 1)))
    assert len(m) == 0


def test_upgma_ties_lexicographic():
    """D-M1: all distances equal -> (0,1) first, then the new cluster (position 0) with 2, ..."""
    from oracle import upgma as U
    n = 5
    D = np.ones((n, n)) - np.eye(n)
    m, h, s = U.upgma(D)
    assert m.tolist() == [[0, 1], [5, 2], [6, 3], [7, 4]]
    assert h.tolist() == [0.5] * 4


def test_upgma_vs_scipy_average_linkage():
    """Special case that reduces to a library routine: on tie-free random metrics, UPGMA equals
    scipy.cluster.hierarchy.linkage(method='average') (same merge sets, heights = d/2)."""
    from scipy.cluster.hierarchy import linkage
    from scipy.spatial.distance import squareform
    from oracle import upgma as U
    rng = np.random.default_rng(3)
    for n in (4, 9, 30, 64):
        X = rng.random((n, 5))
        D = np.sqrt(((X[:, None, :] - X[None, :, :]) ** 2).sum(-1))
        m, h, s = U.upgma(D)
        Z = linkage(squareform(D, checks=False), method="average")
        assert np.allclose(h * 2, Z[:, 2], rtol=0, atol=1e-12)
        assert [sorted(r) for r in m.tolist()] == [sorted(map(int, r)) for r in Z[:, :2]]
        assert s.tolist() == Z[:, 3].astype(int).tolist()
        assert np.all(np.diff(h) >= -1e-15)                       # ultrametric: heights never decrease


# ---------------------------------------------------------------- the oracle's sampled checkers

@pytest.mark.parametrize("alpha,k", [("protein", 3), ("dna", 2), ("dna", 6)])
@pytest.mark.parametrize("p", [1, 2, 3, 8])
def test_sampled_checkers_vs_bruteforce(alpha, k, p):
    """or_rows_T (T_i of selected rows, O4 for one row, PAPER.md:44-46 with reading A5),
    or_rank_vs_set (f1's T' against an arbitrary reference set, reading A27) and or_pairs_S
    (S, den of arbitrary pairs) are the checkers of the full-size sampled GPU tests;
    pinned here to the Counter + Fraction brute force, not to oracle.run."""
    rng = np.random.default_rng(31000 + 100 * p + 10 * k + len(alpha))
    for trial in range(2):
        n = int(rng.integers(max(p, 2) * 3, 40))
        if trial == 0:
            a, o = gen.random_set(rng, n, alpha, k, 50)
        else:
            spec = gen.Spec("t", n, alpha, k, p, 2, "equal", 0.0, ("normal", 30, 10, max(k, 8), 60),
                            (0.05, 0.3), 0.05, int(rng.integers(1 << 30)))
            a, o = gen.generate(spec)
        seqs = gen.to_strings(a, o)
        sh = bf.shards(n, p)
        T = [0] * n
        for s in sh:
            for i in s:
                T[i] = sum(bf.fixed(bf.F(seqs[i], seqs[j], k)) for j in s)
        rows = sorted(set(rng.integers(0, n, 7).tolist()) | {0, n - 1})
        assert [int(t) for t in oracle.rows_T(a, o, k, p, rows)] == [T[r] for r in rows]
        ref = rng.integers(0, n, 5).tolist()
        want = [sum(bf.fixed(bf.F(seqs[i], seqs[t], k)) for t in ref) for i in range(n)]
        assert [int(t) for t in oracle.rank_vs_set(a, o, k, ref)] == want
        pi, pj = rng.integers(0, n, 25), rng.integers(0, n, 25)
        S, d = oracle.pairs_S(a, o, k, pi, pj)
        for x, y, s_, d_ in zip(pi, pj, S, d):
            f = bf.F(seqs[x], seqs[y], k)
            assert int(s_) == bf.S(seqs[x], seqs[y], k)
            assert int(d_) == min(len(seqs[x]), len(seqs[y])) - k + 1
            assert Fraction(int(s_), int(d_)) == f


def test_long_sequences_near_the_key_bound():
    """Sequences with L - k + 1 up to 65 535 (the ABI's SAD_E_TOO_LONG bound, DESIGN A.3): S near
    2^16, checked against closed forms. All-'A' DNA of length L has one k-mer of count L - k + 1,
    so S(x, y) = min(L_x, L_y) - k + 1 and F = 1; a periodic sequence (ACGT)^m has
    four k-mers (k = 3), none of them AAA."""
    k = 3
    Ls = [65537, 65537, 60000, 40001]
    seqs = ["A" * L for L in Ls] + ["ACGT" * 16384 + "A"]
    a, o = gen.from_strings(seqs)
    S, d = oracle.pairs_S(a, o, k, [0, 0, 1, 2, 3, 4, 4], [1, 2, 2, 3, 0, 4, 0])
    assert S.tolist() == [65535, 59998, 59998, 39999, 39999, 65535, 0]
    assert d.tolist() == [65535, 59998, 59998, 39999, 39999, 65535, 65535]
