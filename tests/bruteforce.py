"""Brute-force reimplementation of the path on tiny inputs (pins the oracle).

Independent of oracle/sad_oracle.c: Python strings, collections.Counter for the
k-mer multisets and fractions.Fraction for every similarity, so exact rational
comparison replaces the oracle's cross-multiplication and fixed point is taken
from the reduced fraction.  Follows PAPER.md §2 (lines 40-50, 66-77) with the
readings of SURVEY.md §8(c).
"""
from collections import Counter
from fractions import Fraction


def kmers(x: str, k: int) -> Counter:
    """nx(tau): every contiguous length-k window, overlaps included."""
    return Counter(x[i:i + k] for i in range(len(x) - k + 1))


def S(x: str, y: str, k: int) -> int:
    cx, cy = kmers(x, k), kmers(y, k)
    return sum(min(c, cy[t]) for t, c in cx.items())


def F(x: str, y: str, k: int) -> Fraction:
    """r_ij of PAPER.md:42 without the stray tau (reading A1)."""
    return Fraction(S(x, y, k), min(len(x), len(y)) - k + 1)


def fixed(f: Fraction) -> int:
    """floor(2^32 * f)."""
    return (f.numerator << 32) // f.denominator


def shards(n: int, p: int):
    base, extra = divmod(n, p)
    b = [0]
    for s in range(p):
        b.append(b[-1] + base + (1 if s < extra else 0))
    return [list(range(b[s], b[s + 1])) for s in range(p)]


def pipeline(seqs, k: int, p: int, mode: str = "ga") -> dict:
    """mode "ga": rank against the global ancestor (readings A7, A8); "samples": the paper's
    listing PAPER.md:67-72 literally: local order by T (ties by index), the
    p-1 sequences at positions floor(j w/p) of every shard as rank samples, and the rank
    T'_i = sum_s floor(2^32 F(x_i, s)) (the mean's common 1/(p(p-1)) dropped, reading A27) with
    index tie-break."""
    n = len(seqs)
    sh = shards(n, p)
    T = [0] * n
    for s in sh:
        for i in s:
            T[i] = sum(fixed(F(seqs[i], seqs[j], k)) for j in s)
    anc = [max(s, key=lambda i: (T[i], -i)) for s in sh]
    U = {a: sum(fixed(F(seqs[a], seqs[b], k)) for b in anc) for a in anc}
    ga = max(anc, key=lambda a: (U[a], -a))
    rsamples = None
    if mode == "samples":
        rsamples = []
        for s in sh:
            loc = sorted(s, key=lambda i: (T[i], i))
            w = len(loc)
            rsamples += [loc[(j * w) // p - 1] for j in range(1, p)]
        f = [Fraction(sum(fixed(F(seqs[i], seqs[t], k)) for t in rsamples)) for i in range(n)]
        ga = -1
    else:
        f = [F(seqs[i], seqs[ga], k) for i in range(n)]
    key = lambda i: (f[i], i)
    srt = [sorted(s, key=key) for s in sh]
    samples = []
    for s in srt:
        w = len(s)
        samples += [s[(j * w) // p - 1] for j in range(1, p)]
    Y = sorted(samples, key=key)
    pivots = [Y[p // 2 + i * p - 1] for i in range(p - 1)]
    bucket = []
    for i in range(n):
        b = p - 1
        for t, pv in enumerate(pivots):
            if key(i) <= key(pv):
                b = t
                break
        bucket.append(b)
    buckets = [sorted([i for i in range(n) if bucket[i] == b], key=key) for b in range(p)]
    return dict(T=T, anc=anc, ga=ga, f=f, sorted=[i for s in srt for i in s], samples=samples,
                pivots=pivots, bucket=bucket, buckets=buckets, rsamples=rsamples)
