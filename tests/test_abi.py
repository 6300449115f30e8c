"""CPU checks of the boundary: libsad.so loads, exports every symbol include/sad.h declares,
and its pure host functions (exchange sizes, pack plan) match a direct model. No GPU."""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_0901_2742_b200 import build
    build.build()
    from paper_0901_2742_b200 import _lib
    return _lib


def test_exports_every_declared_symbol(L):
    hdr = open(os.path.join(ROOT, "include", "sad.h")).read()
    declared = sorted(set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(sad_\w+)\s*\(", hdr, flags=re.M)))
    assert len(declared) >= 25
    lib = L.lib()
    for name in declared:
        assert hasattr(lib, name), f"libsad.so does not export {name}"
    assert sorted(declared) == sorted(L.SYMBOLS)
    assert lib.sad_abi_version() == 2


def _model_sizes(p, G, rank, c):
    bpr = p // G
    own = lambda r: range(r * bpr, (r + 1) * bpr)
    ss = [sum(c[s, b, 0] for s in own(rank) for b in own(r)) for r in range(G)]
    sr = [sum(c[s, b, 1] for s in own(rank) for b in own(r)) for r in range(G)]
    rs = [sum(c[s, b, 0] for s in own(r) for b in own(rank)) for r in range(G)]
    rr = [sum(c[s, b, 1] for s in own(r) for b in own(rank)) for r in range(G)]
    return ss, sr, rs, rr


@pytest.mark.parametrize("p,G", [(1, 1), (2, 2), (8, 1), (8, 2), (8, 4), (8, 8), (6, 3)])
def test_exchange_sizes_and_pack_plan(L, p, G):
    from paper_0901_2742_b200.runtime import exchange_sizes, pack_plan
    rng = np.random.default_rng(p * 10 + G)
    c = rng.integers(0, 50, size=(p, p, 2)).astype(np.int64)
    for rank in range(G):
        got = exchange_sizes(p, G, rank, c)
        want = _model_sizes(p, G, rank, c)
        for g, w in zip(got, want):
            assert g.tolist() == w
        seg = pack_plan(p, G, rank, c)
        # slices grouped by destination rank, then (local shard, bucket); offsets are running sums
        bpr = p // G
        cs = cr = 0
        for r in range(G):
            for s in range(bpr):
                for b in range(r * bpr, (r + 1) * bpr):
                    assert seg[s, b].tolist() == [cs, cr]
                    cs += c[rank * bpr + s, b, 0]
                    cr += c[rank * bpr + s, b, 1]
        assert cs == sum(got[0]) and cr == sum(got[1])


def test_bad_args(L):
    from paper_0901_2742_b200.runtime import exchange_sizes
    with pytest.raises(L.SadError):
        exchange_sizes(6, 4, 0, np.zeros((6, 6, 2), np.int64))


def test_rank_stats_spec_examples():
    """SPEC S:633-641 rank_stats examples (SURVEY §8(f) f2 reporting): a == b -> zero spread;
    a = [0, 0], b = [1, 3] -> mean_b 2, diffs [1, 3], population variance 1, stddev 1."""
    from paper_0901_2742_b200 import stats
    r = stats.rank_stats([0.5, 0.25], [0.5, 0.25])
    assert r["Variance w.r.t. Centralized"] == 0 and r["Standard Dev. w.r.t Centralized"] == 0
    r = stats.rank_stats([0, 0], [1, 3])
    assert r["Average Globalized"] == 2 and r["Variance w.r.t. Centralized"] == 1
    assert r["Standard Dev. w.r.t Centralized"] == 1
    assert r["(Maximum, Minimum) Globalized"] == (3, 1)
    # R values of SPEC S:180-182 (natural log)
    assert abs(stats.rank_R([0.0])[0] + 2.302585093) < 1e-9 and abs(stats.rank_R([1.0])[0] - 0.0953101798) < 1e-9
