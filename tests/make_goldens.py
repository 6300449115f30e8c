#!/usr/bin/env python
"""Write the full-size parity goldens of BASELINE.json's five configs (tests/golden/full/).

    python tests/make_goldens.py [--only cfg4_p8,...] [--threads N]

TEST INFRASTRUCTURE. It calls only ``oracle/`` (the plain C oracle)
on the seeded inputs of ``synth/gen.py``; nothing here touches the CUDA path, and no
expected value comes from it. It lives under tests/ because only tests/, smoke() and
bench.py's CPU legs may run the oracle.

Every layout the round-1 verdict lists is written: config 1 (p=2), config 2 (p=8),
config 3 (p=2, 4, 8), config 4 (p=8; the same output for G = 1, 2, 4, 8, since the shards
are the same) and config 5 (p=1, 2, 4, 8). Each golden is a small JSON file holding
  * the SHA-256 of the generated input (ascii, offsets), so a generator drift is caught
    before any comparison;
  * the small outputs in full: local ancestors, GA, sample and pivot sequences, bucket sizes,
    the load report (max bucket vs 2w + p, < 2w when p | w: PAPER.md:188, reading A23);
  * per shard SHA-256 digests of T (u64), S_i and den_i (i64), the key-sorted order (i64);
    per bucket digests of the bucket's sequence order (i64), plus 32 sampled values of
    each array (for a readable diff when a digest differs).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from synth import gen  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "full")

LAYOUTS = [("cfg1", 1, 2, "ga"), ("cfg2", 2, 8, "ga"), ("cfg3", 3, 2, "ga"), ("cfg3", 3, 4, "ga"),
           ("cfg3", 3, 8, "ga"), ("cfg5", 5, 1, "ga"), ("cfg5", 5, 2, "ga"), ("cfg5", 5, 4, "ga"),
           ("cfg5", 5, 8, "ga"), ("cfg4", 4, 8, "ga"),
           # the rank against the k*p gathered samples (reading A27)
           ("cfg1", 1, 2, "samples"), ("cfg2", 2, 8, "samples"), ("cfg3", 3, 8, "samples"),
           ("cfg5", 5, 8, "samples"), ("cfg4", 4, 8, "samples")]


def sha(a, dtype) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype=dtype).tobytes()).hexdigest()


def input_digest(a, o) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(a, dtype=np.uint8).tobytes())
    h.update(np.ascontiguousarray(o, dtype="<i8").tobytes())
    return h.hexdigest()


def sample_positions(n: int, m: int = 32, seed: int = 7):
    rng = np.random.default_rng(seed + n)
    return sorted(set(int(x) for x in rng.integers(0, n, size=min(m, n))))


def make(name: str, cfg: int, p: int, threads: int, mode: str = "ga") -> dict:
    spec = gen.SPECS[cfg]
    a, o = gen.generate(spec)
    n = len(o) - 1
    t0 = time.perf_counter()
    r = oracle.run(a, o, spec.alphabet, spec.k, p, nthreads=threads, mode=mode)
    dt = time.perf_counter() - t0
    sb = gen.shard_bounds(n, p)
    shards = []
    for s in range(p):
        lo, hi = sb[s], sb[s + 1]
        pos = sample_positions(hi - lo)
        shards.append({
            "lo": lo, "hi": hi,
            "T": sha(r.T[lo:hi], "<u8"), "S": sha(r.S[lo:hi], "<i8"), "den": sha(r.den[lo:hi], "<i8"),
            "sorted": sha(r.sorted[lo:hi], "<i8"),
            "sample_pos": pos,
            "T_sample": [int(r.T[lo + i]) for i in pos],
            "S_sample": [int(r.S[lo + i]) for i in pos],
            "den_sample": [int(r.den[lo + i]) for i in pos],
            "sorted_sample": [int(r.sorted[lo + i]) for i in pos],
        })
    buckets, off = [], 0
    for b in range(p):
        m = int(r.bsize[b])
        order = r.border[off: off + m]
        pos = sample_positions(max(m, 1))
        buckets.append({"n": m, "order": sha(order, "<i8"),
                        "sample_pos": [i for i in pos if i < m],
                        "order_sample": [int(order[i]) for i in pos if i < m]})
        off += m
    w_max = max(sb[s + 1] - sb[s] for s in range(p))
    w = n // p
    mb = int(max(r.bsize))
    return {
        "name": f"{name}_p{p}" + ("" if mode == "ga" else f"_{mode}"), "mode": mode, "config": cfg, "p": p, "n": n,
        "alphabet": spec.alphabet, "k": spec.k,
        "seed": spec.seed, "residues": int(o[-1]), "input_sha256": input_digest(a, o),
        "anc": [int(x) for x in r.anc], "ga": int(r.ga),
        "samples": [int(x) for x in r.samples], "pivots": [int(x) for x in r.pivots],
        "rank_samples": None if r.rsamples is None else [int(x) for x in r.rsamples],
        "bsize": [int(x) for x in r.bsize],
        "load": {"max_bucket": mb, "w": w, "w_max": w_max, "bound_2w_plus_p": 2 * w_max + p,
                 "holds": mb <= 2 * w_max + p, "p_divides_w": (n % p == 0 and w % p == 0),
                 "below_2w": mb < 2 * w},
        "shards": shards, "buckets": buckets,
        "oracle": {"threads": oracle.threads(threads), "seconds": round(dt, 2),
                   "stage_ms": [round(float(x), 1) for x in r.stage_ms]},
        "written_by": "tests/make_goldens.py (oracle/ only)",
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="")
    ap.add_argument("--threads", type=int, default=0)
    args = ap.parse_args()
    os.makedirs(OUT, exist_ok=True)
    want = set(x for x in args.only.split(",") if x)
    for name, cfg, p, mode in LAYOUTS:
        tag = f"{name}_p{p}" + ("" if mode == "ga" else f"_{mode}")
        if want and tag not in want:
            continue
        g = make(name, cfg, p, args.threads, mode)
        path = os.path.join(OUT, f"{tag}.json")
        with open(path, "w") as f:
            json.dump(g, f, indent=1)
        print(f"{tag}: n={g['n']} oracle {g['oracle']['seconds']} s on {g['oracle']['threads']} threads "
              f"-> {os.path.relpath(path, ROOT)}", flush=True)


if __name__ == "__main__":
    main()
