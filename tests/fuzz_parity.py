"""Randomized GPU-vs-oracle parity sweep (GPU box): many small random workloads — alphabet, k,
p, sequence count and length mix, repeats, identical and contained sequences — each run through
the full path on every kernel variant and compared with the oracle bit for bit (the same checks
as tests/test_gpu_parity.py::_compare_full). Stops at the first mismatch and prints its seed.

    python tests/fuzz_parity.py [seconds] [first_seed]

(A script, not a pytest module: it lives under tests/ because only tests/ may run the oracle.)
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import oracle  # noqa: E402
from synth import gen  # noqa: E402
from test_gpu_parity import _compare_full, _run_gpu  # noqa: E402

KERNELS = ["tc", "tc1", "tc8", "tc8full", "alu"]


def case(seed):
    rng = np.random.default_rng(seed)
    alpha = "protein" if rng.random() < 0.7 else "dna"
    k = int(rng.choice([2, 3])) if alpha == "protein" else int(rng.choice([3, 4, 6]))
    letters = list("ACDEFGHIKLMNPQRSTVWY" if alpha == "protein" else "ACGT")
    p = int(rng.choice([1, 2, 3, 4, 8]))
    n = int(rng.integers(max(p * p, 4), 700))
    seqs = []
    fam = ["".join(rng.choice(letters, int(rng.integers(20, 400)))) for _ in range(int(rng.integers(1, 8)))]
    for _ in range(n):
        u = rng.random()
        if u < 0.35:                                   # family member: point mutations of a root
            s = list(fam[int(rng.integers(0, len(fam)))])
            for _ in range(int(rng.integers(0, max(1, len(s) // 5)))):
                s[int(rng.integers(0, len(s)))] = str(rng.choice(letters))
            s = "".join(s)
        elif u < 0.45:                                 # low complexity: repeats push counts over caps
            unit = "".join(rng.choice(letters, int(rng.integers(1, 5))))
            s = unit * int(rng.integers(2, 300))
        elif u < 0.5:                                  # containment / identity
            f = fam[int(rng.integers(0, len(fam)))]
            a = int(rng.integers(0, max(1, len(f) - k)))
            s = f[a: a + int(rng.integers(k, len(f) - a + 1))]
        else:
            s = "".join(rng.choice(letters, int(rng.integers(k, 600))))
        if len(s) < k:
            s = s + "".join(rng.choice(letters, k - len(s)))
        seqs.append(s)
    a, o = gen.from_strings(seqs)
    return alpha, k, p, a, o


def main(seconds=240.0, seed0=1):
    t0, seed, runs = time.time(), int(seed0), 0
    while time.time() - t0 < seconds:
        alpha, k, p, a, o = case(seed)
        r = oracle.run(a, o, alpha, k, p)
        for kern in KERNELS:
            try:
                ctx, sizes = _run_gpu(a, o, alpha, k, p, kern)
                _compare_full(ctx, sizes, r, a, o, p)
            except Exception as e:                      # noqa: BLE001
                print(f"MISMATCH seed={seed} kernel={kern} alpha={alpha} k={k} p={p} n={len(o) - 1}: {e!r}")
                raise SystemExit(1)
            runs += 1
        seed += 1
    print(f"fuzz ok: {seed - int(seed0)} workloads x {len(KERNELS)} kernels = {runs} runs bit-identical to the oracle")


if __name__ == "__main__":
    main(*(float(x) for x in sys.argv[1:2]), *(int(x) for x in sys.argv[2:3]))
