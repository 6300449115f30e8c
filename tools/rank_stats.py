"""centralized rank over all N (one shard, the N x N all-pairs on the tensor
cores) next to the globalized rank against the k*p samples (f1, p shards), and Table 1's
statistics. Prints one JSON line.

    python tools/rank_stats.py [config=4] [p=8] [n=0 (full config)]
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0901_2742_b200 import stats  # noqa: E402
from paper_0901_2742_b200.runtime import Context  # noqa: E402
from synth import gen  # noqa: E402


def main(cfg=4, p=8, n=0):
    spec = gen.SPECS[cfg]
    a, o = gen.generate(spec, n=n or None)
    N = len(o) - 1
    dev = torch.device("cuda", 0)
    out = {"workload": f"{spec.name} N={N} {spec.alphabet} k={spec.k}", "p_globalized": p}
    # centralized: one shard holding all N sequences
    c = Context(spec.alphabet, spec.k, 1, kernel="tc")
    c.load(a, o, N, 0)
    c.run()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    c.load(a, o, N, 0)
    c.run()
    torch.cuda.synchronize()
    out["centralized_step_ms"] = (time.perf_counter() - t0) * 1e3
    out["centralized_pairs"] = N * (N - 1) // 2
    Tc = c.local_rank(0)
    c.close()
    # globalized: rank against the k*p samples
    g = Context(spec.alphabet, spec.k, p, kernel="tc", rank_mode="samples")
    g.load(a, o, N, 0)
    g.run()
    keys = np.concatenate([g.ranks(s)[2] for s in range(p)])
    dbar = (keys.astype(np.uint64) >> np.uint64(31)).astype(np.float64)
    g.close()
    Rc = stats.rank_R(stats.centralized_D(Tc, N))
    Rg = stats.rank_R(stats.globalized_D(dbar))
    out["table1"] = stats.rank_stats(Rc, Rg)
    rc_order, rg_order = np.argsort(np.argsort(Rc)), np.argsort(np.argsort(Rg))
    out["spearman"] = float(np.corrcoef(rc_order, rg_order)[0, 1])
    print(json.dumps(out))


if __name__ == "__main__":
    main(*(int(x) for x in sys.argv[1:]))
