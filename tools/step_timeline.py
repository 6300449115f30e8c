"""Per-stage device timeline of one bench step (CUDA events between the API calls on the
library's stream), to separate kernel time from host-side gaps."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_0901_2742_b200.runtime import Context  # noqa: E402
from synth import gen  # noqa: E402


def main(cfg=4, p=8, kernel="tc", steps=5, mode="device"):
    """mode "host": inputs from pinned host memory (the bench's e2e path), keys read back at the end."""
    spec = gen.SPECS[cfg]
    a, o = gen.generate(spec)
    n = len(o) - 1
    dev = torch.device("cuda", 0)
    st = torch.cuda.current_stream(dev)
    d_a, d_o = torch.from_numpy(a).to(dev), torch.from_numpy(o).to(dev)
    h_a, h_o = torch.from_numpy(a).pin_memory().numpy(), torch.from_numpy(o).pin_memory().numpy()
    ctx = Context(spec.alphabet, spec.k, p, kernel=kernel)
    R = int(o[-1])
    names = ["load", "build_profiles", "rank_local", "rank_global", "partition_plan", "finish"]
    for it in range(steps + 2):
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(names) + 1)]
        host = []
        ev[0].record(st)
        t0 = time.perf_counter()
        if mode == "host":
            ctx.load(h_a, h_o, n, 0)
        else:
            ctx.load(d_a, d_o, n, 0, residues=R)
        ev[1].record(st); host.append(time.perf_counter() - t0)
        ctx.build_profiles()
        ev[2].record(st); host.append(time.perf_counter() - t0)
        anc = ctx.rank_local()
        ev[3].record(st); host.append(time.perf_counter() - t0)
        smp = ctx.rank_global(anc)
        ev[4].record(st); host.append(time.perf_counter() - t0)
        ctx.partition_plan(smp)
        ev[5].record(st); host.append(time.perf_counter() - t0)
        ctx.finish(None, sync=False)
        if mode == "host":
            ctx.out_keys().cpu()
        ev[6].record(st); host.append(time.perf_counter() - t0)
        torch.cuda.synchronize()
        if it >= 2:
            dev_ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(len(names))]
            print(f"step {it - 2}: total {ev[0].elapsed_time(ev[-1]):.3f} ms | " +
                  " ".join(f"{nm}={d:.3f}" for nm, d in zip(names, dev_ms)) +
                  " | host enqueue done at " + " ".join(f"{h * 1e3:.2f}" for h in host))
    st_ = ctx.stats()
    print("allpairs kernel ms/call", st_["allpairs_ms_total"] / max(st_["calls"], 1),
          "operand ms/call", st_["operand_ms_total"] / max(st_["calls"], 1))


if __name__ == "__main__":
    main(*(int(x) if x.isdigit() else x for x in sys.argv[1:]))
