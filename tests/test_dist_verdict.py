"""World-size-2 and 4 gloo tests (CPU) of the collective partition's host logic.

sad_partition (include/sad.h) all-gathers, over the library's NCCL communicator, one block per
rank: its [p/world][p][2] sequence/residue counts per (shard, bucket) and a status tail
[operand overflow, input-error kind, output bytes, 0]; every rank then calls the same pure host
function, sad_exchange_verdict, on the same gathered bytes. Here the blocks are built from the
oracle's buckets (counts) and gathered over gloo, and every rank must take the
same decision: exchange with the oracle's count matrix, SAD_E_REPLAN when any rank overflowed,
SAD_E_NCCL naming the first rank with an input error, SAD_E_CAPACITY naming the rank whose output
buffer is short. The exchange sizes derived from the agreed matrix must then pair up across ranks
(what r sends to q is what q receives from r), which is what lets grouped ncclSend/ncclRecv match.
"""
import ctypes
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCENARIOS = ["ok", "overflow", "inputerr", "capacity"]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, p, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        from paper_0901_2742_b200 import _lib as L
        from paper_0901_2742_b200.runtime import exchange_sizes
        from synth import gen

        spec = gen.SPECS[3]
        a, o = gen.generate(spec, n=160 * p)
        n = len(o) - 1
        r = oracle.run(a, o, spec.alphabet, spec.k, p)
        sb = gen.shard_bounds(n, p)
        lens = np.diff(o)
        # the oracle's count matrix: shard s -> bucket b, sequences and residues
        want = np.zeros((p, p, 2), np.int64)
        for i in range(n):
            s = next(t for t in range(p) if sb[t] <= i < sb[t + 1])
            want[s, r.bucket[i], 0] += 1
            want[s, r.bucket[i], 1] += lens[i]
        pl = p // world
        B = pl * p * 2 + 4
        out = {}
        for scen in SCENARIOS:
            blk = np.zeros(B, np.int64)
            blk[: pl * p * 2] = want[rank * pl: (rank + 1) * pl].ravel()
            blk[pl * p * 2 + 2] = 1 << 40                           # a large output buffer
            if scen == "overflow" and rank == world - 1:
                blk[pl * p * 2 + 0] = 1
            if scen == "inputerr" and rank == 1:
                blk[pl * p * 2 + 1] = 2                             # a sequence shorter than k
            if scen == "capacity" and rank == 1:
                blk[pl * p * 2 + 2] = 1000                          # far too small
            t = torch.from_numpy(blk)
            parts = [torch.zeros_like(t) for _ in range(world)]
            dist.all_gather(parts, t)
            gathered = torch.cat(parts).numpy().copy()
            counts_all = np.zeros(p * p * 2, np.int64)
            who, kind = ctypes.c_int32(), ctypes.c_int32()
            rc = L.lib().sad_exchange_verdict(p, world, gathered.ctypes.data_as(ctypes.c_void_p),
                                              counts_all.ctypes.data_as(ctypes.c_void_p), ctypes.byref(who),
                                              ctypes.byref(kind))
            out[scen] = (int(rc), int(who.value), int(kind.value),
                         counts_all.reshape(p, p, 2).tolist() if rc == 0 else None)
            if rc == 0:
                ss, sr, rs, rr = exchange_sizes(p, world, rank, counts_all.reshape(p, p, 2))
                out["sizes"] = [ss.tolist(), sr.tolist(), rs.tolist(), rr.tolist()]
        out["want"] = want.tolist()
        q.put((rank, out))
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        import traceback
        q.put((rank, {"error": f"{e}\n{traceback.format_exc()}"}))


@pytest.mark.parametrize("world,p", [(2, 2), (2, 8), (4, 8)])
def test_exchange_verdict_agrees_on_every_rank(world, p):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, p, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
    for rk, out in res.items():
        assert "error" not in out, out.get("error")
    from paper_0901_2742_b200 import _lib as L
    expect = {"ok": (0, -1), "overflow": (L.SAD_E_REPLAN, -1), "inputerr": (L.SAD_E_NCCL, 1),
              "capacity": (L.SAD_E_CAPACITY, 1)}
    for scen in SCENARIOS:
        decisions = {rk: out[scen][:2] for rk, out in res.items()}
        assert len(set(decisions.values())) == 1, (scen, decisions)   # every rank decides the same
        assert decisions[0] == expect[scen], (scen, decisions[0])
    assert all(out["inputerr"][2] == 2 for out in res.values())     # the failing rank's error kind
    for rk, out in res.items():
        assert out["ok"][3] == out["want"], "the agreed count matrix is the oracle's"
    # what rank r sends to rank q is what q receives from r (sequences and residues)
    for r_ in range(world):
        for q_ in range(world):
            assert res[r_]["sizes"][0][q_] == res[q_]["sizes"][2][r_]
            assert res[r_]["sizes"][1][q_] == res[q_]["sizes"][3][r_]
