"""World-size-2 (and 4) CPU tests of the multi-rank exchange path over gloo.

The device kernels cannot run here, so each rank's kernel outputs (sorted shard keys,
sample keys, count matrix rows, packed send buffers) are emulated from the oracle's
per-shard results, and everything the product does BETWEEN kernels runs for real:
runtime.all_gather_rows (ancestor records, samples, counts), the library's pure host
planners sad_exchange_sizes / sad_pack_plan, and runtime.all_to_all_v for the
{key, L} metadata and the residue bytes. The receiving rank's merge is emulated by a
key sort (what sad_finish's kernel does) and must reproduce the oracle's buckets.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, p, cfg_n, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import oracle
        from paper_0901_2742_b200.runtime import all_gather_rows, all_to_all_v, exchange_sizes, pack_plan
        from synth import gen

        spec = gen.SPECS[2]
        a, o = gen.generate(spec, n=cfg_n)
        n = len(o) - 1
        r = oracle.run(a, o, spec.alphabet, spec.k, p)
        key = np.array([(oracle.q(int(s), int(d)) << 31) + i for i, (s, d) in enumerate(zip(r.S, r.den))],
                       dtype=np.uint64)
        L = np.diff(o)
        sb = gen.shard_bounds(n, p)
        pl = p // world
        mine = range(rank * pl, (rank + 1) * pl)

        # a5: ancestor records (emulated: source index in the first 8 bytes) gathered in shard order
        rec = torch.zeros((pl, 32), dtype=torch.uint8)
        for j, s in enumerate(mine):
            rec[j, :8] = torch.from_numpy(np.array([r.anc[s]], np.int64).view(np.uint8))
        recs = all_gather_rows(rec, world)
        got = recs[:, :8].contiguous().view(torch.int64).flatten().tolist()
        assert got == r.anc.tolist(), (got, r.anc.tolist())

        # a8/a9: samples of my shards (positions floor(j w / p) of each sorted shard), gathered
        srt = [r.sorted[sb[s]: sb[s + 1]] for s in range(p)]
        smp = []
        for s in mine:
            w = sb[s + 1] - sb[s]
            smp += [int(key[srt[s][(j * w) // p - 1]]) for j in range(1, p)]
        smp_all = all_gather_rows(torch.tensor(np.array(smp, np.uint64).view(np.int64)), world)
        assert (smp_all.numpy().view(np.uint64) & np.uint64(0x7FFFFFFF)).tolist() == r.samples.tolist()

        # a10: count rows of my shards (sequences, residues per bucket), gathered to every rank
        cnt = np.zeros((pl, p, 2), np.int64)
        for j, s in enumerate(mine):
            for i in srt[s]:
                cnt[j, r.bucket[i], 0] += 1
                cnt[j, r.bucket[i], 1] += L[i]
        counts_all = all_gather_rows(torch.from_numpy(cnt), world).numpy().reshape(p, p, 2)

        # a11: the library's host planners + the real all-to-all
        ss, sr, rs, rr = exchange_sizes(p, world, rank, counts_all)
        seg = pack_plan(p, world, rank, counts_all)
        meta = np.zeros((int(ss.sum()), 2), np.int64)
        res = np.zeros(max(int(sr.sum()), 1), np.uint8)
        for j, s in enumerate(mine):                       # emulate k_pack
            for b in range(p):
                sl = [i for i in srt[s] if r.bucket[i] == b]
                so, ro = seg[j, b]
                for t, i in enumerate(sl):
                    meta[so + t] = [np.int64(key[i].view(np.int64)), L[i]]
                    res[ro: ro + L[i]] = a[o[i]: o[i + 1]]
                    ro += L[i]
        rmeta = all_to_all_v(torch.from_numpy(meta), ss, rs)
        rres = all_to_all_v(torch.from_numpy(res[: int(sr.sum())]), sr, rr).numpy()
        assert rmeta.shape[0] == int(rs.sum()) and rres.size == int(rr.sum())

        # receive-side merge (emulates sad_finish): sort by key, gather residues
        k_in = rmeta[:, 0].numpy().view(np.uint64)
        L_in = rmeta[:, 1].numpy()
        src = np.concatenate([[0], np.cumsum(L_in)])
        order = np.argsort(k_in, kind="stable")
        idx = (k_in[order] & np.uint64(0x7FFFFFFF)).astype(np.int64)
        want = [i for b in mine for i in r.buckets()[b]]
        assert idx.tolist() == want
        seqs = gen.to_strings(a, o)
        got_seqs = [bytes(rres[src[t]: src[t + 1]]).decode() for t in order]
        assert got_seqs == [seqs[i] for i in want]
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as ex:  # noqa: BLE001
        import traceback
        q.put((rank, "".join(traceback.format_exception(ex))))


@pytest.mark.parametrize("world,p,n", [(2, 2, 300), (2, 8, 700), (4, 8, 800)])
def test_exchange_path_gloo(world, p, n):
    from paper_0901_2742_b200 import build
    build.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, p, n, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    results = dict(q.get(timeout=300) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
    assert all(v == "ok" for v in results.values()), results
