"""Python driver of libsad.so: argument marshalling, torch-owned device memory, and the
rank-to-rank exchange steps over torch.distributed.

The method's arithmetic runs in the library's CUDA kernels. This module only
  * allocates the device buffers the library asks for (grow-only torch tensors),
  * passes the caller's CUDA stream,
  * moves the exchange buffers between ranks ("Send the k samples from each
    processor to all the processors", :74-76 gather/broadcast of the sample ranks, :77
    "Redistributed sequences among processors") with torch.distributed collectives
    (NCCL over NVLink on the GPU box; the same functions run on gloo/CPU in tests).
"""
from __future__ import annotations

import ctypes

import numpy as np
import torch
import torch.distributed as dist

from . import _lib as L

ALPHABETS = {"protein": L.SAD_PROTEIN20, "dna": L.SAD_DNA4}
KERNELS = {"tc": L.SAD_F_KERNEL_TC, "tc1": L.SAD_F_KERNEL_TC | L.SAD_F_TC_1SM,
           "tc8": L.SAD_F_KERNEL_TC | L.SAD_F_TC_INT8, "tc81": L.SAD_F_KERNEL_TC | L.SAD_F_TC_INT8 | L.SAD_F_TC_1SM,
           "tcfull": L.SAD_F_KERNEL_TC | L.SAD_F_TC_ALL_LAYERS,
           "tc8full": L.SAD_F_KERNEL_TC | L.SAD_F_TC_INT8 | L.SAD_F_TC_ALL_LAYERS,
           "alu": L.SAD_F_KERNEL_ALU}


def _vp(t) -> ctypes.c_void_p:
    if t is None:
        return ctypes.c_void_p(None)
    if isinstance(t, int):
        return ctypes.c_void_p(t)
    if isinstance(t, np.ndarray):
        return t.ctypes.data_as(ctypes.c_void_p)
    return ctypes.c_void_p(t.data_ptr())


# ----------------------------------------------------------------------------------------
# exchange steps (device-agnostic: CUDA tensors on NCCL, CPU tensors on gloo)
# ----------------------------------------------------------------------------------------

def all_gather_rows(local: torch.Tensor, world: int, group=None) -> torch.Tensor:
    """Concatenate every rank's `local` (same shape everywhere) in rank order."""
    local = local.contiguous()
    if world == 1:
        return local
    out = torch.empty((world * local.shape[0],) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    if local.is_cuda:
        dist.all_gather_into_tensor(out, local, group=group)
    else:
        dist.all_gather(list(out.chunk(world)), local, group=group)
    return out


def exchange_sizes(p: int, world: int, rank: int, counts_all: np.ndarray):
    """Per-peer send/recv sequence and residue counts (host logic of libsad.so)."""
    c = np.ascontiguousarray(counts_all, dtype=np.int64)
    ss, sr, rs, rr = (np.zeros(world, np.int64) for _ in range(4))
    L.call("sad_exchange_sizes", p, world, rank, _vp(c), _vp(ss), _vp(sr), _vp(rs), _vp(rr))
    return ss, sr, rs, rr


def pack_plan(p: int, world: int, rank: int, counts_all: np.ndarray) -> np.ndarray:
    c = np.ascontiguousarray(counts_all, dtype=np.int64)
    seg = np.zeros((p // world, p, 2), np.int64)
    L.call("sad_pack_plan", p, world, rank, _vp(c), _vp(seg))
    return seg


def all_to_all_v(send: torch.Tensor, send_sizes, recv_sizes, group=None) -> torch.Tensor:
    """Variable all-to-all of a flat tensor (rows of any width), split by rank."""
    recv = torch.empty((int(np.sum(recv_sizes)),) + tuple(send.shape[1:]), dtype=send.dtype, device=send.device)
    dist.all_to_all_single(recv, send.contiguous(), output_split_sizes=[int(x) for x in recv_sizes],
                           input_split_sizes=[int(x) for x in send_sizes], group=group)
    return recv


def upgma(D: torch.Tensor, stream: torch.cuda.Stream | None = None):
    """UPGMA guide tree of a float64 CUDA distance matrix (include/sad.h sad_upgma; D is destroyed).
    Returns host arrays (merges [n-1, 2], heights [n-1], sizes [n-1])."""
    n = int(D.shape[0])
    merges = torch.empty((max(n - 1, 1), 2), dtype=torch.int64, device=D.device)
    heights = torch.empty(max(n - 1, 1), dtype=torch.float64, device=D.device)
    sizes = torch.empty(max(n - 1, 1), dtype=torch.int64, device=D.device)
    wsb = int(L.lib().sad_upgma_workspace(n))
    ws = torch.empty(wsb + 256, dtype=torch.uint8, device=D.device)
    p_ws = (ws.data_ptr() + 255) // 256 * 256
    st = stream if stream is not None else torch.cuda.current_stream(D.device)
    L.check(L.lib().sad_upgma(_vp(D), n, _vp(merges), _vp(heights), _vp(sizes), ctypes.c_void_p(p_ws), wsb,
                              ctypes.c_void_p(st.cuda_stream)), "sad_upgma")
    st.synchronize()
    return merges[: n - 1].cpu().numpy(), heights[: n - 1].cpu().numpy(), sizes[: n - 1].cpu().numpy()


# ----------------------------------------------------------------------------------------
# the context
# ----------------------------------------------------------------------------------------

class Context:
    """One rank's view of the k-mer-rank domain decomposition (include/sad.h).

    kernel: "tc"  tcgen05 threshold-indicator GEMM, packed e2m1 operands, CTA pairs (default)
            "tc1" the same with one CTA per 128-row tile
            "tc8" uint8 operands (kind::i8), CTA pairs; "tc81" uint8, one CTA per tile
            "tcfull"/"tc8full" every threshold layer dense (no layer cap + sparse excess)
            "alu" CUDA-core min-sum
    """

    def __init__(self, alphabet: str, k: int, p: int, *, world: int = 1, rank: int = 0, device: int | None = None,
                 stream: torch.cuda.Stream | None = None, kernel: str = "tc", keep_sim: bool = False, group=None,
                 rank_mode: str = "ga", comm: bool = False, f1_cuda_cores: bool = False,
                 tile_split: bool = False):
        """comm: give the library its own NCCL communicator (sad_create with an id that rank 0 draws
        and torch.distributed broadcasts over `group`): the collective calls sad_rank / sad_partition
        then run every exchange themselves. Needed by run() when world > 1; with world == 1 it makes
        the exchange steps run through NCCL anyway (a single-rank communicator).
        tile_split (SAD_F_TILE_SPLIT, SURVEY §8(f) f2 across GPUs): every rank loads the whole input
        and keeps all p shards; only the all-pairs tiles are split over the world ranks and T summed
        over them on the communicator (comm=True; without it T holds the rank's partial sums)."""
        if not torch.cuda.is_available():
            raise RuntimeError("the k-mer-rank path needs a CUDA device (no CPU fallback)")
        if device is None:
            device = torch.cuda.current_device()
        self.device = torch.device("cuda", device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.alphabet, self.k, self.p, self.world, self.rank, self.group = alphabet, k, p, world, rank, group
        self.tile_world = world if tile_split else 1
        if tile_split:                      # the data path is world 1 on the whole input
            self.world, self.rank, self.pl = 1, 0, p
        else:
            self.pl = p // world
        if kernel not in KERNELS:
            raise ValueError(f"kernel must be one of {sorted(KERNELS)}, not {kernel!r}")
        if rank_mode not in ("ga", "samples"):
            raise ValueError(f"rank_mode must be 'ga' or 'samples', not {rank_mode!r}")
        flags = (L.SAD_F_KEEP_SIM if keep_sim else 0) | KERNELS[kernel] | (
            L.SAD_F_RANK_SAMPLES if rank_mode == "samples" else 0) | (L.SAD_F_F1_CUDA_CORES if f1_cuda_cores else 0) | (
            L.SAD_F_TILE_SPLIT if tile_split else 0)
        self.rank_mode = rank_mode
        self.kernel = kernel
        cfg = L.SadConfig(ALPHABETS[alphabet], k, p, world, rank, device, self.stream.cuda_stream, flags)
        h = ctypes.c_void_p()
        nid = None
        if comm:
            uid = (ctypes.c_uint8 * 128)()
            if rank == 0:
                L.call("sad_nccl_unique_id", uid)
            if world > 1:                      # rank 0's id to every rank (the only torch exchange)
                box = [bytes(uid)]
                dist.broadcast_object_list(box, src=0, group=group)
                ctypes.memmove(uid, box[0], 128)
            nid = uid
        self.comm = comm
        L.call("sad_create", ctypes.byref(cfg), nid, ctypes.byref(h))
        self._h = h
        self._bufs: dict[str, torch.Tensor] = {}
        self.rec_bytes = int(L.lib().sad_ancestor_record_bytes(h))
        self.counts_all = None
        self.bucket_sizes = None
        self.layout = None

    # -- memory ------------------------------------------------------------------------
    def _buf(self, name: str, nbytes: int, align: int = 1024) -> int:
        """Device pointer to a grow-only torch buffer of >= nbytes, aligned to `align`."""
        t = self._bufs.get(name)
        if t is None or t.numel() < nbytes + align:
            t = torch.empty(int(nbytes * 1.1) + align + 256, dtype=torch.uint8, device=self.device)
            self._bufs[name] = t
        base = t.data_ptr()
        return (base + align - 1) // align * align

    def _tensor(self, name: str, shape, dtype) -> torch.Tensor:
        n = int(np.prod(shape)) if len(shape) else 1
        key = f"t:{name}"
        t = self._bufs.get(key)
        if t is None or t.dtype != dtype or t.numel() < n:
            t = torch.empty(max(n, 1), dtype=dtype, device=self.device)
            self._bufs[key] = t
        return t[:n].view(*shape) if len(shape) else t[:1]

    def _call(self, name, *args):
        return L.call(name, self._h, *args, ctx=self._h)

    def close(self):
        if getattr(self, "_h", None):
            L.lib().sad_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- pipeline ------------------------------------------------------------------------
    def load(self, ascii_, offsets, n_global: int, first_index: int = 0, residues: int | None = None):
        """This rank's contiguous slice (numpy host arrays or CUDA tensors). For CUDA tensors pass
        `residues` (= offsets[-1]) to avoid a device read-back."""
        on_dev = isinstance(ascii_, torch.Tensor) and ascii_.is_cuda
        if on_dev:
            n_local = int(offsets.numel()) - 1
            R = int(residues) if residues is not None else int(offsets[-1].item())
            mem = L.SAD_MEM_DEVICE
        else:
            ascii_ = np.ascontiguousarray(ascii_, dtype=np.uint8)
            offsets = np.ascontiguousarray(offsets, dtype=np.int64)
            n_local = len(offsets) - 1
            R = int(offsets[-1])
            mem = L.SAD_MEM_HOST
            if ascii_.size == 0:
                ascii_ = np.zeros(1, np.uint8)
        self.n_local, self.n_global, self.first_index, self.R = n_local, n_global, first_index, R
        ws = ctypes.c_size_t()
        self._call("sad_workspace_size", n_local, R, ctypes.byref(ws))
        p_ws = self._buf("ws", ws.value)
        self._call("sad_load", _vp(ascii_), _vp(offsets), n_local, first_index, n_global, R, mem,
                   ctypes.c_void_p(p_ws), ws.value)
        return self

    def build_profiles(self):
        self._call("sad_build_profiles")

    def rank_local(self) -> torch.Tensor:
        ob = ctypes.c_size_t()
        self._call("sad_operand_size", ctypes.byref(ob))
        p_op = self._buf("operand", ob.value, align=1024)
        nrec = int(L.lib().sad_exchange_records(self._h))
        anc = self._tensor("anc", (nrec, self.rec_bytes), torch.uint8)
        self._call("sad_rank_local", ctypes.c_void_p(p_op), ob.value, _vp(anc))
        return anc

    def rank_global(self, anc_all: torch.Tensor) -> torch.Tensor:
        samples = self._tensor("samples", (max(self.pl * (self.p - 1), 1),), torch.int64)
        self._call("sad_rank_global", _vp(anc_all), _vp(samples))
        return samples[: self.pl * (self.p - 1)]

    def partition_plan(self, samples_all: torch.Tensor) -> torch.Tensor:
        counts = self._tensor("counts", (self.pl, self.p, 2), torch.int64)
        self._call("sad_partition_plan", _vp(samples_all if self.p > 1 else None), _vp(counts))
        return counts

    def pack(self, counts_all: np.ndarray):
        """Send side of the redistribution (world > 1): this rank's sequences grouped by
        destination. Returns (send_meta, send_res, send_seqs, send_res_bytes, recv_seqs, recv_res_bytes)."""
        c = np.ascontiguousarray(counts_all, dtype=np.int64)
        ss, sr, rs, rr = exchange_sizes(self.p, self.world, self.rank, c)
        send_meta = self._tensor("send_meta", (int(ss.sum()), 2), torch.int64)
        send_res = self._tensor("send_res", (max(int(sr.sum()), 1),), torch.uint8)
        self._call("sad_pack", _vp(c), _vp(send_meta), _vp(send_res))
        return send_meta, send_res[: int(sr.sum())], ss, sr, rs, rr

    def finish(self, counts_all, recv_meta=None, recv_res=None, sync: bool = True):
        """Receive side: merge into this rank's buckets (recv_* None for world == 1). With
        world == 1 counts_all may be None (the counts stay on the device); sync=False then
        returns None instead of the bucket sizes (no host synchronization)."""
        c = None if counts_all is None else np.ascontiguousarray(counts_all, dtype=np.int64)
        self.counts_all = c
        if recv_res is not None and recv_res.numel() == 0:
            recv_res = torch.zeros(1, dtype=torch.uint8, device=self.device)
        ob = ctypes.c_size_t()
        self._call("sad_output_size", _vp(c), ctypes.byref(ob))
        p_out = self._buf("out", ob.value, align=256)
        sizes = np.zeros(self.p, np.int64) if (sync or c is not None) else None
        self._call("sad_finish", _vp(c), _vp(recv_meta), _vp(recv_res), ctypes.c_void_p(p_out), ob.value, _vp(sizes))
        lay = np.zeros(6, np.int64)
        self._call("sad_output_layout", _vp(c), _vp(lay))
        self._out_ptr = p_out
        self.layout = lay
        self._keep = (recv_meta, recv_res)
        self.bucket_sizes = sizes
        return sizes

    def redistribute(self, counts_all: np.ndarray):
        """All-to-all of the sequences (world > 1) and the receive-side merge."""
        if self.world == 1:
            return self.finish(counts_all)
        send_meta, send_res, ss, sr, rs, rr = self.pack(counts_all)
        recv_meta = all_to_all_v(send_meta, ss, rs, self.group)
        recv_res = all_to_all_v(send_res, sr, rr, self.group)
        return self.finish(counts_all, recv_meta, recv_res)

    def run(self, sync: bool = True, residues_global: int | None = None):
        """One full step through the collective API (include/sad.h): sad_build_profiles ->
        sad_rank -> sad_partition. Returns the sizes of all p buckets (host); with world == 1 and
        sync=False nothing is read back (the step stays enqueued on the stream; no host
        synchronization at all) and None is returned. world > 1 needs comm=True; residues_global
        (all ranks' residues) sizes the output by the partition bound (sad_output_bound).
        SAD_E_REPLAN (the operand capacity grew) reruns the step."""
        if self.world > 1 and not self.comm:
            return self.run_split()
        for attempt in range(4):
            try:
                return self._step(sync, residues_global)
            except L.SadError as e:
                if e.code != L.SAD_E_REPLAN or attempt == 3:
                    raise

    def _step(self, sync, residues_global):
        self._call("sad_build_profiles")
        ob = ctypes.c_size_t()
        self._call("sad_operand_size", ctypes.byref(ob))
        p_op = self._buf("operand", ob.value, align=1024)
        self._call("sad_rank", ctypes.c_void_p(p_op), ob.value)
        if self.world > 1 and residues_global is None:
            residues_global = self._residues_global()
        obytes = ctypes.c_size_t()
        self._call("sad_output_bound", int(residues_global or self.R), ctypes.byref(obytes))
        p_out = self._buf("out", obytes.value, align=256)
        want = sync or self.world > 1
        sizes = np.zeros(self.p, np.int64) if want else None
        self._call("sad_partition", ctypes.c_void_p(p_out), obytes.value, _vp(sizes))
        self._out_ptr = p_out
        lay = np.zeros(6, np.int64)
        self._call("sad_output_layout", None, _vp(lay))
        self.layout = lay
        self.bucket_sizes = sizes
        return sizes

    def _residues_global(self) -> int:
        """Sum of every rank's residues (once per layout; torch.distributed over `group`)."""
        key = (self.n_local, self.R)
        if getattr(self, "_rg_key", None) != key:
            t = torch.tensor([self.R], dtype=torch.int64,
                             device=self.device if dist.get_backend(self.group) == "nccl" else "cpu")
            dist.all_reduce(t, group=self.group)
            self._rg, self._rg_key = int(t.item()), key
        return self._rg

    def run_split(self):
        """One full step through the split API, the exchanges done here over torch.distributed
        (gloo on CPU tests, NCCL on GPUs): used for world > 1 contexts without a library
        communicator."""
        for attempt in range(4):
            self.build_profiles()
            try:
                anc = self.rank_local()
                break
            except L.SadError as e:
                if e.code != L.SAD_E_REPLAN or attempt == 3:
                    raise
        anc_all = all_gather_rows(anc, self.world, self.group)
        samples = self.rank_global(anc_all)
        samples_all = all_gather_rows(samples, self.world, self.group) if self.p > 1 else samples
        counts = self.partition_plan(samples_all)
        if self.world == 1:
            return self.finish(None)
        counts_all = all_gather_rows(counts, self.world, self.group).cpu().numpy()   # the one D2H of the plan
        return self.redistribute(counts_all.reshape(self.p, self.p, 2))

    # -- CUDA graph of one device-resident step (world == 1, no communicator) --------------
    def capture_step(self, d_ascii: torch.Tensor, d_offsets: torch.Tensor, residues: int):
        """Capture load (device inputs) + one whole step into a CUDA graph on this context's stream
        (which must not be the legacy default stream). Run one eager step on the same inputs first
        (it sizes every buffer and the operand capacity). Returns the torch.cuda.CUDAGraph; after
        each replay() has completed, call graph_account() to add the replay's stage times."""
        if self.world != 1 or self.comm:
            raise ValueError("graph capture needs world == 1 without a communicator")
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=self.stream, capture_error_mode="relaxed"):
            self.load(d_ascii, d_offsets, self.n_global, self.first_index, residues=residues)
            self._step(False, None)
        return g

    def graph_account(self):
        self._call("sad_graph_account")

    def bucket_sizes_now(self) -> np.ndarray:
        out = np.zeros(self.p, np.int64)
        self._call("sad_get_bucket_sizes", _vp(out))
        return out

    @property
    def key_index_bits(self) -> int:
        """Index bits of the rank keys: key = (rank value << bits) + source index (sad_key_index_bits)."""
        return int(L.lib().sad_key_index_bits(self._h))

    def key_index(self, keys) -> np.ndarray:
        """Source indices of uint64 rank keys (pivots, bucket keys)."""
        return (np.asarray(keys, dtype=np.uint64) & np.uint64((1 << self.key_index_bits) - 1)).astype(np.int64)

    def load_report(self) -> dict:
        """the largest bucket against the PSRS bound (sad_get_load_report)."""
        r = np.zeros(6, np.int64)
        self._call("sad_get_load_report", _vp(r))
        return {"max_bucket": int(r[0]), "w": int(r[1]), "bound_2w_plus_p": int(r[2]), "holds": bool(r[3]),
                "p_divides_w": bool(r[4]), "below_2w": bool(r[5])}

    # -- results -------------------------------------------------------------------------
    def out_keys(self) -> torch.Tensor:
        """uint64 keys (as int64) of all owned buckets, back to back, each in key order (device view)."""
        n = int(self.layout[0])
        t = self._bufs["out"]
        off = self._out_ptr - t.data_ptr() + int(self.layout[2])
        return t[off: off + 8 * n].view(torch.int64)

    def local_rank(self, shard: int) -> np.ndarray:
        w = self.shard_size(shard)
        out = np.zeros(w, np.uint64)
        self._call("sad_get_local_rank", shard, _vp(out), w)
        return out

    def shard_size(self, shard: int) -> int:
        base, extra = divmod(self.n_global, self.p)
        s = self.rank * self.pl + shard
        return base + (1 if s < extra else 0)

    def ancestors(self):
        loc = np.zeros(self.p, np.int64)
        ga = ctypes.c_int64()
        self._call("sad_get_ancestors", _vp(loc), ctypes.byref(ga))
        return loc, ga.value

    def ranks(self, shard: int):
        w = self.shard_size(shard)
        S, d, key = np.zeros(w, np.uint32), np.zeros(w, np.uint32), np.zeros(w, np.uint64)
        self._call("sad_get_ranks", shard, _vp(S), _vp(d), _vp(key), w)
        return S, d, key

    def sorted(self, shard: int) -> np.ndarray:
        w = self.shard_size(shard)
        out = np.zeros(w, np.int64)
        self._call("sad_get_sorted", shard, _vp(out), w)
        return out

    def pivots(self) -> np.ndarray:
        out = np.zeros(max(self.p - 1, 1), np.uint64)
        self._call("sad_get_pivots", _vp(out))
        return out[: self.p - 1]

    def bucket(self, b: int):
        n, r = ctypes.c_int64(), ctypes.c_int64()
        self._call("sad_get_bucket", b, None, None, None, None, 0, 0, ctypes.byref(n), ctypes.byref(r))
        idx, key = np.zeros(n.value + 1, np.int64), np.zeros(n.value + 1, np.uint64)
        res, off = np.zeros(max(r.value, 1), np.uint8), np.zeros(n.value + 1, np.int64)
        self._call("sad_get_bucket", b, _vp(idx), _vp(key), _vp(res), _vp(off), n.value + 1, r.value,
                   ctypes.byref(n), ctypes.byref(r))
        return idx[: n.value], key[: n.value], res[: r.value], off

    def bucket_view(self, b: int):
        """Device view of owned bucket b: (residue pointer, absolute offsets pointer, n, residues)."""
        res, off = ctypes.c_void_p(), ctypes.c_void_p()
        n, r = ctypes.c_int64(), ctypes.c_int64()
        self._call("sad_get_bucket_view", b, ctypes.byref(res), ctypes.byref(off), ctypes.byref(n), ctypes.byref(r))
        return res.value, off.value, n.value, r.value

    def bucket_distances(self, b: int, kernel: str | None = None):
        """the k-mer distance matrix 1 - F of owned bucket b (the input of
        the per-bucket aligner's guide tree), computed on this device by a child
        context (one shard = the bucket, similarities kept). Returns (D float32 [n, n] CUDA tensor
        in the bucket's order, S uint16 [n, n] host array)."""
        res, off, n, r = self.bucket_view(b)
        child = Context(self.alphabet, self.k, 1, device=self.device.index, stream=self.stream,
                        kernel=kernel or self.kernel, keep_sim=True)
        child.load_device_view(res, off, n, r)
        child.build_profiles()
        child.rank_local()
        D = torch.empty((n, n), dtype=torch.float32, device=self.device)
        child._call("sad_get_distance", 0, _vp(D), n * n)
        S = child.similarity(0)
        child.close()
        return D, S

    def bucket_guide_tree(self, b: int, kernel: str | None = None):
        """the UPGMA guide tree of owned bucket b on this device (sad_upgma on
        the bucket's float64 k-mer distances). Returns host arrays (merges [n-1, 2] cluster ids,
        heights [n-1], sizes [n-1]); leaves are positions in the bucket's order."""
        res, off, n, r = self.bucket_view(b)
        child = Context(self.alphabet, self.k, 1, device=self.device.index, stream=self.stream,
                        kernel=kernel or self.kernel, keep_sim=True)
        child.load_device_view(res, off, n, r)
        child.build_profiles()
        child.rank_local()
        D = torch.empty((n, n), dtype=torch.float64, device=self.device)
        child._call("sad_get_distance_f64", 0, _vp(D), n * n)
        out = upgma(D, self.stream)
        child.close()
        return out

    def load_device_view(self, res_ptr: int, off_ptr: int, n: int, residues: int):
        """Load n sequences from device memory whose offsets start at an arbitrary base (a bucket
        view of another context); source indices 0..n-1."""
        self.n_local, self.n_global, self.first_index, self.R = n, n, 0, residues
        ws = ctypes.c_size_t()
        self._call("sad_workspace_size", n, residues, ctypes.byref(ws))
        p_ws = self._buf("ws", ws.value)
        self._call("sad_load", ctypes.c_void_p(res_ptr), ctypes.c_void_p(off_ptr), n, 0, n, residues,
                   L.SAD_MEM_DEVICE_REBASE, ctypes.c_void_p(p_ws), ws.value)
        return self

    def similarity(self, shard: int) -> np.ndarray:
        w = self.shard_size(shard)
        out = np.zeros(w * w, np.uint16)
        self._call("sad_get_similarity", shard, _vp(out), w * w)
        return out.reshape(w, w)

    def profile_info(self):
        a, b, c = (np.zeros(self.pl, np.int64) for _ in range(3))
        self._call("sad_get_profile_info", _vp(a), _vp(b), _vp(c))
        return a, b, c

    def stats(self):
        ms = np.zeros(2, np.float64)
        cnt = np.zeros(4, np.int64)
        self._call("sad_get_stats", _vp(ms), _vp(cnt))
        return {"allpairs_ms_total": float(ms[0]), "operand_ms_total": float(ms[1]), "calls": int(cnt[0]),
                "pairs": int(cnt[1]), "dense_macs": int(cnt[2]), "launches": int(cnt[3])}

    def reset_stats(self):
        self._call("sad_reset_stats")

    def selftest_fixed_point(self, max_den: int = 8000) -> int:
        bad = ctypes.c_int64()
        self._call("sad_selftest_fixed_point", max_den, ctypes.byref(bad))
        return bad.value


class Pipeline:
    """End-to-end steps over host inputs, double-buffered (world == 1): `depth` contexts, each on its
    own stream, take the steps in turn, so that the pinned host-to-device copy and k-mer counts of
    step k+1 (sad_load, copy engine + K1/K2) run while the device works on step k, and the keys of
    step k are read back (device-to-host into pinned memory) while step k+1 runs. Every step is a
    complete sad_load .. sad_partition over its own inputs; submit() returns once the step's inputs
    have been copied (the host buffers may then be reused), collect() returns the oldest step's keys
    (pinned host tensor, every owned bucket back to back in key order) and bucket sizes."""

    def __init__(self, alphabet: str, k: int, p: int, *, depth: int = 2, device: int | None = None, **kw):
        if depth < 1:
            raise ValueError("depth must be >= 1")
        if kw.get("world", 1) != 1:
            raise ValueError("Pipeline overlaps whole steps of one rank (world == 1)")
        dev = torch.device("cuda", device if device is not None else torch.cuda.current_device())
        self.ctx = [Context(alphabet, k, p, device=dev.index, stream=torch.cuda.Stream(dev), **kw) for _ in range(depth)]
        self._next = 0
        self._pending = []
        self._host = {}

    def submit(self, ascii_, offsets, n_global: int | None = None, first_index: int = 0):
        if len(self._pending) == len(self.ctx):
            raise RuntimeError("every context holds an uncollected step: collect() first")
        c = self.ctx[self._next]
        self._next = (self._next + 1) % len(self.ctx)
        n = len(offsets) - 1
        c.load(ascii_, offsets, n if n_global is None else n_global, first_index)
        c.run(sync=False)                     # world == 1: the step is enqueued, nothing read back
        keys = c.out_keys()
        h = self._host.get(id(c))
        if h is None or h.shape != keys.shape:
            h = torch.empty(keys.shape, dtype=keys.dtype, pin_memory=True)
            self._host[id(c)] = h
        with torch.cuda.stream(c.stream):
            h.copy_(keys, non_blocking=True)  # D2H of the step's result, ordered after the step
            ev = torch.cuda.Event()
            ev.record(c.stream)
        self._pending.append((c, h, ev))

    def collect(self):
        c, h, ev = self._pending.pop(0)
        ev.synchronize()
        return h, c.bucket_sizes_now()

    def close(self):
        for c in self.ctx:
            c.close()
